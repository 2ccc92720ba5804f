"""Row-window sharding across GPUs (north-star subsystem 4).

Row windows own disjoint output rows (reference executors.py:169), and windows,
features and selector decisions depend only on a window's own rows
(windows.py:90-105).  So a matrix is split into contiguous window ranges,
balanced by nnz; each rank partitions its row slice locally (bit-identical to
the corresponding windows of the global partition) and computes its output
rows; features for the next layer are exchanged with one all-gather.

The collective is torch.distributed (NCCL on GPUs, gloo in CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch

from .matrices import DeviceCsr


def shard_window_ranges(row_ptr, n_rows: int, world: int, wh: int = 16) -> list[tuple[int, int]]:
    """Split windows [0, W) into `world` contiguous ranges with ~equal nnz.

    Boundary r is the first window whose starting entry offset reaches r*nnz/world,
    snapped to whole windows; deterministic and identical on every rank."""
    rp = row_ptr.cpu().numpy() if isinstance(row_ptr, torch.Tensor) else np.asarray(row_ptr)
    W = -(-n_rows // wh)
    starts = rp[np.minimum(np.arange(W + 1) * wh, n_rows)].astype(np.int64)  # entry offset at each window start
    nnz = int(starts[-1])
    bounds = [0]
    for r in range(1, world):
        target = (nnz * r) // world
        b = int(np.searchsorted(starts, target, side="left"))
        bounds.append(min(max(b, bounds[-1]), W))
    bounds.append(W)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def row_slice(a: DeviceCsr, r0: int, r1: int) -> DeviceCsr:
    """Rows [r0, r1) of a DeviceCsr (all columns kept), re-based row_ptr."""
    e0 = int(a.row_ptr[r0])
    e1 = int(a.row_ptr[r1])
    out = DeviceCsr(r1 - r0, a.num_cols, (a.row_ptr[r0:r1 + 1] - e0).contiguous(), a.col_idx[e0:e1],
                    a.values[e0:e1])
    if getattr(a, "values_f64", None) is not None:
        out.values_f64 = a.values_f64[e0:e1]
    return out


def allgather_rows(local: torch.Tensor, ranges, n_rows: int, wh: int = 16, group=None) -> torch.Tensor:
    """Ragged all-gather of per-rank output rows (padded to the largest shard) -> full [n_rows, d]."""
    import torch.distributed as dist

    world = len(ranges)
    rows = [min(b * wh, n_rows) - a * wh for a, b in ranges]
    maxr = max(rows) if rows else 0
    d = local.shape[1]
    send = torch.zeros((maxr, d), dtype=local.dtype, device=local.device)
    send[: local.shape[0]] = local
    recv = torch.empty((world * maxr, d), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(recv, send, group=group)
    else:  # gloo (CPU tests): list form
        dist.all_gather(list(recv.chunk(world)), send, group=group)
    parts = [recv[i * maxr: i * maxr + rows[i]] for i in range(world)]
    return torch.cat(parts, 0)


class _GatherRows(torch.autograd.Function):
    @staticmethod
    def forward(ctx, local, shard):
        ctx.shard = shard
        return shard.all_gather_rows(local)

    @staticmethod
    def backward(ctx, g):
        s = ctx.shard
        return g[s.row0:s.row1].contiguous(), None


class Shard:
    """This rank's contiguous row range [row0, row1) of a row-window-sharded operator plus
    the collectives the sharded GCN needs: all-gather of output rows between
    layers (ragged, padded to the largest shard) and all-reduce(sum) of grad_W."""

    def __init__(self, ranges, rank: int, n_rows: int, wh: int = 16, group=None):
        self.ranges = ranges
        self.rank = rank
        self.world = len(ranges)
        self.n_rows = n_rows
        self.wh = wh
        self.group = group
        self.row0 = min(ranges[rank][0] * wh, n_rows)
        self.row1 = min(ranges[rank][1] * wh, n_rows)

    @classmethod
    def from_operator(cls, a: DeviceCsr, world: int, rank: int, wh: int = 16, group=None) -> "Shard":
        return cls(shard_window_ranges(a.row_ptr, a.num_rows, world, wh), rank, a.num_rows, wh, group)

    def local_operator(self, a: DeviceCsr) -> DeviceCsr:
        """This rank's rows of A.  A row slice is not symmetric itself; `global_symmetric` records
        that the full operator is, so the backward can reuse the forward windows (A^T = A)."""
        loc = row_slice(a, self.row0, self.row1)
        loc.global_symmetric = bool(getattr(a, "symmetric", False) or getattr(a, "global_symmetric", False))
        return loc

    def all_gather_rows(self, local: torch.Tensor) -> torch.Tensor:
        return allgather_rows(local.contiguous(), self.ranges, self.n_rows, self.wh, self.group)

    def all_gather_rows_autograd(self, local: torch.Tensor) -> torch.Tensor:
        return _GatherRows.apply(local, self)

    def all_reduce(self, t: torch.Tensor) -> None:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def embed_rows(self, local: torch.Tensor) -> torch.Tensor:
        """A full-height tensor holding `local` in this rank's rows (zeros elsewhere)."""
        full = torch.zeros((self.n_rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        full[self.row0:self.row1] = local
        return full
