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

import os
from datetime import timedelta

import numpy as np
import torch

from .matrices import DeviceCsr

NCCL_TIMEOUT_S = float(os.environ.get("HCS_NCCL_TIMEOUT_S", "600"))


def init_process_group(backend: str = "nccl", device: torch.device | None = None, timeout_s: float | None = None):
    """Join the job's process group (one process per GPU; RANK/WORLD_SIZE/MASTER_* from the
    launcher).  NCCL failure handling: TORCH_NCCL_ASYNC_ERROR_HANDLING=1 makes a failed or timed
    out collective abort the communicator and raise in every rank (instead of a silent hang),
    and every collective gets a deadline of HCS_NCCL_TIMEOUT_S seconds (default 600)."""
    import torch.distributed as dist

    if backend == "nccl":
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    kw = {"timeout": timedelta(seconds=timeout_s or NCCL_TIMEOUT_S)}
    if backend == "nccl" and device is not None:
        kw["device_id"] = device
    dist.init_process_group(backend, **kw)
    if backend == "nccl":
        reserve_sms_for_exchange()


NCCL_RESERVED_SMS = 16


def reserve_sms_for_exchange(reserved: int | None = None) -> int:
    """Leave `reserved` SMs (HCS_NCCL_RESERVED_SMS, default 16) out of every tile launch, so the NCCL
    kernels of the overlapped exchange (part k's all-gather under part k+1's SpMM) find free SMs: a
    tile CTA fills its SM's shared memory and most of its registers.  Returns the tile CTAs per launch."""
    from . import _lib

    if reserved is None:
        reserved = int(os.environ.get("HCS_NCCL_RESERVED_SMS", str(NCCL_RESERVED_SMS)))
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    ctas = max(1, sms - max(0, reserved)) if reserved > 0 else 0
    _lib.call("hcs_set_tile_grid", ctas)
    return ctas or sms


def shard_window_ranges(row_ptr, n_rows: int, world: int, wh: int = 16,
                        window_cost=None) -> list[tuple[int, int]]:
    """Split windows [0, W) into `world` contiguous ranges with ~equal nnz -- or, given a per-window
    cost (window_costs), ~equal cost.

    Boundary r is the first window whose prefix (entries, or cost) reaches r/world of the total,
    snapped to whole windows; deterministic and identical on every rank."""
    W = -(-n_rows // wh)
    if window_cost is not None:
        c = np.asarray(window_cost, dtype=np.float64)
        if c.shape != (W,):
            raise ValueError(f"window_cost must have one entry per window ({W}), got {c.shape}")
        starts = np.zeros(W + 1, dtype=np.float64)
        np.cumsum(c, out=starts[1:])
        total = float(starts[-1])
        targets = [total * r / world for r in range(1, world)]
    else:
        rp = row_ptr.cpu().numpy() if isinstance(row_ptr, torch.Tensor) else np.asarray(row_ptr)
        starts = rp[np.minimum(np.arange(W + 1) * wh, n_rows)].astype(np.int64)  # entry offset at each window
        nnz = int(starts[-1])
        targets = [(nnz * r) // world for r in range(1, world)]
    bounds = [0]
    for target in targets:
        b = int(np.searchsorted(starts, target, side="left"))
        bounds.append(min(max(b, bounds[-1]), W))
    bounds.append(W)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


# Measured B200 cost of the two paths (profiles/r02_shard_compute.txt): the tile
# kernel moves one X row slice per condensed column (C5: ~31 ps per column at N = 128), the scalar
# kernel one per entry with less reuse (~75 ps per entry); a window also pays a fixed launch share.
TILE_COL_COST = 1.0
SCALAR_ENTRY_COST = 2.4
WINDOW_COST = 4.0


def window_costs(windows, codes) -> np.ndarray:
    """Per-window cost for shard_window_ranges: TILE windows by condensed columns, SCALAR windows
    by entries (the nnz balance alone left C5's slowest of 8 shards 22 % above the mean)."""
    ncols = windows.ncols().to(torch.float64)
    nnz = windows.nnz_per_window().to(torch.float64)
    tile = torch.as_tensor(np.asarray(codes), device=ncols.device).to(torch.bool)
    cost = torch.where(tile, TILE_COL_COST * ncols, SCALAR_ENTRY_COST * nnz) + WINDOW_COST * (nnz > 0)
    return cost.cpu().numpy()


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

    def __init__(self, ranges, rank: int, n_rows: int, wh: int = 16, group=None, window_starts=None):
        self.ranges = ranges
        self.rank = rank
        self.world = len(ranges)
        self.n_rows = n_rows
        self.wh = wh
        self.group = group
        self.row0 = min(ranges[rank][0] * wh, n_rows)
        self.row1 = min(ranges[rank][1] * wh, n_rows)
        # entry offset at every global window start (nnz-balanced exchange parts); None -> by count
        self.window_starts = None if window_starts is None else np.asarray(window_starts, dtype=np.int64)
        self._spans: dict = {}

    @classmethod
    def from_operator(cls, a: DeviceCsr, world: int, rank: int, wh: int = 16, group=None,
                      window_cost=None) -> "Shard":
        rp = a.row_ptr.cpu().numpy() if isinstance(a.row_ptr, torch.Tensor) else np.asarray(a.row_ptr)
        W = -(-a.num_rows // wh)
        starts = rp[np.minimum(np.arange(W + 1) * wh, a.num_rows)]
        return cls(shard_window_ranges(rp, a.num_rows, world, wh, window_cost), rank, a.num_rows, wh, group, starts)

    def part_spans(self, parts: int) -> list[list[tuple[int, int]]]:
        """Every rank's `parts` exchange parts as LOCAL window bounds [(lw0, lw1)] (contiguous,
        ~equal nnz when the window starts are known); identical on every rank, so each rank knows
        where every peer's part lands without a count exchange."""
        if parts not in self._spans:
            out = []
            for a, b in self.ranges:
                if self.window_starts is not None and b > a:
                    st = self.window_starts[a:b + 1]
                    tg = st[0] + (np.arange(1, parts) * (st[-1] - st[0])) // parts
                    cuts = [0] + [int(v) for v in np.searchsorted(st, tg, side="left")] + [b - a]
                else:
                    cuts = [((b - a) * k) // parts for k in range(parts + 1)]
                cuts = np.maximum.accumulate(np.minimum(cuts, b - a))
                out.append([(int(cuts[k]), int(cuts[k + 1])) for k in range(parts)])
            self._spans[parts] = out
        return self._spans[parts]

    def rank_rows(self, r: int) -> tuple[int, int]:
        a, b = self.ranges[r]
        return min(a * self.wh, self.n_rows), min(b * self.wh, self.n_rows)

    def start_gather(self, local_rows: torch.Tensor, counts: list[int]):
        """Async all-gather of this rank's `local_rows` (counts[r] rows on rank r, padded to the
        largest); returns (work, recv, maxr) for finish_gather."""
        import torch.distributed as dist

        maxr = max(max(counts), 1)
        d = local_rows.shape[1]
        send = torch.zeros((maxr, d), dtype=local_rows.dtype, device=local_rows.device)
        send[: local_rows.shape[0]] = local_rows
        recv = torch.empty((self.world * maxr, d), dtype=local_rows.dtype, device=local_rows.device)
        if dist.get_backend(self.group) == "nccl":
            work = dist.all_gather_into_tensor(recv, send, group=self.group, async_op=True)
        else:
            work = dist.all_gather(list(recv.chunk(self.world)), send, group=self.group, async_op=True)
        return work, recv, maxr

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
