"""LOA layout reorganisation on the GPU (reference layout.py; paper Alg. 5/6).

  sort_by_min_neighbor     layout.py:99-109   device stable sort of (min neighbour, id)
  build_windows_optimized  layout.py:186-263  K8 hcs_loa: one persistent CTA runs the
  build_windows_basic      layout.py:142-183  greedy loop (identical groupings, as the
                                              reference guarantees for its two builders)
  reorder                  layout.py:266-274  induced permutation + K9 permute_symmetric
  permute_symmetric        matrices.py:310-318 P A P^T on the device

Groupings are bit-exact with the reference (integer algorithm).  The GPU builder
computes every candidate's cns by intersection (pull), so the reference's
check_counters invariant holds by construction; per-candidate `audit` callbacks
are a host-side debugging hook and are not supported on the device builder.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .matrices import DeviceCsr, Graph, to_device_csr
from .windows import WINDOW_HEIGHT


class WindowGrouping:
    """Ordered vertex groups (layout.py:25-61); device arrays flat/gptr, host lists on demand."""

    def __init__(self, groups, num_vertices: int):
        self.num_vertices = int(num_vertices)
        if isinstance(groups, tuple) and len(groups) == 2 and isinstance(groups[0], torch.Tensor):
            self.flat, self.gptr = groups
            self._groups = None
        else:
            self._groups = [list(map(int, g)) for g in groups]
            flat = [v for g in self._groups for v in g]
            self.flat = torch.tensor(flat, dtype=torch.int64)
            self.gptr = torch.tensor(np.cumsum([0] + [len(g) for g in self._groups]), dtype=torch.int64)

    @property
    def groups(self) -> list[list[int]]:
        if self._groups is None:
            flat = self.flat.cpu().numpy()
            gp = self.gptr.cpu().numpy()
            self._groups = [flat[gp[i]:gp[i + 1]].tolist() for i in range(len(gp) - 1)]
        return self._groups

    def __len__(self) -> int:
        return int(self.gptr.numel()) - 1

    @property
    def induced_perm(self) -> np.ndarray:
        """perm[old_id] = new_id (layout.py:32-41)."""
        return self.induced_perm_device().cpu().numpy()

    def induced_perm_device(self) -> torch.Tensor:
        flat = self.flat
        perm = torch.empty(self.num_vertices, dtype=torch.int64, device=flat.device)
        perm[flat] = torch.arange(flat.numel(), dtype=torch.int64, device=flat.device)
        return perm

    def validate(self, group_size: int = WINDOW_HEIGHT) -> None:
        """layout.py:43-61 (same messages), vectorised."""
        n = self.num_vertices
        sizes = (self.gptr[1:] - self.gptr[:-1]).cpu().numpy()
        flat = self.flat.cpu().numpy()
        for gi, sz in enumerate(sizes):
            if not 0 < sz <= group_size:
                raise ValueError(f"group size must be in 1..{group_size}")
            if sz < group_size and gi != len(sizes) - 1:
                raise ValueError(f"group {gi} is short but not last")
        if flat.size and (flat.min() < 0 or flat.max() >= n):
            bad = flat[(flat < 0) | (flat >= n)][0]
            raise ValueError(f"vertex id {bad} out of range")
        counts = np.bincount(flat, minlength=n) if flat.size else np.zeros(n, dtype=np.int64)
        if (counts > 1).any():
            raise ValueError(f"vertex {int(np.flatnonzero(counts > 1)[0])} appears twice")
        if flat.size != n:
            raise ValueError("groups must cover every vertex exactly once")


def _require_undirected(g, what: str) -> None:
    if not (isinstance(g, Graph) and g.undirected):
        raise ValueError(f"{what} requires an undirected graph")


def _adj(g) -> DeviceCsr:
    return to_device_csr(g.adjacency if isinstance(g, Graph) else g)


def sort_by_min_neighbor_device(adj: DeviceCsr) -> torch.Tensor:
    n = adj.num_rows
    deg = adj.row_ptr[1:] - adj.row_ptr[:-1]
    key = torch.full((n,), n, dtype=torch.int64, device=adj.device)
    nz = deg > 0
    key[nz] = adj.col_idx[adj.row_ptr[:-1][nz]].to(torch.int64)
    _, order = torch.sort(key, stable=True)  # ties keep id order == lexsort((arange, key))
    return order


def sort_by_min_neighbor(g) -> np.ndarray:
    """layout.py:99-109: ids by ascending lowest neighbour id, ties by id; isolated last."""
    return sort_by_min_neighbor_device(_adj(g)).cpu().numpy()


@_lib.nvtx("hcs.loa")
def build_windows_optimized(g, vw: int = 128, group_size: int = WINDOW_HEIGHT, check_counters: bool = False,
                            audit=None) -> WindowGrouping:
    """layout.py:186-263 on the GPU (K8).  Byte-identical grouping to the reference."""
    _require_undirected(g, "window grouping")
    if vw < 1:
        raise ValueError("vw must be >= 1")
    if audit is not None:
        raise ValueError("audit callbacks are not supported by the GPU builder (counters are exact by construction)")
    adj = _adj(g)
    n = adj.num_rows
    dev = adj.device
    order = sort_by_min_neighbor_device(adj).to(torch.int32)
    out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    gptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    ng = torch.zeros(1, dtype=torch.int64, device=dev)
    wsb = _lib.ctypes.c_size_t(0)
    _lib.check(_lib.lib().hcs_loa_workspace_bytes(n, _lib.ctypes.byref(wsb)))
    ws = torch.empty(max(int(wsb.value), 16), dtype=torch.uint8, device=dev)
    _lib.call("hcs_loa", adj.row_ptr.data_ptr(), adj.col_idx.data_ptr() if adj.nnz else None, n, vw, group_size,
              order.data_ptr(), out.data_ptr(), gptr.data_ptr(), ng.data_ptr(), ws.data_ptr(), ws.numel(),
              _lib.stream())
    k = int(ng.item())
    return WindowGrouping((out[:n].to(torch.int64), gptr[:k + 1].clone()), n)


def build_windows_basic(g, vw: int = 128, group_size: int = WINDOW_HEIGHT) -> WindowGrouping:
    """layout.py:142-183: the reference guarantees the same grouping as the optimized builder."""
    return build_windows_optimized(g, vw=vw, group_size=group_size)


def permute_symmetric(csr, perm) -> DeviceCsr:
    """matrices.py:310-318 (K9): entry (i, j) -> (perm[i], perm[j]); rows re-sorted.
    Integer relabel + value moves only, so bit-exact."""
    a = to_device_csr(csr)
    n = a.num_rows
    if a.num_rows != a.num_cols:
        raise ValueError("symmetric permutation requires a square matrix")
    p = perm if isinstance(perm, torch.Tensor) else torch.from_numpy(np.asarray(perm, dtype=np.int64))
    p = p.to(device=a.device, dtype=torch.int64)
    if p.shape != (n,) or not torch.equal(torch.sort(p).values, torch.arange(n, device=a.device)):
        raise ValueError("perm must be a bijection on 0..n-1")
    deg = a.row_ptr[1:] - a.row_ptr[:-1]
    rows = torch.repeat_interleave(torch.arange(n, device=a.device), deg)
    nr = p[rows]
    nc = p[a.col_idx.to(torch.int64)]
    key = nr * max(n, 1) + nc
    del rows
    _, order = torch.sort(key, stable=True)
    del key
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=a.device)
    torch.cumsum(torch.bincount(nr, minlength=n), 0, out=row_ptr[1:])
    out = DeviceCsr(n, n, row_ptr, nc[order].to(torch.int32), a.values[order])
    if a.values_f64 is not None:
        out.values_f64 = a.values_f64[order]
    elif a.host_values_f64 is not None:
        out.values_f64 = torch.from_numpy(a.host_values_f64).to(a.device)[order]
    out.symmetric = a.symmetric
    return out


def reorder(g, grouping: WindowGrouping):
    """layout.py:266-274: relabel so each group occupies one contiguous 16-row window."""
    _require_undirected(g, "reorder")
    grouping.validate()
    if grouping.num_vertices != g.num_vertices:
        raise ValueError("grouping does not match graph size")
    perm = grouping.induced_perm_device()
    adj = permute_symmetric(_adj(g), perm)
    return Graph(g.num_vertices, adj, g.undirected), perm.cpu().numpy()
