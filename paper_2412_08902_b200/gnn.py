"""Graph-convolution layer over the hybrid SpMM engine (reference gnn.py).

forward:  x_next = (A_norm X) W, z_cache = A_norm X                   (gnn.py:121-159)
backward: grad_W = Z^T G;  grad_X = A_norm^T (G W^T)                   (gnn.py:162-205)

Modes keep the reference's meaning and TrafficReport accounting:
  unfused: SpMM writes Z, a separate GEMM reads it (2 passes)
  fused:   one pass per row window -- the aggregated window tile stays on chip
           and is multiplied by W before the output rows are written (K6/K7).
The backward aggregation uses grad_X = (A^T G) W^T, which equals the
reference's A^T (G W^T) (gnn.py:202 recomputes G[cols] W^T per window; see
SURVEY.md §7) -- tolerance parity.

All math runs on the GPU; the reference's float64 host math is not available
(no CPU path).  Precision follows the executors ("bf16" default, or "tf32").
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .executors import Assignment, Path, spmm_hybrid, stage_operand, _resolve_precision
from .matrices import DenseMatrix, DeviceCsr, Graph, to_device_csr
from .windows import WindowSet, partition

NORMALIZATIONS = ("gcn", "row", "raw", "gin")


@dataclass(frozen=True)
class GnnLayer:
    """gnn.py:30-46."""

    weight: DenseMatrix

    @property
    def d_in(self) -> int:
        return self.weight.rows

    @property
    def d_out(self) -> int:
        return self.weight.dim

    @classmethod
    def random(cls, d_in: int, d_out: int, seed: int) -> "GnnLayer":
        rng = np.random.default_rng(seed)
        bound = np.sqrt(6.0 / (d_in + d_out))
        return cls(DenseMatrix(rng.uniform(-bound, bound, size=(d_in, d_out))))


@dataclass
class TrafficReport:
    """gnn.py:49-62 (element counts, not bytes)."""

    intermediate_writes: int = 0
    intermediate_reads: int = 0
    cache_writes: int = 0
    pass_launches: int = 0

    def as_dict(self) -> dict:
        return {"intermediate_writes": self.intermediate_writes, "intermediate_reads": self.intermediate_reads,
                "cache_writes": self.cache_writes, "pass_launches": self.pass_launches}


# --------------------------------------------------------------------------- normalisation
def _adjacency(g):
    return g.adjacency if isinstance(g, Graph) else g


@_lib.nvtx("hcs.normalize_adj")
def normalize_adj(g, kind: str = "gcn") -> DeviceCsr:
    """gnn.py:68-95 on the device.  Structure: A (+ I merged by a sorted key union);
    values: float64 kernels with the reference's operation order (csrc/normalize.cu),
    so the operator is bit-identical; kernels consume the float32 copy."""
    if kind not in NORMALIZATIONS:
        raise ValueError(f"kind must be one of {NORMALIZATIONS}, got {kind!r}")
    undirected = isinstance(g, Graph) and g.undirected
    adj = to_device_csr(_adjacency(g))
    dev = adj.device
    n = adj.num_rows
    v64 = (torch.from_numpy(adj.host_values_f64).to(dev) if adj.host_values_f64 is not None
           else adj.values.double())
    if kind == "raw":
        out = DeviceCsr(n, adj.num_cols, adj.row_ptr, adj.col_idx, adj.values, host_values_f64=adj.host_values_f64)
        out.symmetric = bool(undirected)
        return out
    if kind == "row":
        o64 = torch.empty_like(v64)
        o32 = torch.empty(v64.numel(), dtype=torch.float32, device=dev)
        _lib.call("hcs_normalize_values", 1, adj.row_ptr.data_ptr(), adj.col_idx.data_ptr(), v64.data_ptr(), n,
                  None, o64.data_ptr(), o32.data_ptr(), _lib.stream())
        out = DeviceCsr(n, adj.num_cols, adj.row_ptr, adj.col_idx, o32)
        out.values_f64 = o64
        out.symmetric = False
        return out
    if adj.num_rows != adj.num_cols:
        raise ValueError("self loops need a square adjacency")
    # A + I: merge the diagonal into the sorted (row, col) key set, summing duplicates
    rows = torch.repeat_interleave(torch.arange(n, device=dev), adj.row_ptr[1:] - adj.row_ptr[:-1])
    keys = torch.cat([rows * n + adj.col_idx.long(), torch.arange(n, device=dev) * (n + 1)])
    vals = torch.cat([v64, torch.ones(n, dtype=torch.float64, device=dev)])
    skeys, order = torch.sort(keys, stable=True)
    uk, inv = torch.unique_consecutive(skeys, return_inverse=True)
    summed = torch.zeros(uk.numel(), dtype=torch.float64, device=dev)
    summed.index_add_(0, inv, vals[order])  # at most two terms per key (A_ii + 1): order-free
    del keys, vals, skeys, order, inv
    r = torch.div(uk, n, rounding_mode="floor")
    c = (uk - r * n).to(torch.int32)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(torch.bincount(r, minlength=n), 0, out=row_ptr[1:])
    del r, uk
    if kind == "gin":
        out = DeviceCsr(n, n, row_ptr, c, summed.to(torch.float32))
        out.values_f64 = summed
        out.symmetric = bool(undirected) or getattr(adj, "symmetric", False)
        return out
    deg = torch.empty(n, dtype=torch.float64, device=dev)
    o64 = torch.empty_like(summed)
    o32 = torch.empty(summed.numel(), dtype=torch.float32, device=dev)
    _lib.call("hcs_normalize_values", 0, row_ptr.data_ptr(), c.data_ptr(), summed.data_ptr(), n, deg.data_ptr(),
              o64.data_ptr(), o32.data_ptr(), _lib.stream())
    out = DeviceCsr(n, n, row_ptr, c, o32)
    out.values_f64 = o64
    out.symmetric = bool(undirected) or getattr(adj, "symmetric", False)
    return out


def transpose_csr(a: DeviceCsr) -> DeviceCsr:
    """A^T on the device (gnn.py:181-182)."""
    if getattr(a, "symmetric", False):
        return a
    if "transpose" in a._derived:
        return a._derived["transpose"]
    dev = a.device
    n_r, n_c = a.num_rows, a.num_cols
    rows = torch.repeat_interleave(torch.arange(n_r, device=dev), a.row_ptr[1:] - a.row_ptr[:-1])
    keys = a.col_idx.long() * n_r + rows
    sk, order = torch.sort(keys, stable=True)
    r = torch.div(sk, n_r, rounding_mode="floor")
    c = (sk - r * n_r).to(torch.int32)
    row_ptr = torch.zeros(n_c + 1, dtype=torch.int64, device=dev)
    torch.cumsum(torch.bincount(r, minlength=n_c), 0, out=row_ptr[1:])
    out = DeviceCsr(n_c, n_r, row_ptr, c, a.values[order])
    if getattr(a, "values_f64", None) is not None:
        out.values_f64 = a.values_f64[order]
    a._derived["transpose"] = out
    return out


# --------------------------------------------------------------------------- layer
def _resolve_windows(a_norm, windows, assignment):
    """gnn.py:98-107: default assignment is all SCALAR (the reference does not classify)."""
    if windows is None:
        windows = partition(a_norm)
    elif not isinstance(windows, WindowSet):
        from .windows import as_windowset

        windows = as_windowset(windows)
    if assignment is None:
        assignment = Assignment.uniform(len(windows), Path.SCALAR)
    return windows, assignment


def _weight(layer: GnnLayer, dev) -> torch.Tensor:
    w = layer.weight.data
    t = w if isinstance(w, torch.Tensor) else torch.from_numpy(np.asarray(w))
    return t.to(device=dev, dtype=torch.float32)


def _out(t: torch.Tensor, host: bool) -> DenseMatrix:
    return DenseMatrix(t.cpu().numpy() if host else t)


def forward(layer: GnnLayer, a_norm, x, mode: str = "unfused", assignment: Assignment | None = None,
            windows=None, threads: int = 1, precision: str = "bf16"):
    """gnn.py:121-159: returns (x_next, z_cache, traffic)."""
    xdim = x.dim if isinstance(x, DenseMatrix) else int(x.shape[1])
    if xdim != layer.d_in:
        raise ValueError(f"X has {xdim} features, layer expects {layer.d_in}")
    if mode not in ("fused", "unfused"):
        raise ValueError(f"mode must be 'fused' or 'unfused', got {mode!r}")
    precision = _resolve_precision(precision)
    a = to_device_csr(a_norm) if not isinstance(a_norm, WindowSet) else a_norm.csr
    windows, assignment = _resolve_windows(a, windows, assignment)
    n = windows.total_rows()
    dev = windows.csr.device
    w = _weight(layer, dev)
    host = not isinstance(x.data if isinstance(x, DenseMatrix) else x, torch.Tensor)
    traffic = TrafficReport()
    if mode == "unfused":
        from .fused import dense_matmul

        z = spmm_hybrid(windows, assignment, x, precision=precision).z.data
        z = torch.as_tensor(z, device=dev)
        x_next = dense_matmul(z, w)
        traffic.intermediate_writes = n * layer.d_in
        traffic.intermediate_reads = n * layer.d_in
        traffic.pass_launches = 2
        return _out(x_next, host), _out(z, host), traffic
    from .fused import gcn_forward_fused

    x_next, z = gcn_forward_fused(windows, assignment, x, w, precision)
    traffic.cache_writes = n * layer.d_in
    traffic.pass_launches = 1
    return _out(x_next, host), _out(z, host), traffic


def backward(layer: GnnLayer, a_norm, z_cache, grad_out, mode: str = "unfused",
             assignment: Assignment | None = None, threads: int = 1, precision: str = "bf16"):
    """gnn.py:162-205: returns (grad_w, grad_x, traffic)."""
    if mode not in ("fused", "unfused"):
        raise ValueError(f"mode must be 'fused' or 'unfused', got {mode!r}")
    a = a_norm.csr if isinstance(a_norm, WindowSet) else a_norm
    if a.num_rows != a.num_cols:
        raise ValueError("backward requires a square aggregation operator")
    precision = _resolve_precision(precision)
    a = to_device_csr(a)
    at = transpose_csr(a)
    windows, assignment = _resolve_windows(at, None, assignment)
    dev = windows.csr.device
    w = _weight(layer, dev)
    gdata = grad_out.data if isinstance(grad_out, DenseMatrix) else grad_out
    host = not isinstance(gdata, torch.Tensor)
    g = torch.as_tensor(np.ascontiguousarray(gdata) if host else gdata).to(device=dev, dtype=torch.float32)
    zd = z_cache.data if isinstance(z_cache, DenseMatrix) else z_cache
    z = torch.as_tensor(np.ascontiguousarray(zd) if not isinstance(zd, torch.Tensor) else zd).to(
        device=dev, dtype=torch.float32)
    traffic = TrafficReport()
    from .fused import grad_weight

    grad_w = grad_weight(z, g)
    if mode == "unfused":
        from .fused import dense_matmul

        grad_z = dense_matmul(g, w.t())
        traffic.intermediate_writes = a.num_rows * layer.d_in
        traffic.intermediate_reads = a.num_rows * layer.d_in
        traffic.pass_launches = 2
        gx = spmm_hybrid(windows, assignment, grad_z, precision=precision).z.data
        return _out(grad_w, host), _out(gx, host), traffic
    from .fused import gcn_backward_fused

    gx = gcn_backward_fused(windows, assignment, g, w, precision)
    traffic.pass_launches = 1
    return _out(grad_w, host), _out(gx, host), traffic


def layer_bench(g, layer: GnnLayer, assignment_for=None, repeats: int = 3, seed: int = 0, kind: str = "gcn",
                precision: str = "bf16") -> dict:
    """gnn.py:208-244 with CUDA-event timing."""
    a_norm = normalize_adj(g, kind)
    x = torch.from_numpy(DenseMatrix.random(a_norm.num_rows, layer.d_in, seed=seed).data).float().cuda()
    windows = partition(a_norm)
    assignment = assignment_for(windows) if assignment_for is not None else None
    report: dict = {"num_vertices": a_norm.num_rows, "nnz": a_norm.nnz, "repeats": repeats}
    outputs = {}
    for mode in ("unfused", "fused"):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record()
        for _ in range(repeats):
            x_next, z, fwd_t = forward(layer, a_norm, x, mode=mode, assignment=assignment, windows=windows,
                                       precision=precision)
            gw, gx, bwd_t = backward(layer, a_norm, z, x_next, mode=mode, assignment=assignment,
                                     precision=precision)
        end.record()
        torch.cuda.synchronize()
        outputs[mode] = (x_next.data, gw.data, gx.data)
        report[mode] = {"seconds_per_iter": start.elapsed_time(end) / 1e3 / repeats,
                        "forward_traffic": fwd_t.as_dict(), "backward_traffic": bwd_t.as_dict()}
    diffs = []
    for a, b in zip(outputs["unfused"], outputs["fused"]):
        denom = max(float(a.abs().max()), 1e-300)
        diffs.append(float((a - b).abs().max()) / denom)
    report["max_rel_diff"] = max(diffs)
    return report
