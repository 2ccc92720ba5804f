"""Fused GCN aggregation + update (K6 forward, K7 backward) and grad_W.

Reference: gnn.py:147-159 (fused forward: per window z_w = A_w X, out[rows] = z_w W,
z_cache[rows] = z_w) and gnn.py:195-205 (fused backward).  Here one launch per path
(tile windows: hcs_gcn_tile, scalar windows: hcs_gcn_scalar) aggregates each row
window and multiplies the on-chip 16 x d_in tile by M before writing the output rows:
    forward   out = (A X) W,      z = A X   (z_cache, needed for grad_W)
    backward  grad_X = (A^T G) W^T          (the reference's A^T (G W^T))
grad_W = Z^T G is a plain dense GEMM (d_in x n times n x d_out, K = n) and is left to
cuBLAS via torch.matmul on TF32 tensor cores (fp32 accumulate; deterministic for a fixed
shape).  Measured at C3 (n = 232,965): the fp32 SIMT GEMM took 303-330 us per call.

Sizes outside the fused kernels' on-chip budget (d_in or d_out > 128) run the same
math as two GPU passes (SpMM kernel, then a cuBLAS GEMM).
"""

from __future__ import annotations

import torch

from . import _lib
from .executors import _alloc_z, get_plan, stage_operand

FUSED_MAX_DIM = 128


GRAD_W_SPLIT = 2048  # rows per K-slice of the split-K grad_W GEMM


def grad_weight(z: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """Z^T G as a deterministic split-K GEMM: K = n rows in slices of GRAD_W_SPLIT, one batched
    TF32 tensor-core GEMM over the slices (a CTA per slice instead of one per 64 x 64 output
    tile: the plain GEMM took 125 us at C3), then the slice partials summed in slice order."""
    z, g = z.float(), g.float()
    n = int(z.shape[0])
    s = n // GRAD_W_SPLIT
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        if s < 2:
            return z.t() @ g
        head = s * GRAD_W_SPLIT
        zb = z[:head].reshape(s, GRAD_W_SPLIT, z.shape[1])
        gb = g[:head].reshape(s, GRAD_W_SPLIT, g.shape[1])
        out = torch.bmm(zb.transpose(1, 2), gb).sum(0)
        if head < n:
            out = out + z[head:].t() @ g[head:]
        return out
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def fused_aggregate_update(windows, assignment, x, m: torch.Tensor, precision: str, want_z: bool):
    """Returns (out [n, d_out] fp32, z [n, dim] fp32 or None) on the device."""
    ws = windows
    dev = ws.csr.device
    plan = get_plan(ws, assignment, precision)
    xop, _ = stage_operand(x, precision, dev, tf32_round=(precision == "tf32" and plan.n_tile > 0))
    m = m.to(device=dev, dtype=torch.float32).contiguous()
    dim, d_out = xop.dim, int(m.shape[1])
    if int(m.shape[0]) != dim:
        raise ValueError(f"X has {dim} features, weight expects {int(m.shape[0])}")
    n = ws.num_rows
    if dim > FUSED_MAX_DIM or d_out > FUSED_MAX_DIM or (plan.n_tile and precision != "bf16"):
        # outside the fused kernels' on-chip budget, or tf32 tile windows (the fused tile
        # epilogue is bf16-only): SpMM kernels, then a cuBLAS GEMM on the device
        z, ldz = _alloc_z(n, dim, dev)
        plan.run(xop, z, ldz)
        zz = z[:, :dim]
        return zz @ m, (zz if want_z else None)
    z, ldz = _alloc_z(n, dim, dev) if want_z else (None, 0)
    out = torch.empty((n, d_out), dtype=torch.float32, device=dev)
    csr = ws.csr
    s = _lib.stream()
    zp = z.data_ptr() if z is not None else None
    if plan.n_tile:
        _lib.call("hcs_gcn_tile", plan.tile_list.data_ptr(), plan.n_tile, plan.chunk_ptr.data_ptr(),
                  plan.gidx.data_ptr(), plan.ent_ptr.data_ptr(), plan.ent.data_ptr(), plan.ent_dtype, csr.num_rows,
                  ws.window_height, xop.t.data_ptr(), xop.dtype_code, xop.rows, dim, xop.ld, zp, ldz, m.data_ptr(),
                  d_out, out.data_ptr(), d_out, plan.scratch(s).data_ptr(), plan.scratch(s).numel() * 4, s)
    if plan.scalar_list.numel():
        _lib.call("hcs_gcn_scalar", csr.row_ptr.data_ptr(), csr.col_idx.data_ptr(), plan.scalar_vals.data_ptr(),
                  plan.scalar_vals_code, csr.num_rows, ws.window_height, plan.scalar_list.data_ptr(),
                  plan.scalar_list.numel(), xop.t.data_ptr(), xop.dtype_code, xop.rows, dim, xop.ld, zp, ldz,
                  m.data_ptr(), d_out, out.data_ptr(), d_out, s)
    return out, (z[:, :dim] if z is not None else None)


def gcn_forward_fused(windows, assignment, x, w, precision):
    out, z = fused_aggregate_update(windows, assignment, x, w, precision, want_z=True)
    return out, z


def gcn_backward_fused(windows, assignment, g, w, precision):
    gx, _ = fused_aggregate_update(windows, assignment, g, w.t(), precision, want_z=False)
    return gx
