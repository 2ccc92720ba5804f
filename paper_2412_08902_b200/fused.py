"""Fused GCN aggregation + update (K6 forward, K7 backward), grad_W and the dense update.

Reference: gnn.py:147-159 (fused forward: per window z_w = A_w X, out[rows] = z_w W,
z_cache[rows] = z_w) and gnn.py:195-205 (fused backward).  Here one launch per path
(tile windows: hcs_gcn_tile, scalar windows: hcs_gcn_scalar) aggregates each row
window and multiplies the on-chip 16 x d_in tile by M before writing the output rows:
    forward   out = (A X) W,      z = A X   (z_cache, needed for grad_W)
    backward  grad_X = (A^T G) W^T          (the reference's A^T (G W^T))
Fused shapes: d_out <= 64; bf16 d_in <= 128; tf32 any d_in on tile windows (M rounded to tf32),
d_in <= 128 on scalar windows.  Other shapes run the same math unfused: the SpMM kernels, then
the hand-written tall-skinny GEMM (csrc/dense.cu hcs_gemm).
grad_W = Z^T G (gnn.py:188, 195-199) is csrc/dense.cu hcs_grad_w: a deterministic split-K
tf32 tensor-core GEMM (fixed row slices summed in slice order).  No GCN pass calls cuBLAS.
"""

from __future__ import annotations

import torch

from . import _lib
from .executors import _alloc_z, get_plan, stage_operand

FUSED_MAX_DIM = 128      # scalar-window fused epilogue (d_in and d_out), bf16 tile epilogue (d_in)
FUSED_TILE_MAX_OUT = 64  # tile-window fused epilogues (out accumulators in registers)


def _f32_2d(t: torch.Tensor, dev) -> torch.Tensor:
    t = t.to(device=dev, dtype=torch.float32)
    if t.dim() != 2:
        raise ValueError("dense operands must be 2-dimensional")
    if t.stride(1) != 1 or t.stride(0) < t.shape[1]:
        t = t.contiguous()
    return t


@_lib.nvtx("hcs.grad_w")
def grad_weight(z: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """Z^T G (grad_W, gnn.py:188) on the hand-written deterministic split-K kernel."""
    dev = z.device
    z, g = _f32_2d(z, dev), _f32_2d(g, dev)
    K, M, N = int(z.shape[0]), int(z.shape[1]), int(g.shape[1])
    if int(g.shape[0]) != K:
        raise ValueError(f"z has {K} rows, grad has {int(g.shape[0])}")
    out = torch.empty((M, N), dtype=torch.float32, device=dev)
    if M == 0 or N == 0:
        return out
    wsb = _lib.ctypes.c_size_t(0)
    _lib.check(_lib.lib().hcs_grad_w_workspace_bytes(K, M, N, _lib.ctypes.byref(wsb)))
    ws = torch.empty(max(int(wsb.value) // 4, 1), dtype=torch.float32, device=dev)
    _lib.call("hcs_grad_w", z.data_ptr(), z.stride(0), g.data_ptr(), g.stride(0), K, M, N, out.data_ptr(), N,
              ws.data_ptr(), ws.numel() * 4, _lib.stream())
    return out


@_lib.nvtx("hcs.gemm")
def dense_matmul(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """a [K x M] @ b [M x N] on the hand-written tall-skinny tf32 GEMM (csrc/dense.cu).
    `out`: optional fp32 [K x N] destination with unit column stride (e.g. a row slice)."""
    dev = a.device
    a, b = _f32_2d(a, dev), _f32_2d(b, dev)
    K, M, N = int(a.shape[0]), int(a.shape[1]), int(b.shape[1])
    if int(b.shape[0]) != M:
        raise ValueError(f"inner dimensions differ: {M} vs {int(b.shape[0])}")
    if out is None:
        out = torch.empty((K, N), dtype=torch.float32, device=dev)
    elif out.dtype != torch.float32 or tuple(out.shape) != (K, N) or out.stride(1) != 1:
        raise ValueError(f"out must be float32 ({K}, {N}) with unit column stride")
    if K and N and M:
        _lib.call("hcs_gemm", a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), K, M, N, out.data_ptr(),
                  out.stride(0), _lib.stream())
    elif K and N:
        out.zero_()
    return out


def slice_padded(dim: int) -> int:
    """Row length of a bf16 operand padded to whole gather slices (executors.stage_operand)."""
    from .executors import PAD_TO_SLICE, _round_up

    s = 32 if dim <= 32 else 64
    return _round_up(dim, s) if PAD_TO_SLICE else _round_up(dim, 8)


def dense_matmul_bf16(a: torch.Tensor, b: torch.Tensor, mask: torch.Tensor | None = None):
    """The next aggregation's operand straight from the GEMM (hcs_gemm_bf16): a DeviceOperand of
    bf16(a @ b * 1[mask > 0]) with rows padded to whole gather slices."""
    from .executors import DeviceOperand

    dev = a.device
    a, b = _f32_2d(a, dev), _f32_2d(b, dev)
    K, M, N = int(a.shape[0]), int(a.shape[1]), int(b.shape[1])
    if int(b.shape[0]) != M:
        raise ValueError(f"inner dimensions differ: {M} vs {int(b.shape[0])}")
    ld = slice_padded(N)
    out = torch.empty((K, ld), dtype=torch.bfloat16, device=dev)
    mp, ldm = 0, 0
    if mask is not None:
        if tuple(mask.shape) != (K, N) or mask.dtype != torch.float32 or mask.stride(1) != 1:
            raise ValueError(f"mask must be float32 ({K}, {N}) with unit column stride")
        mp, ldm = mask.data_ptr(), mask.stride(0)
    if K:
        _lib.call("hcs_gemm_bf16", a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), K, M, N, out.data_ptr(), ld,
                  ld, mp, ldm, _lib.stream())
    return DeviceOperand(out, N, ld, _lib.DTYPE_BF16)


_XENT_WS: dict = {}


def softmax_xent(logits: torch.Tensor, labels: torch.Tensor, grad_scale: float | None = None):
    """(loss, grad operand): loss = -mean log_softmax(logits)[labels] (device scalar), grad =
    grad_scale * (softmax - onehot) (default scale 1/rows: d loss / d logits) as a bf16
    DeviceOperand padded to whole gather slices, ready for the backward aggregation (hcs_softmax_xent)."""
    from .executors import DeviceOperand

    dev = logits.device
    if logits.dtype != torch.float32 or logits.dim() != 2 or logits.stride(1) != 1:
        raise ValueError("logits must be a float32 matrix with unit column stride")
    rows, classes = int(logits.shape[0]), int(logits.shape[1])
    labels = labels.to(device=dev, dtype=torch.int64).contiguous()
    if labels.numel() != rows:
        raise ValueError(f"{labels.numel()} labels for {rows} rows")
    ld = slice_padded(classes)
    grad = torch.empty((rows, ld), dtype=torch.bfloat16, device=dev)
    loss = torch.empty((), dtype=torch.float32, device=dev)
    wsb = _lib.ctypes.c_size_t(0)
    _lib.check(_lib.lib().hcs_softmax_xent_workspace_bytes(rows, _lib.ctypes.byref(wsb)))
    key = (dev, _lib.stream())  # one workspace (counter + partials) per stream
    ws = _XENT_WS.get(key)
    if ws is None or ws.numel() * 4 < wsb.value:
        ws = _XENT_WS[key] = torch.zeros(max(int(wsb.value) // 4, 64), dtype=torch.float32, device=dev)
    scale = (1.0 / rows) if grad_scale is None else float(grad_scale)
    _lib.call("hcs_softmax_xent", logits.data_ptr(), logits.stride(0), rows, classes, labels.data_ptr(), scale,
              loss.data_ptr(), grad.data_ptr(), _lib.DTYPE_BF16, ld, ld, ws.data_ptr(), ws.numel() * 4,
              _lib.stream())
    return loss, DeviceOperand(grad, classes, ld, _lib.DTYPE_BF16)


class FusedLayer:
    """One GCN aggregation + update over a WindowSet: out = (A X) M (and z = A X), staged once and
    launched for all windows or for row-window parts (plan.parts / window bounds), so a sharded
    layer can start exchanging part k's rows while part k+1 computes (model.ShardedGcnLayer)."""

    def __init__(self, windows, assignment, x, m: torch.Tensor, precision: str, want_z: bool):
        ws = windows
        dev = ws.csr.device
        self.ws, self.precision = ws, precision
        self.plan = plan = get_plan(ws, assignment, precision)
        self.xop, _ = stage_operand(x, precision, dev, tf32_round=(precision == "tf32" and plan.n_tile > 0))
        self.m = m = m.to(device=dev, dtype=torch.float32).contiguous()
        self.dim, self.d_out = dim, d_out = self.xop.dim, int(m.shape[1])
        if int(m.shape[0]) != dim:
            raise ValueError(f"X has {dim} features, weight expects {int(m.shape[0])}")
        n = ws.num_rows
        has_scalar = plan.scalar_list.numel() > 0
        self.fused = ((not plan.n_tile or (d_out <= FUSED_TILE_MAX_OUT and (precision == "tf32" or dim <= FUSED_MAX_DIM)))
                      and (not has_scalar or (dim <= FUSED_MAX_DIM and d_out <= FUSED_MAX_DIM)))
        # outside the fused kernels' on-chip budget: SpMM kernels, then the dense update kernel
        self.want_z = want_z
        self.z, self.ldz = _alloc_z(n, dim, dev) if (want_z or not self.fused) else (None, 0)
        self.out = torch.empty((n, d_out), dtype=torch.float32, device=dev)
        self.mt = m
        if self.fused and plan.n_tile and precision == "tf32":  # tile epilogue B operand: M rounded to tf32
            self.mt = torch.empty_like(m)
            _lib.call("hcs_convert", m.data_ptr(), self.mt.data_ptr(), m.numel(), _lib.DTYPE_F32, _lib.stream())

    def parts(self, bounds) -> list:
        """Window bounds (local window ids) -> parts for run()."""
        return self.plan.parts_from_bounds(bounds)

    def run(self, part=None) -> None:
        """Launch the kernels of windows part = (w0, w1, t0, t1, s0, s1) (all windows if None)."""
        plan, ws, xop = self.plan, self.ws, self.xop
        dim, d_out = self.dim, self.d_out
        n = ws.num_rows
        if not self.fused:
            plan.run(xop, self.z, self.ldz, part=part)
            r0, r1 = (0, n) if part is None else (min(part[0] * ws.window_height, n), min(part[1] * ws.window_height, n))
            if r1 > r0:
                dense_matmul(self.z[r0:r1, :dim], self.m, out=self.out[r0:r1])
            return
        t0, t1 = (0, plan.n_tile) if part is None else part[2:4]
        s0, s1 = (0, int(plan.scalar_list.numel())) if part is None else part[4:6]
        csr = ws.csr
        s = _lib.stream()
        zp = self.z.data_ptr() if self.z is not None else None
        if t1 > t0:
            scr = plan.scratch(s)
            _lib.call("hcs_gcn_tile", plan.tile_list.data_ptr() + 4 * t0, t1 - t0, plan.chunk_ptr.data_ptr() + 8 * t0,
                      plan.gidx.data_ptr(), plan.ent_ptr.data_ptr(), plan.ent.data_ptr(), plan.ent_dtype,
                      csr.num_rows, ws.window_height, xop.t.data_ptr(), xop.dtype_code, xop.rows, dim, xop.ld, zp,
                      self.ldz, self.mt.data_ptr(), d_out, self.out.data_ptr(), d_out, scr.data_ptr(),
                      scr.numel() * 4, s)
        if s1 > s0:
            _lib.call("hcs_gcn_scalar", csr.row_ptr.data_ptr(), csr.col_idx.data_ptr(), plan.scalar_vals.data_ptr(),
                      plan.scalar_vals_code, csr.num_rows, ws.window_height, plan.scalar_list.data_ptr() + 4 * s0,
                      s1 - s0, xop.t.data_ptr(), xop.dtype_code, xop.rows, dim, xop.ld, zp, self.ldz,
                      self.m.data_ptr(), d_out, self.out.data_ptr(), d_out, s)

    def result(self):
        return self.out, (self.z[:, :self.dim] if (self.z is not None and self.want_z) else None)


@_lib.nvtx("hcs.gcn_fused")
def fused_aggregate_update(windows, assignment, x, m: torch.Tensor, precision: str, want_z: bool):
    """Returns (out [n, d_out] fp32, z [n, dim] fp32 or None) on the device."""
    layer = FusedLayer(windows, assignment, x, m, precision, want_z)
    layer.run()
    return layer.result()


def gcn_forward_fused(windows, assignment, x, w, precision):
    out, z = fused_aggregate_update(windows, assignment, x, w, precision, want_z=True)
    return out, z


def gcn_backward_fused(windows, assignment, g, w, precision):
    gx, _ = fused_aggregate_update(windows, assignment, g, w.t(), precision, want_z=False)
    return gx
