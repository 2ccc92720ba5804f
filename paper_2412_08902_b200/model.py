"""2-layer GCN training on the fused kernels (BASELINE config C3).

The reference has a single GCN layer with no activation, loss or optimizer
(gnn.py:121-205).  The epoch defined here is
    fwd L1 (fused: out1 = (A X) W1, z1 = A X)      K6
    ReLU
    fwd L2 (fused: out2 = (A H) W2, z2 = A H)      K6
    softmax cross-entropy on seeded random labels
    bwd L2: grad_W2 = z2^T G2 (cuBLAS); grad_H = (A^T G2) W2^T (fused K7)
    ReLU backward
    bwd L1: grad_W1 = z1^T G1 (no grad_X for the input features)
    SGD update
The layer is a torch.autograd.Function whose forward/backward call the fused
kernels, so the loop body is plain PyTorch.  Multi-GPU (row-window shards):
each rank computes its rows; the layer output rows are all-gathered between
layers and grad_W is all-reduced.
"""

from __future__ import annotations

import numpy as np
import torch

from .executors import Assignment
from .fused import fused_aggregate_update, grad_weight
from .windows import WindowSet


class GcnAggregateUpdate(torch.autograd.Function):
    """y = (A x) W with A given by row windows; saves z = A x for grad_W."""

    @staticmethod
    def forward(ctx, x, w, windows, windows_t, assignment, precision, shard):
        out, z = fused_aggregate_update(windows, assignment, x.detach(), w.detach(), precision, want_z=True)
        ctx.save_for_backward(z, w)
        ctx.windows_t, ctx.assignment, ctx.precision, ctx.shard = windows_t, assignment, precision, shard
        return out

    @staticmethod
    def backward(ctx, g):
        # g: gradient of this rank's output rows (all rows on one GPU)
        z, w = ctx.saved_tensors
        g = g.contiguous()
        shard = ctx.shard
        gw = grad_weight(z, g)
        if shard is not None:
            shard.all_reduce(gw)  # grad_W = sum over ranks of z_r^T G_r
        gx = None
        if ctx.needs_input_grad[0]:
            # grad_X = (A^T G) W^T over the backward windows (A^T's; the forward windows when A is
            # symmetric); sharded: (A^T G)[rows_r] needs every rank's G rows
            g_full = g if shard is None else shard.all_gather_rows(g)
            gx, _ = fused_aggregate_update(ctx.windows_t, ctx.assignment, g_full, w.t(), ctx.precision,
                                           want_z=False)
            if shard is not None:
                gx = shard.embed_rows(gx)  # the input was all-gathered: only our rows flow back
        return gx, gw, None, None, None, None, None


def backward_windows(windows: WindowSet, shard=None) -> WindowSet:
    """Row windows of A^T for grad_X = A^T (G W^T) (gnn.py:181-183).  A symmetric operator (gcn /
    gin / raw on an undirected graph) is its own transpose, so the forward windows are reused;
    otherwise A^T is built and partitioned once and cached on the forward windows.  A sharded
    rank holds only its rows of A, which do not determine its rows of A^T: pass windows_t."""
    if getattr(windows.csr, "symmetric", False) or getattr(windows.csr, "global_symmetric", False):
        return windows
    if shard is not None:
        raise ValueError("a sharded layer over a non-symmetric operator needs windows_t (this rank's "
                         "row windows of A^T)")
    cached = getattr(windows, "_transpose_windows", None)
    if cached is None:
        from .gnn import transpose_csr
        from .windows import partition

        cached = partition(transpose_csr(windows.csr), windows.window_height)
        windows._transpose_windows = cached
    return cached


def gcn_layer(x, w, windows, windows_t=None, assignment=None, precision="bf16", shard=None):
    if assignment is None:
        assignment = Assignment(windows.codes)
    if windows_t is None:
        windows_t = backward_windows(windows, shard)
    out = GcnAggregateUpdate.apply(x, w, windows, windows_t, assignment, precision, shard)
    if shard is not None:
        out = shard.all_gather_rows_autograd(out)
    return out


class Gcn2:
    """Two GCN layers (d_in -> hidden -> classes), Glorot-uniform init from a seed
    (gnn.py:40-46 GnnLayer.random), full-batch SGD."""

    def __init__(self, d_in: int, hidden: int, classes: int, seed: int = 0, device="cuda", lr: float = 0.1):
        rng = np.random.default_rng(seed)

        def glorot(a, b):
            bound = np.sqrt(6.0 / (a + b))
            return torch.tensor(rng.uniform(-bound, bound, size=(a, b)), dtype=torch.float32, device=device,
                                requires_grad=True)

        self.w1 = glorot(d_in, hidden)
        self.w2 = glorot(hidden, classes)
        self.lr = lr

    def parameters(self):
        return [self.w1, self.w2]

    def forward(self, x, windows: WindowSet, windows_t=None, precision="bf16", shard=None):
        asg = Assignment(windows.codes)
        h = torch.relu(gcn_layer(x, self.w1, windows, windows_t, asg, precision, shard))
        return gcn_layer(h, self.w2, windows, windows_t, asg, precision, shard)

    def epoch(self, x, labels, windows: WindowSet, windows_t=None, precision="bf16", shard=None):
        """One training epoch; returns the loss tensor (on the device)."""
        logits = self.forward(x, windows, windows_t, precision, shard)
        # mean softmax cross-entropy as -mean(log_softmax[label]): warp-per-row softmax kernels
        # (F.cross_entropy's nll_loss reduction took 250 + 143 us at C3, logsumexp 110 us)
        loss = -torch.log_softmax(logits, dim=1).gather(1, labels.view(-1, 1).long()).mean()
        for p in self.parameters():
            p.grad = None
        loss.backward()
        with torch.no_grad():
            for p in self.parameters():
                p -= self.lr * p.grad
        return loss
