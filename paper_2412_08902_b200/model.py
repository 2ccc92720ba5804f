"""2-layer GCN training on the fused kernels (BASELINE config C3).

The reference has a single GCN layer with no activation, loss or optimizer
(gnn.py:121-205).  The epoch defined here is, with
order="fused" (the reference's (A X) W order):
    fwd L1 (fused: out1 = (A X) W1, z1 = A X)      K6
    ReLU
    fwd L2 (fused: out2 = (A H) W2, z2 = A H)      K6
    softmax cross-entropy on seeded random labels
    bwd L2: grad_W2 = z2^T G2 (K7 split-K kernel); grad_H = (A^T G2) W2^T (fused K7)
    ReLU backward
    bwd L1: grad_W1 = z1^T G1 (no grad_X for the input features)
    SGD update
and with order="auto" (the default; update first where d_out < d_in, both C3 layers) each layer
is A (X W): a GEMM, then a plain SpMM over d_out-wide rows; backward S = A^T G (SpMM),
grad_W = X^T S, grad_X = S W^T.  C3 layer 1 then gathers 64-wide rows twice (forward and
backward) instead of 128-wide ones once: 5.69 -> 5.46 ms per epoch (tools/exp_order.py).
The layer is a torch.autograd.Function whose forward/backward call the fused
kernels, so the loop body is plain PyTorch.  Multi-GPU (row-window shards,
ShardedGcnLayer): each rank computes its rows in parts whose all-gathers overlap
the next part's kernels, and grad_W is all-reduced under the grad_X aggregation
(SURVEY §5, §8e).
"""

from __future__ import annotations

import numpy as np
import torch

from .fused import (FusedLayer, dense_matmul, dense_matmul_bf16, fused_aggregate_update, grad_weight,
                    softmax_xent)
from .windows import WindowSet


class GcnAggregateUpdate(torch.autograd.Function):
    """y = (A x) W with A given by row windows (one GPU); saves z = A x for grad_W."""

    @staticmethod
    def forward(ctx, x, w, windows, windows_t, assignment, precision, shard):
        out, z = fused_aggregate_update(windows, assignment, x.detach(), w.detach(), precision, want_z=True)
        ctx.save_for_backward(z, w)
        ctx.windows_t, ctx.assignment, ctx.precision = windows_t, assignment, precision
        return out

    @staticmethod
    def backward(ctx, g):
        z, w = ctx.saved_tensors
        g = g.contiguous()
        gw = grad_weight(z, g)
        gx = None
        if ctx.needs_input_grad[0]:
            # grad_X = (A^T G) W^T over the backward windows (A^T's; the forward windows when A is
            # symmetric)
            gx, _ = fused_aggregate_update(ctx.windows_t, ctx.assignment, g, w.t(), ctx.precision, want_z=False)
        return gx, gw, None, None, None, None, None


class UpdateAggregate(torch.autograd.Function):
    """y = A (x W): the update first, when it narrows the rows (d_out < d_in), so the aggregation
    gathers d_out-wide rows instead of d_in-wide ones -- the same product as (A x) W, in the other
    order (C3 layer 1: one 64-wide SpMM instead of a 128-wide fused one).  No z_cache is needed:
    grad_W = x^T (A^T G), and A^T G is also what grad_x = (A^T G) W^T aggregates."""

    @staticmethod
    def forward(ctx, x, w, windows, windows_t, assignment, precision):
        from .executors import spmm_hybrid

        t = dense_matmul(x.detach(), w.detach())
        out = spmm_hybrid(windows, assignment, t, precision=precision).z.data
        ctx.save_for_backward(x, w)
        ctx.windows_t, ctx.assignment, ctx.precision = windows_t, assignment, precision
        return out

    @staticmethod
    def backward(ctx, g):
        from .executors import spmm_hybrid

        x, w = ctx.saved_tensors
        gt = spmm_hybrid(ctx.windows_t, ctx.assignment, g.contiguous(), precision=ctx.precision).z.data
        gw = grad_weight(x, gt)
        gx = dense_matmul(gt, w.t()) if ctx.needs_input_grad[0] else None
        return gx, gw, None, None, None, None


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


def gcn_layer(x, w, windows, windows_t=None, assignment=None, precision="bf16", shard=None, order="fused"):
    """One GCN layer y = A x W.  order: "fused" (aggregate then update in one kernel, saving
    z = A x: the reference's forward), "update_first" (A (x W), UpdateAggregate), or "auto"
    (update first when it narrows the rows, d_out < d_in, on one GPU)."""
    if assignment is None:
        assignment = windows.assignment()
    if windows_t is None:
        windows_t = backward_windows(windows, shard)
    if shard is not None:
        return ShardedGcnLayer.apply(x, w, windows, windows_t, assignment, precision, shard, EXCHANGE_PARTS)
    if order == "update_first" or (order == "auto" and int(w.shape[1]) < int(w.shape[0])):
        return UpdateAggregate.apply(x, w, windows, windows_t, assignment, precision)
    return GcnAggregateUpdate.apply(x, w, windows, windows_t, assignment, precision, None)


class ShardedGcnLayer(torch.autograd.Function):
    """One row-window-sharded GCN layer: y_full = all_gather_r((A_r x) W).

    Forward: the rank's windows run in EXCHANGE_PARTS nnz-balanced parts; right after part k's
    kernels its output rows start an async all-gather (NCCL runs it on its own stream), so the
    exchange of part k overlaps the aggregation of part k+1 and only the last part's transfer is
    exposed.  Backward: the all-gather of G's rows (needed because A^T G reads every column) is
    issued first and grad_W = z_r^T G_r is computed while it flies; grad_W's all-reduce then
    overlaps the grad_X aggregation."""

    @staticmethod
    def forward(ctx, x, w, windows, windows_t, assignment, precision, shard, parts):
        layer = FusedLayer(windows, assignment, x.detach(), w.detach(), precision, want_z=True)
        spans = shard.part_spans(parts)
        mine = layer.parts([lo for lo, _ in spans[shard.rank]] + [spans[shard.rank][-1][1]])
        n_loc = shard.row1 - shard.row0
        wh = shard.wh

        def rows_of(r, k):
            r0, r1 = shard.rank_rows(r)
            lo, hi = spans[r][k]
            return min(lo * wh, r1 - r0), min(hi * wh, r1 - r0)

        pending = []
        for k, part in enumerate(mine):
            layer.run(part)
            a, b = rows_of(shard.rank, k)
            counts = [rows_of(r, k)[1] - rows_of(r, k)[0] for r in range(shard.world)]
            pending.append((k, counts) + shard.start_gather(layer.out[a:b], counts))
        full = torch.empty((shard.n_rows, layer.d_out), dtype=layer.out.dtype, device=layer.out.device)
        for k, counts, work, recv, maxr in pending:
            work.wait()
            for r in range(shard.world):
                a, b = rows_of(r, k)
                if b > a:
                    g0 = shard.rank_rows(r)[0]
                    full[g0 + a:g0 + b] = recv[r * maxr: r * maxr + (b - a)]
        out, z = layer.result()
        assert out.shape[0] == n_loc
        ctx.save_for_backward(z, w)
        ctx.windows_t, ctx.assignment, ctx.precision, ctx.shard = windows_t, assignment, precision, shard
        return full

    @staticmethod
    def backward(ctx, g_full):
        import torch.distributed as dist

        z, w = ctx.saved_tensors
        shard = ctx.shard
        g_loc = g_full[shard.row0:shard.row1].contiguous()
        counts = [shard.rank_rows(r)[1] - shard.rank_rows(r)[0] for r in range(shard.world)]
        gather = shard.start_gather(g_loc, counts) if ctx.needs_input_grad[0] else None
        gw = grad_weight(z, g_loc)  # overlaps the all-gather of G
        red = dist.all_reduce(gw, op=dist.ReduceOp.SUM, group=shard.group, async_op=True)
        gx = None
        if gather is not None:
            work, recv, maxr = gather
            work.wait()
            g_all = torch.cat([recv[r * maxr: r * maxr + counts[r]] for r in range(shard.world)], 0)
            gx_loc, _ = fused_aggregate_update(ctx.windows_t, ctx.assignment, g_all, w.t(), ctx.precision,
                                               want_z=False)  # overlaps grad_W's all-reduce
            gx = shard.embed_rows(gx_loc)  # the input was replicated / gathered: our rows flow back
        red.wait()
        return gx, gw, None, None, None, None, None, None


EXCHANGE_PARTS = 4  # row-window parts per sharded layer (exchange of part k under compute of k+1)


class Gcn2:
    """Two GCN layers (d_in -> hidden -> classes), Glorot-uniform init from a seed
    (gnn.py:40-46 GnnLayer.random), full-batch SGD."""

    def __init__(self, d_in: int, hidden: int, classes: int, seed: int = 0, device="cuda", lr: float = 0.1,
                 order=("auto", "auto")):
        """order: per-layer gcn_layer order ("fused" | "update_first" | "auto"; sharded layers are
        always fused)."""
        self.order = (order, order) if isinstance(order, str) else tuple(order)
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
        asg = windows.assignment()
        h = torch.relu(gcn_layer(x, self.w1, windows, windows_t, asg, precision, shard, self.order[0]))
        return gcn_layer(h, self.w2, windows, windows_t, asg, precision, shard, self.order[1])

    def update_first(self, layer: int, shard=None) -> bool:
        """Whether gcn_layer runs layer 0/1 as A (X W)."""
        o = self.order[layer]
        w = (self.w1, self.w2)[layer]
        return shard is None and (o == "update_first" or (o == "auto" and int(w.shape[1]) < int(w.shape[0])))

    def epoch(self, x, labels, windows: WindowSet, windows_t=None, precision="bf16", shard=None,
              explicit: bool | None = None):
        """One training epoch; returns the loss tensor (on the device).  explicit (default: whenever
        both layers are update-first on one GPU in bf16): the hand-written epoch below instead of
        autograd through gcn_layer -- same math, fewer and fused launches."""
        if explicit is None:
            explicit = precision == "bf16" and self.update_first(0, shard) and self.update_first(1, shard)
        if explicit:
            if not (precision == "bf16" and self.update_first(0, shard) and self.update_first(1, shard)):
                raise ValueError("the explicit epoch needs bf16 and both layers update-first on one GPU")
            return self._epoch_update_first(x, labels, windows, windows_t)
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

    def _epoch_update_first(self, x, labels, windows: WindowSet, windows_t=None):
        """The C3 epoch with both layers A (X W), written out:
            T1 = X W1 -> bf16 operand (GEMM epilogue)   H = relu(A T1)          (SpMM)
            T2 = H W2 -> bf16 operand                    logits = A T2           (SpMM)
            loss, G2 = softmax cross-entropy, G2 written as the bf16 operand    (one kernel)
            S2 = A^T G2 (SpMM)   grad_W2 = H^T S2 (split-K)
            G1 = (S2 W2^T) * 1[H > 0] -> bf16 operand (GEMM epilogue)
            S1 = A^T G1 (SpMM)   grad_W1 = X^T S1 (split-K)   SGD
        The operands of the four aggregations come straight out of the kernels that produce them
        (no staging copies), and torch's loss / ReLU-backward kernels are gone (C3: 45 -> 17
        launches per epoch).  Gradients equal the autograd path's to bf16 rounding of the operands
        (tests/test_gpu_gnn.py)."""
        from .executors import spmm_staged

        asg = windows.assignment()
        wt = backward_windows(windows) if windows_t is None else windows_t
        asg_t = asg if wt is windows else wt.assignment()
        w1, w2 = self.w1.detach(), self.w2.detach()
        h = spmm_staged(windows, asg, dense_matmul_bf16(x, w1))
        h.relu_()
        logits = spmm_staged(windows, asg, dense_matmul_bf16(h, w2))
        loss, g2 = softmax_xent(logits, labels)
        s2 = spmm_staged(wt, asg_t, g2)
        gw2 = grad_weight(h, s2)
        s1 = spmm_staged(wt, asg_t, dense_matmul_bf16(s2, w2.t(), mask=h))
        gw1 = grad_weight(x, s1)
        with torch.no_grad():
            self.w1.grad, self.w2.grad = gw1, gw2
            self.w1.sub_(gw1, alpha=self.lr)
            self.w2.sub_(gw2, alpha=self.lr)
        return loss
