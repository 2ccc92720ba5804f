"""Multi-process (world_size 2, gloo, CPU) tests of the row-window sharding host logic
(SURVEY §5, §8e): nnz-balanced contiguous window ranges, exactness of per-shard windows
(windows are row-local, reference windows.py:90-105), the ragged row all-gather between
layers, and the sharded 2-layer GCN autograd plumbing (all-gather forward / slice
backward, grad_W all-reduce, embedded grad_X) against one process.  The per-rank SpMM
kernels need a GPU; here the fused layer is replaced by its dense float64 definition."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rowwin_oracle as orc

from paper_2412_08902_b200 import model as gcn_model
from paper_2412_08902_b200.shard import Shard, shard_window_ranges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_ranges_cover_and_balance():
    a = orc.random_csr(1000, 1000, 0.03, seed=4)
    for world in (1, 2, 3, 4, 8):
        r = shard_window_ranges(a.row_ptr, a.num_rows, world)
        W = -(-a.num_rows // 16)
        assert r[0][0] == 0 and r[-1][1] == W
        assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
        starts = a.row_ptr[np.minimum(np.arange(W + 1) * 16, a.num_rows)]
        per = [int(starts[b] - starts[e0]) for e0, b in r]
        wmax = int(np.diff(starts).max())
        assert max(per) - min(per) <= 2 * wmax + 1


def test_shard_windows_equal_global_windows():
    """Partition + features + selector of a rank's row slice == the same windows globally."""
    a = orc.random_csr(700, 900, 0.05, seed=8)
    full = orc.partition(a)
    nc, dens, _ = orc.features(full)
    codes = orc.classify(nc, dens)
    for world in (2, 3):
        for w0, w1 in shard_window_ranges(a.row_ptr, a.num_rows, world):
            r0, r1 = w0 * 16, min(w1 * 16, a.num_rows)
            e0, e1 = a.row_ptr[r0], a.row_ptr[r1]
            sl = orc.Csr(r1 - r0, a.num_cols, a.row_ptr[r0:r1 + 1] - e0, a.col_idx[e0:e1], a.values[e0:e1])
            part = orc.partition(sl)
            snc, sdens, _ = orc.features(part)
            assert np.array_equal(snc, nc[w0:w1]) and np.array_equal(sdens.view(np.int64), dens[w0:w1].view(np.int64))
            assert np.array_equal(orc.classify(snc, sdens), codes[w0:w1])
            c0, c1 = full.win_col_ptr[w0], full.win_col_ptr[w1]
            assert np.array_equal(part.nonzero_cols, full.nonzero_cols[c0:c1])
            assert np.array_equal(part.cond_cols, full.cond_cols[e0:e1])


class _DenseWindows:
    """Stand-in for a WindowSet on CPU: the rows [r0, r1) of a dense operator."""

    def __init__(self, a_rows):
        self.a = a_rows
        self.codes = torch.zeros(1, dtype=torch.uint8)


def _dense_fused(windows, assignment, x, m, precision, want_z):
    z = windows.a @ x.to(torch.float64)
    return z @ m.to(torch.float64), (z if want_z else None)


class _DenseLayer:
    """Stand-in for fused.FusedLayer (same part interface) over a _DenseWindows."""

    def __init__(self, windows, assignment, x, m, precision, want_z):
        self.a, self.x, self.m = windows.a, x.to(torch.float64), m.to(torch.float64)
        self.d_out = int(m.shape[1])
        self.out = torch.full((self.a.shape[0], self.d_out), float("nan"), dtype=torch.float64)
        self.z = torch.full((self.a.shape[0], self.x.shape[1]), float("nan"), dtype=torch.float64)

    def parts(self, bounds):
        return [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1)]

    def run(self, part):
        r0, r1 = min(16 * part[0], self.a.shape[0]), min(16 * part[1], self.a.shape[0])
        self.z[r0:r1] = self.a[r0:r1] @ self.x
        self.out[r0:r1] = self.z[r0:r1] @ self.m

    def result(self):
        return self.out, self.z


def _worker(rank, world, port, a_np, x_np, labels_np, w1_np, w2_np, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gcn_model.fused_aggregate_update = _dense_fused
        gcn_model.FusedLayer = _DenseLayer
        gcn_model.grad_weight = lambda z, g: z.t() @ g.to(z.dtype)  # dense stand-in for the K7 kernel
        a = torch.from_numpy(a_np)
        n = a.shape[0]
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum((a_np != 0).sum(1), out=rp[1:])
        ranges = shard_window_ranges(rp, n, world)
        sh = Shard(ranges, rank, n)
        # ragged all-gather of rows
        full = torch.arange(n * 3, dtype=torch.float64).reshape(n, 3)
        assert torch.equal(sh.all_gather_rows(full[sh.row0:sh.row1]), full)
        # sharded 2-layer epoch (dense stand-in for the fused kernels)
        x = torch.from_numpy(x_np)
        labels = torch.from_numpy(labels_np)
        w1 = torch.from_numpy(w1_np).requires_grad_(True)
        w2 = torch.from_numpy(w2_np).requires_grad_(True)
        win = _DenseWindows(a[sh.row0:sh.row1])
        asg = object()
        h = torch.relu(gcn_model.gcn_layer(x, w1, win, win, asg, "bf16", sh))
        logits = gcn_model.gcn_layer(h, w2, win, win, asg, "bf16", sh)
        loss = torch.nn.functional.cross_entropy(logits, labels)
        loss.backward()
        out_q.put((rank, float(loss.detach()), w1.grad.numpy(), w2.grad.numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_gcn_autograd_matches_single_process():
    rng = np.random.default_rng(0)
    n = 100
    a = (rng.random((n, n)) < 0.08).astype(np.float64)
    a = np.maximum(a, a.T) + np.eye(n)
    d = 1.0 / np.sqrt(a.sum(1))
    a = a * d[:, None] * d[None, :]  # symmetric gcn operator
    x = rng.uniform(-1, 1, (n, 12))
    labels = rng.integers(0, 5, n)
    w1 = rng.uniform(-0.5, 0.5, (12, 8))
    w2 = rng.uniform(-0.5, 0.5, (8, 5))
    # single process reference
    tw1 = torch.from_numpy(w1).requires_grad_(True)
    tw2 = torch.from_numpy(w2).requires_grad_(True)
    ta = torch.from_numpy(a)
    logits = ta @ torch.relu(ta @ torch.from_numpy(x) @ tw1) @ tw2
    loss = torch.nn.functional.cross_entropy(logits, torch.from_numpy(labels))
    loss.backward()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, a, x, labels, w1, w2, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, l, g1, g2 in res:
        assert abs(l - float(loss.detach())) < 1e-12
        np.testing.assert_allclose(g1, tw1.grad.numpy(), rtol=1e-4, atol=1e-9)
        np.testing.assert_allclose(g2, tw2.grad.numpy(), rtol=1e-4, atol=1e-9)


def test_shard_ranges_by_window_cost():
    """shard_window_ranges with a per-window cost: contiguous, covering, ~equal cost (each range's
    cost within one window's cost of total/world); a cost array of the wrong length is rejected."""
    import numpy as np

    from paper_2412_08902_b200.shard import shard_window_ranges

    rng = np.random.default_rng(0)
    n, wh = 1000, 16
    W = -(-n // wh)
    lens = rng.integers(0, 50, n)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    cost = rng.uniform(0.0, 10.0, W)
    for world in (1, 2, 3, 8):
        r = shard_window_ranges(rp, n, world, wh, window_cost=cost)
        assert r[0][0] == 0 and r[-1][1] == W and all(r[i][1] == r[i + 1][0] for i in range(world - 1))
        sums = [cost[a:b].sum() for a, b in r]
        assert max(sums) - cost.sum() / world <= cost.max() + 1e-9
    try:
        shard_window_ranges(rp, n, 2, wh, window_cost=cost[:-1])
        raise AssertionError("expected ValueError")
    except ValueError as e:
        assert "one entry per window" in str(e)
