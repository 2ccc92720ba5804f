"""Bounded CPU baseline of the reference algorithm -- TEST / BENCH INFRASTRUCTURE ONLY.

Times the reference's hybrid SpMM (restated in oracle/rowwin_oracle.py:
partition windows.py:81-106, classify selector.py:48-64, spmm_hybrid
executors.py:160-251 in float32) on a deterministic sample of 16-row windows of
the benchmark graph, on the host cores, and extrapolates GFLOP/s (2*nnz*dim/t).

Windows are row-local (windows.py:90-105), so a window cut from a 16-aligned
row slice is identical to the same window of the full partition; the gcn
normalisation of the sampled rows uses the reference formula (gnn.py:84-95)
with degrees taken from the full adjacency (unit values, no self loops).
Used only by bench.py (cpu_baseline leg and --impl reference).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import rowwin_oracle as orc

_G = {}


def _gcn_window_csr(rp, ci, deg_loops, lo, hi):
    """Rows [lo, hi) of D^-1/2 (A + I) D^-1/2 for a unit-valued A without self loops."""
    n = len(rp) - 1
    rows, cols = [], []
    for r in range(lo, hi):
        c = ci[rp[r]:rp[r + 1]].astype(np.int64)
        c = np.sort(np.append(c, r))
        rows.append(np.full(c.size, r - lo, dtype=np.int64))
        cols.append(c)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    inv = 1.0 / np.sqrt(deg_loops)
    vals = np.ones(rows.size) * inv[rows + lo] * inv[cols]
    counts = np.bincount(rows, minlength=hi - lo)
    row_ptr = np.zeros(hi - lo + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return orc.Csr(hi - lo, n, row_ptr, cols, vals)


def _work(args):
    wids, budget_s = args
    rp, ci, x, deg = _G["rp"], _G["ci"], _G["x"], _G["deg"]
    n = len(rp) - 1
    done_nnz = 0
    done = 0
    t0 = time.perf_counter()
    for w in wids:
        lo, hi = w * 16, min(w * 16 + 16, n)
        a = _gcn_window_csr(rp, ci, deg, lo, hi)
        ws = orc.partition(a)
        nc, dens, _ = orc.features(ws)
        codes = orc.classify(nc, dens)
        orc.spmm_hybrid(ws, codes, x, "f32")
        done_nnz += a.nnz
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return done_nnz, done, time.perf_counter() - t0


def sampled_gflops(row_ptr: np.ndarray, col_idx: np.ndarray, x: np.ndarray, budget_s: float = 10.0,
                   processes: int | None = None, stride: int = 73) -> dict:
    """Run the reference hybrid SpMM on every `stride`-th window (round-robin over
    `processes` forked workers) for about `budget_s` seconds; returns GFLOP/s."""
    n = len(row_ptr) - 1
    W = -(-n // 16)
    procs = processes or max(1, min(os.cpu_count() or 1, 32))
    wids = list(range(0, W, stride)) + [w for w in range(W) if w % stride]
    per = [wids[i::procs] for i in range(procs)]
    _G.update(rp=row_ptr, ci=col_idx, x=np.ascontiguousarray(x, dtype=np.float32),
              deg=(np.diff(row_ptr) + 1).astype(np.float64))
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    if procs == 1:
        res = [_work((per[0], budget_s))]
    else:
        with ctx.Pool(procs) as pool:
            res = pool.map(_work, [(p, budget_s) for p in per])
    wall = time.perf_counter() - t0
    nnz = sum(r[0] for r in res)
    windows = sum(r[1] for r in res)
    t = max(r[2] for r in res)
    dim = x.shape[1]
    return dict(gflops=2.0 * nnz * dim / t / 1e9, nnz=nnz, windows=windows, seconds=t, wall=wall, cores=procs,
                dim=dim)
