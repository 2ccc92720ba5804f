"""Experiment (not product): the drop-in call spmm_hybrid(windows, asg, DenseMatrix(float64 numpy))
at C2 / N = 128 split into its phases: host staging (conversion + H2D), the kernels, the D2H."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200 import _lib, executors as ex, graphgen  # noqa: E402
from paper_2412_08902_b200.gnn import normalize_adj  # noqa: E402


def t_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(sorted(ts)[len(ts) // 2], 3)


torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0)
adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
dim = 128
x = graphgen.dense_features(a.num_rows, dim, seed=1)
x64 = x.double().cpu().numpy()
dm = hc.DenseMatrix(x64)
dev = x.device
res = {"cpus": len(os.sched_getaffinity(0))}
res["numpy_copy_238MB_1thread"] = t_ms(lambda: x64.copy())
for th in (1, 4, 8, 16):
    ex.HOST_STAGE_THREADS = th
    res[f"stage_f64_threads{th}"] = t_ms(lambda: ex.stage_operand(dm, "bf16", dev))
ex.HOST_STAGE_THREADS = None
res["h2d_pageable_f64_then_cast"] = t_ms(lambda: torch.from_numpy(x64).to(dev).to(torch.bfloat16))
res["kernels_device_operand"] = t_ms(lambda: hc.spmm_hybrid(ws, asg, x))
res["dropin_total"] = t_ms(lambda: hc.spmm_hybrid(ws, asg, dm))
xb = x.cpu().pin_memory()
res["pinned_bf16_sync_total"] = t_ms(lambda: hc.spmm_hybrid(ws, asg, xb))
for blk in (2, 4, 16, 32):
    ex.HOST_STAGE_BLOCK_BYTES = blk << 20
    res[f"stage_block{blk}MB"] = t_ms(lambda: ex.stage_operand(dm, "bf16", dev))
print(res, flush=True)
