"""Experiment (evidence, not product): the compute side of row-window sharding measured on ONE GPU,
with shards balanced by nnz (default) or by the path cost model (shard.window_costs).
For P = 1, 2, 4, 8 every rank's shard of C2 / C5 is built exactly as bench.py --gpus P builds it
(Shard.from_operator + local_operator + partition + plan) and its hybrid SpMM timed in turn (CUDA
events, median of 5); reported: max over ranks (the step's critical path), min, and the bytes each
rank receives in the all-gather of bf16 output rows.  The exchange itself needs the 8-GPU box."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200 import _lib, graphgen  # noqa: E402
from paper_2412_08902_b200.executors import DeviceOperand, _alloc_z, get_plan  # noqa: E402
from paper_2412_08902_b200.gnn import normalize_adj  # noqa: E402
from paper_2412_08902_b200.shard import Shard, window_costs  # noqa: E402

torch.cuda.set_device(0)
dim = 128
for cfg in os.environ.get("CFGS", "c2,c5").split(","):
    adj = graphgen.reddit_shaped(seed=0) if cfg == "c2" else graphgen.rmat(24, 33, seed=0)
    adj.symmetric = True
    a = normalize_adj(adj, "gcn")
    del adj
    x = graphgen.dense_features(a.num_rows, dim, seed=1)
    xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
    wsf = hc.partition(a)
    costs = window_costs(wsf, hc.classify_windows(hc.default_model(), wsf).codes)
    del wsf
    torch.cuda.empty_cache()
    for mode, P in [(m, p) for m in ("nnz", "cost") for p in (1, 2, 4, 8) if not (m == "cost" and p == 1)]:
        times = []
        for r in range(P):
            sh = Shard.from_operator(a, P, r, window_cost=costs if mode == "cost" else None)
            loc = sh.local_operator(a)
            ws = hc.partition(loc)
            plan = get_plan(ws, hc.classify_windows(hc.default_model(), ws), "bf16")
            z, ldz = _alloc_z(loc.num_rows, dim, x.device)
            for _ in range(2):
                plan.run(xop, z, ldz)
            ts = []
            for _ in range(5):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                plan.run(xop, z, ldz)
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e))
            times.append(sorted(ts)[2])
            del plan, ws, loc, z
            torch.cuda.empty_cache()
        recv = (a.num_rows - a.num_rows // P) * dim * 2 if P > 1 else 0
        print(json.dumps({"config": cfg, "balance": mode, "P": P, "max_rank_ms": round(max(times), 3), "min_rank_ms": round(min(times), 3),
                          "per_rank_ms": [round(t, 3) for t in times],
                          "allgather_recv_bytes_per_rank": recv}), flush=True)
    del a, x, xop
    torch.cuda.empty_cache()
