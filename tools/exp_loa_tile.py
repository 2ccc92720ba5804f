"""Experiment (not product): tile-path SpMM on the community Reddit-shaped graph before and
after LOA, with plan statistics (chunks, entries per chunk, overflow chunks).
EXP_ONLY=after|before restricts the run (for ncu -c 1 captures)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, layout, _lib
from paper_2412_08902_b200.executors import DeviceOperand, get_plan
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.matrices import Graph

torch.cuda.set_device(0)
only = os.environ.get("EXP_ONLY")
adj = graphgen.reddit_community(seed=0); adj.symmetric = True
n, dim = adj.num_rows, 128
x = graphgen.dense_features(n, dim, seed=1)
cases = []
if only != "after":
    cases.append(("before", normalize_adj(adj, "gcn"), x))
if only != "before":
    g = Graph(n, adj, True)
    grouping = layout.build_windows_optimized(g, vw=128)
    g2, perm = layout.reorder(g, grouping)
    cases.append(("after", normalize_adj(g2, "gcn"), x[torch.from_numpy(np.argsort(perm)).cuda()].contiguous()))
for name, a, xx in cases:
    ws = hc.partition(a)
    asg = hc.classify_windows(hc.default_model(), ws)
    plan = get_plan(ws, asg, "bf16")
    ept = (plan.ent_ptr[1:] - plan.ent_ptr[:-1]).float()
    xop = DeviceOperand(xx, dim, dim, _lib.DTYPE_BF16)
    z = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    for _ in range(3):
        plan.run(xop, z, dim)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(10):
        plan.run(xop, z, dim)
    e.record(); torch.cuda.synchronize()
    print(json.dumps({"case": name, "nnz": a.nnz, "chunks": plan.nchunks, "ent_per_chunk": float(ept.mean()),
                      "chunks_gt128": int((ept > 128).sum()), "ent_max": int(ept.max()),
                      "sum_ncols": int(ws.ncols().sum()), "ms": s.elapsed_time(e) / 10}), flush=True)
