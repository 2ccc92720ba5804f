"""Experiment (not product): time the C2 SpMM with the shipped assignment, all-TILE and
all-SCALAR paths on the same graph, dims 32/128 (CUDA events)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan, Assignment

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
W = len(ws)
res = {}
for name, asg in [("scalar", Assignment(torch.zeros(W, dtype=torch.uint8, device="cuda"))),
                  ("tile", hc.classify_windows(hc.default_model(), ws))]:
    plan = get_plan(ws, asg, "bf16")
    for dim in (32, 64, 128):
        x = graphgen.dense_features(a.num_rows, dim, seed=1)
        xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
        z = torch.empty((a.num_rows, dim), dtype=torch.float32, device="cuda")
        for _ in range(3): plan.run(xop, z, dim)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(20): plan.run(xop, z, dim)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 20
        res[f"{name}_d{dim}"] = ms
        print(name, dim, f"{ms:.3f} ms", f"{2*a.nnz*dim/ms/1e6:.0f} GFLOP/s", flush=True)
print(json.dumps(res))
