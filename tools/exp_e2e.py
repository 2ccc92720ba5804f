"""Experiment (not product): where does the end-to-end spmm_hybrid time go (C2, dim 128)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import get_plan, stage_operand, _alloc_z, _check_window_bounds

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a); asg = hc.classify_windows(hc.default_model(), ws)
x = graphgen.dense_features(a.num_rows, 128, seed=1)
xh = x.cpu().pin_memory()
plan = get_plan(ws, asg, "bf16")

def timeit(name, fn, k=10):
    for _ in range(2): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); print(f"{name:40s} {(time.perf_counter() - t) / k * 1e3:8.3f} ms", flush=True)

timeit("full spmm_hybrid (host in/out)", lambda: hc.spmm_hybrid(ws, asg, xh))
timeit("check_window_bounds", lambda: _check_window_bounds(ws, a.num_rows))
timeit("get_plan", lambda: get_plan(ws, asg, "bf16"))
timeit("stage_operand (H2D 60 MB)", lambda: stage_operand(xh, "bf16", torch.device("cuda", 0)))
xop, _ = stage_operand(xh, "bf16", torch.device("cuda", 0))
z, ldz = _alloc_z(a.num_rows, 128, torch.device("cuda", 0))
timeit("plan.run (device)", lambda: plan.run(xop, z, ldz))
def parts_run():
    for p in plan.parts(4): plan.run(xop, z, ldz, part=p)
timeit("plan.run 4 parts (device)", parts_run)
host = torch.empty((a.num_rows, 128), dtype=torch.float32, pin_memory=True)
timeit("D2H 119 MB pinned", lambda: host.copy_(z[:, :128], non_blocking=True))
timeit("pinned alloc", lambda: torch.empty((a.num_rows, 128), dtype=torch.float32, pin_memory=True))
