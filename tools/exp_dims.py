"""Experiment (not product): C2 tile SpMM time for odd feature widths through stage_operand
(padded copies), and spmm_hybrid wall time for a device fp32 operand."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import get_plan, stage_operand, _alloc_z

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
for dim in (41, 48, 64, 96, 128):
    x = torch.rand(a.num_rows, dim, device="cuda")
    xop, _ = stage_operand(x, "bf16", torch.device("cuda"))
    z, ldz = _alloc_z(a.num_rows, dim, torch.device("cuda"))
    for _ in range(3):
        plan.run(xop, z, ldz)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(10):
        plan.run(xop, z, ldz)
    e.record(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        r = hc.spmm_hybrid(ws, asg, x)
    torch.cuda.synchronize()
    print(json.dumps({"dim": dim, "ld": xop.ld, "kernel_ms": s.elapsed_time(e) / 10,
                      "spmm_hybrid_wall_ms": (time.perf_counter() - t) / 10 * 1e3}), flush=True)
