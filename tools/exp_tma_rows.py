"""Experiment (not product): part of each chunk's X rows by TMA gather4 (hcs_set_tile_tma_rows
4 / 8 of every 16) vs all rows by cp.async, C2 hybrid SpMM at N = 64 / 128 (CUDA events)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import get_plan, stage_operand, _alloc_z

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
plan = get_plan(ws, hc.classify_windows(hc.default_model(), ws), "bf16")
reps = int(os.environ.get("REPS", "20"))
for dim in (64, 128):
    x = torch.rand(a.num_rows, dim, device="cuda")
    xop, _ = stage_operand(x, "bf16", torch.device("cuda"))
    z, ldz = _alloc_z(a.num_rows, dim, torch.device("cuda"))
    res = {"dim": dim}
    outs = {}
    for rows in (0, 4, 8, 0, 4, 8):
        _lib.call("hcs_set_tile_tma_rows", rows)
        for _ in range(3):
            plan.run(xop, z, ldz)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(reps):
            plan.run(xop, z, ldz)
        e.record(); torch.cuda.synchronize()
        res.setdefault(f"tma{rows}_ms", []).append(round(s.elapsed_time(e) / reps, 4))
        outs[rows] = z.clone()
    res["equal"] = [bool(torch.equal(outs[0], outs[r])) for r in (4, 8)]
    print(json.dumps(res), flush=True)
_lib.call("hcs_set_tile_tma_rows", 0)
