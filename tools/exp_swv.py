"""Experiment (not product): tile-kernel slice width (hcs_set_tile_slice 4 vs 8) per feature width on C2."""
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
for dim in (40, 48, 72, 80, 96, 136, 160, 192):
    x = torch.rand(a.num_rows, dim, device="cuda")
    xop, _ = stage_operand(x, "bf16", torch.device("cuda"))
    z, ldz = _alloc_z(a.num_rows, dim, torch.device("cuda"))
    res = {"dim": dim, "ld": xop.ld}
    for swv in (4, 8):
        _lib.call("hcs_set_tile_slice", swv)
        for _ in range(3):
            plan.run(xop, z, ldz)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(10):
            plan.run(xop, z, ldz)
        e.record(); torch.cuda.synchronize()
        res[f"swv{swv}_ms"] = s.elapsed_time(e) / 10
    print(json.dumps(res), flush=True)
_lib.call("hcs_set_tile_slice", 0)
