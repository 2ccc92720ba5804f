"""Experiment (not product): K2 tile-plan build time per builder (CUDA events around
HybridPlan construction and around the hcs_tile_plan launch alone) on C2 / C5."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import HybridPlan

torch.cuda.set_device(0)
cfg = os.environ.get("PLAN_CFG", "c2")
adj = graphgen.reddit_shaped(seed=0) if cfg == "c2" else graphgen.rmat(24, 33, seed=0)
adj.symmetric = True
a = normalize_adj(adj, "gcn")
del adj
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
codes = asg.device_codes(torch.device("cuda"))
orig = _lib.call
for builder in (1, 0, 1, 0):
    _lib.call("hcs_set_tile_plan_builder", builder)
    ev = {}

    def timed_call(name, *args, _orig=orig):
        if name == "hcs_tile_plan":
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); _orig(name, *args); e.record(); ev["k"] = (s, e)
        else:
            _orig(name, *args)
    _lib.call = timed_call
    torch.cuda.synchronize(); t = time.perf_counter()
    p = HybridPlan(ws, codes, "bf16")
    torch.cuda.synchronize(); wall = (time.perf_counter() - t) * 1e3
    _lib.call = orig
    print(json.dumps({"cfg": cfg, "builder": builder, "plan_wall_ms": wall,
                      "hcs_tile_plan_ms": ev["k"][0].elapsed_time(ev["k"][1]) if "k" in ev else None}), flush=True)
    del p
