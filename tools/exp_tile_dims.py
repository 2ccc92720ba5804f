"""Experiment (not product): C2 hybrid SpMM time per feature width (CUDA events, 20 launches)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200 import executors as ex
from paper_2412_08902_b200.executors import get_plan, stage_operand, _alloc_z

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
prec = os.environ.get("PREC", "bf16")
plan = get_plan(ws, hc.classify_windows(hc.default_model(), ws), prec)
res = {}
pads = [int(p) for p in os.environ.get("PADS", "1").split(",")]
if os.environ.get("NPR3") is not None:
    from paper_2412_08902_b200 import _lib
    _lib.call("hcs_set_tile_npr3", int(os.environ["NPR3"]))
for dim in [int(d) for d in os.environ.get("DIMS", "16,32").split(",")]:
  for pad in pads:
    ex.PAD_TO_SLICE = bool(pad)
    x = torch.rand(a.num_rows, dim, device="cuda")
    xop, _ = stage_operand(x, prec, torch.device("cuda"), tf32_round=prec == "tf32")
    z, ldz = _alloc_z(a.num_rows, dim, torch.device("cuda"))
    for _ in range(3):
        plan.run(xop, z, ldz)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(20):
        plan.run(xop, z, ldz)
    e.record(); torch.cuda.synchronize()
    res[f"{dim}" + (f"_pad{pad}" if len(pads) > 1 else "")] = round(s.elapsed_time(e) / 20, 4)
print(json.dumps(res), flush=True)
