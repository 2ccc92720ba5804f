"""Experiment (not product): tile kernel with pipeline parts switched off (C2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a); asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
for dim in [int(d) for d in os.environ.get("DIMS", "128,32").split(",")]:
    x = graphgen.dense_features(a.num_rows, dim, seed=1)
    xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
    z = torch.empty((a.num_rows, dim), dtype=torch.float32, device="cuda")
    for np_ in [int(v) for v in os.environ.get("NPS", "4").split(",")]:
        _lib.call("hcs_set_tile_producers", np_)
        combos = [(0, "full"), (1, "no-mma"), (3, "no-mma,no-build"), (7, "nothing (sync only)"), (4, "no-gather"),
                  (6, "no-gather,no-build"), (7 | 8, "sync only, no ent TMA"), (7 | 16, "sync only, no idx TMA"),
                  (7 | 24, "sync only, no TMAs"), (3 | 8, "gather only, no ent TMA"), (1 | 8, "gather+build, no ent TMA")]
        for bits, name in combos:
            _lib.call("hcs_debug_tile_switches", bits)
            for _ in range(2): plan.run(xop, z, dim)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); s.record()
            for _ in range(10): plan.run(xop, z, dim)
            e.record(); torch.cuda.synchronize()
            print(f"dim {dim} np {np_} {name:22s} {s.elapsed_time(e)/10:.3f} ms", flush=True)
_lib.call("hcs_debug_tile_switches", 0)
