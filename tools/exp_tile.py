"""Experiment (not product): tile-kernel variants (producer warps x engine) on C2, dims 32/64/128."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan, set_tile_engine

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
nps = [int(v) for v in os.environ.get("NPS", "4,8,16").split(",")]
engines = os.environ.get("ENGINES", "mma_sync,tcgen05").split(",")
dims = [int(v) for v in os.environ.get("DIMS", "32,64,128").split(",")]
res = {}
ref = {}
for dim in dims:
    x = graphgen.dense_features(a.num_rows, dim, seed=1)
    xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
    z = torch.empty((a.num_rows, dim), dtype=torch.float32, device="cuda")
    for eng in engines:
        set_tile_engine(eng)
        for np_ in nps:
            if eng == "warp":
                _lib.call("hcs_set_tile_slice", np_ if np_ in (4, 8, 16) else 0)
            else:
                _lib.call("hcs_set_tile_producers", np_)
            for _ in range(3): plan.run(xop, z, dim)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); s.record()
            for _ in range(20): plan.run(xop, z, dim)
            e.record(); torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 20
            if dim not in ref:
                ref[dim] = z.clone()
            diff = float((z - ref[dim]).abs().max())
            res[f"{eng}_np{np_}_d{dim}"] = ms
            print(f"{eng:9s} np={np_:2d} dim={dim:3d} {ms:.3f} ms  {2*a.nnz*dim/ms/1e6:.0f} GFLOP/s  maxdiff_vs_first {diff:.3g}", flush=True)
set_tile_engine("auto"); _lib.call("hcs_set_tile_producers", 8)
print(json.dumps(res))
