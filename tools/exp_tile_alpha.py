"""Experiment (not product): tile launch time vs the cost-weighted warp-range alpha
(HybridPlan.tile_alpha -> hcs_spmm_tile_balanced; 0 = uniform chunk counts) on C5 (tile windows only) or C2."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan

cfg = os.environ.get("CFG", "c5")
alphas = [int(v) for v in os.environ.get("ALPHAS", "0,16,64,256,0").split(",")]
dims = [int(v) for v in os.environ.get("DIMS", "128").split(",")]
torch.cuda.set_device(0)
dev = torch.device("cuda")
adj = graphgen.rmat(24, 33, seed=0) if cfg == "c5" else graphgen.reddit_shaped(seed=0)
adj.symmetric = True
a = normalize_adj(adj, "gcn")
del adj
ws = hc.partition(a)
plan = get_plan(ws, hc.classify_windows(hc.default_model(), ws), "bf16")
n, W = a.num_rows, len(ws)
part = (0, W, 0, plan.n_tile, 0, 0)
for dim in dims:
    x = graphgen.dense_features(n, dim, seed=1)
    xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
    ref = None
    for al in alphas:
        plan.tile_alpha = al
        z = torch.zeros((n, dim), dtype=torch.float32, device=dev)
        for _ in range(2):
            plan.run(xop, z, dim, part=part)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(7 if cfg == "c5" else 20):
            s.record(); plan.run(xop, z, dim, part=part); e.record(); e.synchronize()
            ts.append(s.elapsed_time(e))
        z2 = z.clone(); plan.run(xop, z2, dim, part=part); torch.cuda.synchronize()
        if ref is None:
            ref = z.clone()
        print(json.dumps({"cfg": cfg, "dim": dim, "alpha": al, "tile_ms": sorted(ts)[len(ts) // 2],
                          "min_ms": min(ts), "run_to_run_bitwise": bool(torch.equal(z, z2)),
                          "max_rel_vs_alpha0": float(((z - ref).abs().max() / ref.abs().max()).item())}), flush=True)
