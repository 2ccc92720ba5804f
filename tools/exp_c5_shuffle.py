"""Experiment (not product): C5 tile launch with the plan's tile windows in a shuffled order (the
hub windows at the start of the id range then no longer land in the first warps' chunk ranges).
Shipping order vs random permutations; Z compared with the shipping order (summation order of
split windows differs)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan, HybridPlan

cfg = os.environ.get("CFG", "c5")
dim = 128
torch.cuda.set_device(0)
dev = torch.device("cuda")
adj = graphgen.rmat(24, 33, seed=0) if cfg == "c5" else graphgen.reddit_shaped(seed=0)
adj.symmetric = True
a = normalize_adj(adj, "gcn")
del adj
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
codes = asg.device_codes(dev)
n, W = a.num_rows, len(ws)
x = graphgen.dense_features(n, dim, seed=1)
xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)


def run(p, reps=5):
    z = torch.zeros((n, dim), dtype=torch.float32, device=dev)
    part = (0, W, 0, p.n_tile, 0, 0)
    for _ in range(2):
        p.run(xop, z, dim, part=part)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); p.run(xop, z, dim, part=part); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    return z, sorted(ts)[len(ts) // 2], ts


z0, t0, ts = run(plan)
print(json.dumps({"cfg": cfg, "order": "shipping", "tile_ms": t0, "all": ts}), flush=True)
orig_nonzero = torch.nonzero
for seed in (1, 2):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)

    def shuffled_nonzero(t, *args, **kw):  # HybridPlan.__init__: tile_list = nonzero(tile_mask)
        r = orig_nonzero(t, *args, **kw)
        if t.dtype == torch.bool and t.numel() == W and kw.get("_inner") is None and shuffled_nonzero.first:
            shuffled_nonzero.first = False
            f = r.flatten()
            return f[torch.randperm(f.numel(), generator=g, device=dev)][:, None]
        return r
    shuffled_nonzero.first = True
    torch.nonzero = shuffled_nonzero
    try:
        p2 = HybridPlan(ws, codes, "bf16")
    finally:
        torch.nonzero = orig_nonzero
    z2, t2, ts = run(p2)
    rel = float(((z2 - z0).abs().max() / z0.abs().max()).item())
    print(json.dumps({"cfg": cfg, "order": f"shuffle{seed}", "tile_ms": t2, "all": ts, "max_rel_vs_shipping": rel}),
          flush=True)
    del p2, z2
