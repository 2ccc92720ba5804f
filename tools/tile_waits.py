"""Wait-time breakdown of the tile kernel on the C2 graph (debug counters)."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import _lib, graphgen
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan

adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a); asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
names = ["prod wait idx_full", "prod wait empty", "prod wait_group(publish)", "idx wait idx_empty",
         "ent wait empty", "builder wait full", "mma wait built", "mma wait acce", "epi wait accf", "mma issue block",
         "prod total", "loaders total", "builders total", "mma+epi total", "builder build", "cta total"]
sw = int(os.environ.get("SWITCHES", "0"))
_lib.call("hcs_debug_tile_switches", sw)
print("switches", sw)
for dim in [int(d) for d in (sys.argv[1:] or ["128", "32"])]:
    x = graphgen.dense_features(a.num_rows, dim, seed=1)
    xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
    ldz = -(-dim // 4) * 4
    z = torch.empty((a.num_rows, ldz), device="cuda")
    plan.run(xop, z, ldz); torch.cuda.synchronize()
    L = _lib.lib()
    L.hcs_debug_tile_profile(1, None, 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.run(xop, z, ldz); e1.record(); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (16 * 148))()
    L.hcs_debug_tile_profile(1, buf, 16 * 148)
    L.hcs_debug_tile_profile(0, None, 0)
    arr = np.frombuffer(buf, dtype=np.uint64).reshape(148, 16).astype(np.float64)
    tot = arr[:, 15].mean()
    print(f"dim {dim}: {e0.elapsed_time(e1):.3f} ms, cta cycles {tot:.0f}")
    warps = {0: 4, 1: 4, 2: 4, 3: 1, 4: 1, 5: 2, 6: 1, 7: 1, 8: 1, 9: 1, 14: 2}
    for i, nm in enumerate(names):
        if nm == "-":
            continue
        v = arr[:, i].mean() / warps.get(i, 1)
        print(f"  {nm:26s} {v:14.0f}  {100 * v / tot:5.1f}% of CTA time (per warp)")
