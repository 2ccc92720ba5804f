"""Experiment (not product): C5 (R-MAT scale 24) tile launch vs the L2 hot-row budget of the
class-tagged plan (executors.L2_HOT_BYTES): budget 0 = every gathered X row evict_first, huge =
every row evict_last (the round-1 behaviour); results must be bitwise identical (cache policy
only).  Prints the class histogram and the tile-launch time per budget (CUDA events, 5 reps)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200 import _lib, executors, graphgen  # noqa: E402
from paper_2412_08902_b200.executors import DeviceOperand, get_plan  # noqa: E402
from paper_2412_08902_b200.gnn import normalize_adj  # noqa: E402

scale = int(os.environ.get("C5_SCALE", "24"))
dim = int(os.environ.get("C5_DIM", "128"))
torch.cuda.set_device(0)
adj = graphgen.rmat(scale, 33, seed=0)
adj.symmetric = True
a = normalize_adj(adj, "gcn")
del adj
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
print(json.dumps({"n": a.num_rows, "nnz": a.nnz, "tile": plan.n_tile, "l2_shift": plan.l2_shift,
                  "hist": plan.l2_hist}), flush=True)
x = graphgen.dense_features(a.num_rows, dim, seed=1)
xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
z = torch.empty((a.num_rows, dim), dtype=torch.float32, device="cuda")
W = len(ws)
part = (0, W, 0, plan.n_tile, 0, 0)
ref = None
# same-harness baseline: the untagged plan (plain row indices, the CLS = false kernel)
tagged = plan.gidx.clone()
low = (1 << plan.l2_shift) - 1
plan.gidx.copy_(torch.where(plan.gidx >= 0, plan.gidx & low, plan.gidx))
shift = plan.l2_shift
plan.l2_shift = 0
for _ in range(2):
    plan.run(xop, z, dim, part=part)
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    plan.run(xop, z, dim, part=part)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ref = z.clone()
print(json.dumps({"untagged": True, "tile_ms": sorted(ts)[len(ts) // 2], "all_ms": ts}), flush=True)
plan.gidx.copy_(tagged)
del tagged
plan.l2_shift = shift
budgets = [int(v) for v in os.environ.get("C5_BUDGETS_MB", "0,64,100000").split(",")]
for mb in budgets:
    executors.L2_HOT_BYTES_OVERRIDE = mb << 20
    hot = plan.l2_hot_min(dim * 2)
    for _ in range(2):
        plan.run(xop, z, dim, part=part)
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        plan.run(xop, z, dim, part=part)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    same = bool(torch.equal(ref, z))
    hot_rows = sum(plan.l2_hist[c] for c in range(hot, 32))
    print(json.dumps({"budget_mb": mb, "hot_min": hot, "hot_rows": hot_rows, "tile_ms": sorted(ts)[len(ts) // 2],
                      "all_ms": ts, "bitwise_same": same}), flush=True)
