"""Experiment (not product): C5 (R-MAT scale 24) tile launch with / without the L2 row prefetch one
chunk ahead of the cp.async ring (hcs_set_tile_prefetch); results must be bitwise identical."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200 import _lib, graphgen  # noqa: E402
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
x = graphgen.dense_features(a.num_rows, dim, seed=1)
xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
W = len(ws)
parts = {"tile": (0, W, 0, plan.n_tile, 0, 0), "all": None}
ref = None
for on in (0, 1, 0, 1):
    _lib.call("hcs_set_tile_prefetch", on)
    res = {"prefetch": on}
    for name, part in parts.items():
        z = torch.empty((a.num_rows, dim), dtype=torch.float32, device="cuda")
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
        res[name + "_ms"] = sorted(ts)[2]
        if name == "all":
            if ref is None:
                ref = z.clone()
            res["bitwise_same"] = bool(torch.equal(ref, z))
    print(json.dumps(res), flush=True)
_lib.call("hcs_set_tile_prefetch", 1)
