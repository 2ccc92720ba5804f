"""C3 epoch time per layer order (model.gcn_layer order): fused (A X) W vs update-first A (X W)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200 import graphgen  # noqa: E402
from paper_2412_08902_b200.model import Gcn2  # noqa: E402

adj, a, _ = bench.make_graph("c2", 0, "powerlaw")
n = a.num_rows
ws = hc.partition(a)
x = graphgen.dense_features(n, 128, seed=1, dtype=torch.float32)
dev = torch.device("cuda")
labels = torch.randint(0, 41, (n,), generator=torch.Generator(device=dev).manual_seed(2), device=dev)
for order in [("fused", "fused"), ("update_first", "fused"), ("fused", "update_first"),
              ("update_first", "update_first"), ("fused", "fused")]:
    m = Gcn2(128, 64, 41, seed=0, order=order)
    for _ in range(5):
        m.epoch(x, labels, ws)
    torch.cuda.synchronize()
    best = []
    for rep in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            loss = m.epoch(x, labels, ws)
        e.record()
        torch.cuda.synchronize()
        best.append(s.elapsed_time(e) / 20)
    k = bench.epoch_kernels(lambda: m.epoch(x, labels, ws))
    print(json.dumps({"order": order, "ms": best, "loss": float(loss),
                      "kernels_us": k.get("hcs_us_in_order") if k else None}), flush=True)
