"""Experiment (not product): how evenly the tile kernel's chunk-balanced warp ranges split the
per-chunk work (entries, a proxy for the dense-chunk path) on C2 / C5 plans."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import get_plan

cfg = os.environ.get("CFG", "c5")
torch.cuda.set_device(0)
if cfg == "c5":
    adj = graphgen.rmat(24, 33, seed=0)
else:
    adj = graphgen.reddit_shaped(seed=0)
adj.symmetric = True
a = normalize_adj(adj, "gcn")
del adj
ws = hc.partition(a)
plan = get_plan(ws, hc.classify_windows(hc.default_model(), ws), "bf16")
ept = (plan.ent_ptr[1:] - plan.ent_ptr[:-1]).double()
C = ept.numel()
groups = 148 * 8 // 2  # paired 64-feature slices: 592 warp pairs walk balanced chunk ranges
bnd = (torch.arange(groups + 1, device=ept.device, dtype=torch.float64) * C / groups).floor().long()
cs = torch.zeros(C + 1, dtype=torch.float64, device=ept.device)
torch.cumsum(ept, 0, out=cs[1:])
per = cs[bnd[1:]] - cs[bnd[:-1]]
dense = (ept > 128)
cs2 = torch.zeros(C + 1, dtype=torch.float64, device=ept.device)
torch.cumsum(torch.where(dense, ept - 128, torch.zeros_like(ept)), 0, out=cs2[1:])
per_over = cs2[bnd[1:]] - cs2[bnd[:-1]]
hist = torch.histc(ept.float(), bins=8, min=0, max=1024).tolist()
print(json.dumps({"cfg": cfg, "chunks": C, "ent_mean": float(ept.mean()), "chunks_gt128": int(dense.sum()),
                  "ent_over128": float(cs2[-1]), "hist_0_1024_by128": hist,
                  "range_entries_max_over_mean": float(per.max() / per.mean()),
                  "range_entries_p99_over_mean": float(per.quantile(0.99) / per.mean()),
                  "range_over128_max": float(per_over.max()), "range_over128_mean": float(per_over.mean()),
                  "worst_ranges": [int(i) for i in torch.topk(per, 5).indices.tolist()]}), flush=True)
