"""Experiment (not product): one C2 N=128 tile launch with pairing PAIR (env) for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan

torch.cuda.set_device(0)
_lib.call("hcs_set_tile_pairing", int(os.environ.get("PAIR", "1")))
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
plan = get_plan(ws, hc.classify_windows(hc.default_model(), ws), "bf16")
x = graphgen.dense_features(a.num_rows, 128, seed=1)
xop = DeviceOperand(x, 128, 128, _lib.DTYPE_BF16)
z = torch.empty((a.num_rows, 128), dtype=torch.float32, device="cuda")
for _ in range(3):
    plan.run(xop, z, 128)
torch.cuda.synchronize()
