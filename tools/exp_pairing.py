"""Experiment (not product): tile kernel with paired feature slices on/off on C2 (dims 96/128/
192/256), timing (CUDA events) and max relative difference between the two modes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
plan = get_plan(ws, hc.classify_windows(hc.default_model(), ws), "bf16")
for dim in (96, 128, 192, 256):
    x = graphgen.dense_features(a.num_rows, dim, seed=1)
    xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
    zs = {}
    for pair in (0, 1):
        _lib.call("hcs_set_tile_pairing", pair)
        z = torch.empty((a.num_rows, dim), dtype=torch.float32, device="cuda")
        for _ in range(3):
            plan.run(xop, z, dim)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(20):
            plan.run(xop, z, dim)
        e.record(); torch.cuda.synchronize()
        z2 = torch.empty_like(z); plan.run(xop, z2, dim)
        zs[pair] = (z, s.elapsed_time(e) / 20, bool(torch.equal(z, z2)))
    d = float((zs[0][0] - zs[1][0]).abs().max() / zs[0][0].abs().max())
    print(json.dumps({"dim": dim, "ms_unpaired": zs[0][1], "ms_paired": zs[1][1], "max_rel_diff": d,
                      "deterministic": [zs[0][2], zs[1][2]]}), flush=True)
_lib.call("hcs_set_tile_pairing", 1)
