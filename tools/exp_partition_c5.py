"""Experiment (not product): K1 partition + selection time at C5 (R-MAT scale 24, sort path)
and at C2 (bitmap path), warm, CUDA events; window-size histogram of C5."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen
from paper_2412_08902_b200.gnn import normalize_adj

torch.cuda.set_device(0)
for name in ("c2", "c5"):
    adj = graphgen.reddit_shaped(seed=0) if name == "c2" else graphgen.rmat(24, 33, seed=0)
    adj.symmetric = True
    a = normalize_adj(adj, "gcn")
    del adj
    rp = a.row_ptr
    W = (a.num_rows + 15) // 16
    idx = torch.arange(W + 1, device=rp.device) * 16
    wn = rp[idx.clamp(max=a.num_rows)].diff()
    hist = {k: [int(((wn > lo) & (wn <= hi)).sum()), int(wn[(wn > lo) & (wn <= hi)].sum())]
            for k, lo, hi in (("<=1024", 0, 1024), ("<=8192", 1024, 8192), (">8192", 8192, 1 << 40))}
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        ws = hc.partition(dataclasses.replace(a, _derived={}))  # no cached windows
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
        del ws
    print(json.dumps({"graph": name, "nnz": int(a.nnz), "windows_count_nnz": hist,
                      "partition_ms": [round(x, 2) for x in ts]}), flush=True)
    del a
    torch.cuda.empty_cache()
