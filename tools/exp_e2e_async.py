"""Experiment (not product): end-to-end host-memory SpMM at C2 N=128 -- synchronous spmm_hybrid vs
spmm_hybrid_async with 1 / 2 / 3 requests in flight, with and without a caller-owned ring of
pinned result buffers (wall clock over 20 requests after warm-up)."""
import sys, os, json, time
from collections import deque
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen
from paper_2412_08902_b200.gnn import normalize_adj

torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
n, dim, k = a.num_rows, 128, 20
xh = (torch.rand(n, dim) * 2 - 1).to(torch.bfloat16).pin_memory()
ring = [torch.empty(n, dim, dtype=torch.float32, pin_memory=True) for _ in range(4)]


def run(depth, use_ring):
    def one(i):
        return hc.spmm_hybrid_async(ws, asg, xh, out=ring[i % len(ring)] if use_ring else None)
    for i in range(4):
        one(i).result()
    torch.cuda.synchronize()
    q = deque()
    t = time.perf_counter()
    for i in range(k):
        q.append(one(i))
        if len(q) == depth:
            q.popleft().result()
    while q:
        q.popleft().result()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e3


for _ in range(3):
    hc.spmm_hybrid(ws, asg, xh)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(k):
    r = hc.spmm_hybrid(ws, asg, xh)
    del r
torch.cuda.synchronize()
res = {"sync_ms": round((time.perf_counter() - t) / k * 1e3, 3)}
if os.environ.get("PARTS_SWEEP"):
    from paper_2412_08902_b200 import executors as ex
    for parts in (1, 2, 4, 8, 1, 2, 4, 8):
        ex.ASYNC_PIPELINE_PARTS = parts
        res.setdefault(f"async_d2_ring_parts{parts}_ms", []).append(round(run(2, True), 3))
else:
    for depth in (1, 2, 3):
        for use_ring in (False, True):
            res[f"async_d{depth}_{'ring' if use_ring else 'alloc'}_ms"] = round(run(depth, use_ring), 3)
print(json.dumps(res), flush=True)
