"""Experiment (not product): does binding the host thread to the GPU's NVML-reported local CPUs
(before allocating the pinned buffers) steady the async end-to-end time?  Prints the GPU's
affinity mask, then e2e ms for the default affinity and for the local cores."""
import sys, os, json, time
from collections import deque
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen
from paper_2412_08902_b200.gnn import normalize_adj

mode = os.environ.get("MODE", "local")
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
words = pynvml.nvmlDeviceGetCpuAffinity(h, 4)
cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
info = {"ncpu": os.cpu_count(), "gpu_local_cpus": len(cpus), "first": cpus[:4], "mode": mode}
if mode == "local" and cpus:
    os.sched_setaffinity(0, cpus)
torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
n, dim, k = a.num_rows, 128, 20
xh = (torch.rand(n, dim) * 2 - 1).to(torch.bfloat16).pin_memory()
ring = [torch.empty(n, dim, dtype=torch.float32, pin_memory=True) for _ in range(3)]
for i in range(4):
    hc.spmm_hybrid_async(ws, asg, xh, out=ring[i % 3]).result()
res = []
for rep in range(3):
    torch.cuda.synchronize()
    q = deque()
    t = time.perf_counter()
    for i in range(k):
        q.append(hc.spmm_hybrid_async(ws, asg, xh, out=ring[i % 3]))
        if len(q) == 2:
            q.popleft().result()
    while q:
        q.popleft().result()
    torch.cuda.synchronize()
    res.append(round((time.perf_counter() - t) / k * 1e3, 3))
info["e2e_ms"] = res
print(json.dumps(info), flush=True)
