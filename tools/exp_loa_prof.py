"""Experiment (not product): LOA per-phase SM cycles on C2 (needs the instrumented build
tools/exp_libs/lib_loa_prof.so via HCS_LIB_PATH)."""
import sys, os, ctypes, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_08902_b200 import graphgen, layout, _lib
from paper_2412_08902_b200.matrices import Graph
torch.cuda.set_device(0)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
g = Graph(adj.num_rows, adj, True)
t = time.perf_counter(); layout.build_windows_optimized(g, vw=128); torch.cuda.synchronize()
print("loa s", time.perf_counter() - t)
buf = (ctypes.c_ulonglong * 8)()
_lib.lib().hcs_loa_prof(buf)
names = ["scan", "cand+prefix", "pull", "argmax", "admit", "-", "steps"]
tot = sum(buf[i] for i in range(5))
for i, nm in enumerate(names[:5]):
    print(f"{nm:12s} {buf[i] / 1e6:10.1f} Mcycles {100 * buf[i] / tot:5.1f}%  {buf[i] / max(buf[6], 1):8.0f} cyc/step")
print("steps", buf[6])
