"""Experiment (not product): end-to-end spmm_hybrid (pinned host X -> host Z) on C2 vs the
number of pipelined parts, plus raw pinned H2D / D2H bandwidth of this box."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, executors
from paper_2412_08902_b200.gnn import normalize_adj

torch.cuda.set_device(0)
dev = torch.device("cuda")
for mb in (60, 120):
    h = torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    h2d = (mb << 20) * 10 / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    d2h = (mb << 20) * 10 / (time.perf_counter() - t) / 1e9
    print(json.dumps({"MB": mb, "h2d_GBps": h2d, "d2h_GBps": d2h}), flush=True)
adj = graphgen.reddit_shaped(seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
xh = graphgen.dense_features(a.num_rows, 128, seed=1).cpu().pin_memory()
for parts in (4, 8, 16, 32):
    executors.HOST_PIPELINE_PARTS = parts
    for _ in range(3):
        hc.spmm_hybrid(ws, asg, xh)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        r = hc.spmm_hybrid(ws, asg, xh)
        del r
    torch.cuda.synchronize()
    print(json.dumps({"parts": parts, "e2e_ms": (time.perf_counter() - t) / 10 * 1e3}), flush=True)

# device timeline of one pipelined call (events on the compute and copy streams)
from paper_2412_08902_b200.executors import get_plan, stage_operand, _alloc_z
executors.HOST_PIPELINE_PARTS = 8
plan = get_plan(ws, asg, "bf16")
cur = torch.cuda.current_stream()
cs = torch.cuda.Stream()
host = torch.empty((a.num_rows, 128), dtype=torch.float32, pin_memory=True)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(cur)
    xop, _ = stage_operand(xh, "bf16", dev)
    e[1].record(cur)
    z, ldz = _alloc_z(a.num_rows, 128, dev)
    th = time.perf_counter()
    for part in plan.parts(8):
        plan.run(xop, z, ldz, part=part)
        r0, r1 = min(part[0] * 16, a.num_rows), min(part[1] * 16, a.num_rows)
        ev = torch.cuda.Event(); ev.record(cur); cs.wait_event(ev)
        with torch.cuda.stream(cs):
            host[r0:r1].copy_(z[r0:r1, :128], non_blocking=True)
    e[2].record(cur)
    e[3].record(cs)
    tl = time.perf_counter()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(json.dumps({"h2d_ms": e[0].elapsed_time(e[1]), "compute_done_ms": e[0].elapsed_time(e[2]),
                      "d2h_done_ms": e[0].elapsed_time(e[3]), "host_stage_ms": (th - t0) * 1e3,
                      "host_launch_ms": (tl - th) * 1e3, "wall_ms": (t1 - t0) * 1e3}), flush=True)

# compute-only time of the part launches (device-resident X and Z, no copies)
xop, _ = stage_operand(xh, "bf16", dev)
z, ldz = _alloc_z(a.num_rows, 128, dev)
for k in (1, 2, 4, 8, 16):
    parts = plan.parts(k)
    for _ in range(3):
        for p in parts:
            plan.run(xop, z, ldz, part=p)
    s, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(10):
        for p in parts:
            plan.run(xop, z, ldz, part=p)
    e2.record(); torch.cuda.synchronize()
    print(json.dumps({"parts": k, "compute_only_ms": s.elapsed_time(e2) / 10}), flush=True)
