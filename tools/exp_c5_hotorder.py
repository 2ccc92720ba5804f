"""Experiment (not product): C5 (R-MAT scale 24) tile launch with each window's condensed columns
re-ordered by how many windows share the column (hot first / cold first), so a 64-column chunk
holds rows of similar L2 hit likelihood -- a chunk waits for its slowest row, and today nearly
every chunk holds at least one L2 miss.  Optional: the hottest rows compacted into a block at
the end of X and pinned by a persisting access-policy window (C5_PERSIST_MB).  Z is compared
with the shipping order (summation order differs: max relative difference reported)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.windows import WindowSet
from paper_2412_08902_b200.executors import DeviceOperand, get_plan, HybridPlan

scale = int(os.environ.get("C5_SCALE", "24"))
dim = int(os.environ.get("C5_DIM", "128"))
persist_mb = [int(v) for v in os.environ.get("C5_PERSIST_MB", "0,64").split(",")]
torch.cuda.set_device(0)
dev = torch.device("cuda")
adj = graphgen.rmat(scale, 33, seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
del adj
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
codes = asg.device_codes(dev)
n, W, wh = a.num_rows, len(ws), ws.window_height
x = graphgen.dense_features(n, dim, seed=1)
stream = torch.cuda.Stream()


def reorder(sign):
    """WindowSet whose nonzero_cols are sorted per window by sign * (windows sharing the column)."""
    nzc = ws.nonzero_cols.long()
    cnt = torch.bincount(nzc, minlength=n)
    L = nzc.numel()
    wcp = ws.win_col_ptr
    wid = torch.repeat_interleave(torch.arange(W, device=dev), wcp[1:] - wcp[:-1])
    c = cnt[nzc]
    c = (c.max() - c) if sign > 0 else c
    key = (wid << 42) | (c << 24) | nzc
    del wid, c
    idx = torch.argsort(key)
    del key
    new_nzc = nzc[idx].to(torch.int32)
    inv = torch.empty(L, dtype=torch.int64, device=dev)
    inv[idx] = torch.arange(L, device=dev)
    del idx
    rp = a.row_ptr
    rows = torch.repeat_interleave(torch.arange(n, device=dev), rp[1:] - rp[:-1])
    ws0 = wcp[rows // wh]
    del rows
    new_cc = (inv[ws0 + ws.cond_cols.long()] - ws0).to(ws.cond_cols.dtype)
    del inv, ws0
    return WindowSet(a, wh, wcp, new_nzc, new_cc, ws.density, ws.ci, ws.codes, ws.selector)


def set_window(ptr, nbytes, pmb):
    from cuda.bindings import runtime as rt
    rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, pmb * 2**20)
    v = rt.cudaStreamAttrValue()
    v.accessPolicyWindow.base_ptr = ptr
    v.accessPolicyWindow.num_bytes = nbytes
    v.accessPolicyWindow.hitRatio = 1.0 if nbytes else 0.0
    v.accessPolicyWindow.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    v.accessPolicyWindow.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    rt.cudaStreamSetAttribute(stream.cuda_stream, rt.cudaStreamAttrID(rt.cudaStreamAttributeAccessPolicyWindow), v)
    rt.cudaCtxResetPersistingL2Cache()


def run(p, xt, reps=5):
    xop = DeviceOperand(xt, dim, dim, _lib.DTYPE_BF16)
    z = torch.zeros((n, dim), dtype=torch.float32, device=dev)
    part = (0, W, 0, p.n_tile, 0, 0)
    with torch.cuda.stream(stream):
        for _ in range(2):
            p.run(xop, z, dim, part=part)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            s.record(); p.run(xop, z, dim, part=part); e.record(); e.synchronize()
            ts.append(s.elapsed_time(e))
    torch.cuda.synchronize()
    return z, sorted(ts)[len(ts) // 2], ts


z_ref, t_ref, ts = run(plan, x)
print(json.dumps({"variant": "shipping", "tile_ms": t_ref, "all": ts}), flush=True)
for sign, name in ((1, "hot_first"), (-1, "cold_first")):
    ws2 = reorder(sign)
    _lib.call("hcs_set_tile_plan_builder", 1)  # global radix sort: no per-row monotonic chunk assumption
    p2 = HybridPlan(ws2, codes, "bf16")
    _lib.call("hcs_set_tile_plan_builder", 0)
    z2, t2, ts = run(p2, x)
    rel = float(((z2 - z_ref).abs().max() / z_ref.abs().max()).item())
    print(json.dumps({"variant": name, "tile_ms": t2, "all": ts, "max_rel_vs_shipping": rel}), flush=True)
    if sign > 0:
        g0 = p2.gidx
        valid = g0 >= 0
        cnt = torch.bincount(g0[valid].long(), minlength=n)
        order = torch.argsort(cnt, descending=True)
        for pmb in persist_mb:
            if pmb == 0:
                continue
            K = pmb * 2**20 // (2 * dim)
            hot = order[:K]
            xb = torch.empty((n + K, dim), dtype=x.dtype, device=dev)
            xb[:n] = x
            xb[n:] = x[hot]
            remap = torch.arange(n, dtype=torch.int32, device=dev)
            remap[hot] = n + torch.arange(K, dtype=torch.int32, device=dev)
            p2.gidx = torch.where(valid, remap[g0.clamp(min=0).long()], g0)
            set_window(xb.data_ptr() + n * dim * 2, K * dim * 2, min(pmb, 79))
            z3, t3, ts = run(p2, xb)
            set_window(0, 0, 0)
            print(json.dumps({"variant": name + "+persist", "mb": pmb, "tile_ms": t3, "all": ts,
                              "bitwise_vs_hot_first": bool(torch.equal(z3, z2))}), flush=True)
            p2.gidx = g0
            del xb
    del ws2, p2, z2
