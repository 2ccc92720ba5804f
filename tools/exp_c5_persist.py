"""Experiment (not product): C5 (R-MAT scale 24) tile launch with its hottest X rows copied into a
compact block at the end of X (plan gidx remapped), optionally pinned in L2 by a persisting
access-policy window on the launch stream.  Load an experimental library with HCS_LIB_PATH
(e.g. tools/exp_libs/xpol_none: X gathers without an L2 cache hint, so the window's policy
applies).  Prints one JSON line per variant; Z is compared bitwise with the shipping layout."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan
from cuda.bindings import runtime as rt

scale = int(os.environ.get("C5_SCALE", "24"))
dim = int(os.environ.get("C5_DIM", "128"))
budgets = [int(b) for b in os.environ.get("C5_BUDGETS_MB", "0,32,64,96").split(",")]
torch.cuda.set_device(0)
dev = torch.device("cuda")
err, maxp = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
err2, l2 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0)
err3, maxwin = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
print(json.dumps({"lib": _lib.LIB_PATH, "l2": l2, "max_persisting_l2": maxp, "max_window": maxwin}), flush=True)

adj = graphgen.rmat(scale, 33, seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
del adj
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
n = a.num_rows
x = graphgen.dense_features(n, dim, seed=1)
W = len(ws)
part = (0, W, 0, plan.n_tile, 0, 0)
g0 = plan.gidx
valid = g0 >= 0
counts = torch.bincount(g0[valid].long(), minlength=n)
order = torch.argsort(counts, descending=True)
csum = torch.cumsum(counts[order].double(), 0)
tot = float(csum[-1])
print(json.dumps({"n": n, "tile": plan.n_tile, "gathers": int(tot), "distinct": int((counts > 0).sum()),
                  "share_top": {mb: float(csum[min(n, mb * 2**20 // (2 * dim)) - 1] / tot) for mb in (16, 32, 64, 96, 128)}}),
      flush=True)
stream = torch.cuda.Stream()


def set_window(ptr, nbytes, persist_mb):
    rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, persist_mb * 2**20)
    v = rt.cudaStreamAttrValue()
    v.accessPolicyWindow.base_ptr = ptr
    v.accessPolicyWindow.num_bytes = nbytes
    v.accessPolicyWindow.hitRatio = 1.0 if nbytes else 0.0
    v.accessPolicyWindow.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    v.accessPolicyWindow.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    r = rt.cudaStreamSetAttribute(stream.cuda_stream, rt.cudaStreamAttrID(rt.cudaStreamAttributeAccessPolicyWindow), v)
    rt.cudaCtxResetPersistingL2Cache()
    return int(r[0]) if isinstance(r, tuple) else int(r)


def run(xbig, gidx, reps=5):
    plan.gidx = gidx
    xop = DeviceOperand(xbig, dim, dim, _lib.DTYPE_BF16)
    z = torch.empty((n, dim), dtype=torch.float32, device=dev)
    with torch.cuda.stream(stream):
        for _ in range(2):
            plan.run(xop, z, dim, part=part)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            s.record(); plan.run(xop, z, dim, part=part); e.record(); e.synchronize()
            ts.append(s.elapsed_time(e))
    plan.gidx = g0
    return z, sorted(ts)[len(ts) // 2], ts


z_ref, t_ref, _ = run(x, g0)
print(json.dumps({"variant": "shipping", "tile_ms": t_ref}), flush=True)
for mb in budgets:
    if mb == 0:
        continue
    K = mb * 2**20 // (2 * dim)
    hot = order[:K]
    xb = torch.empty((n + K, dim), dtype=x.dtype, device=dev)
    xb[:n] = x
    xb[n:] = x[hot]
    remap = torch.arange(n, dtype=torch.int32, device=dev)
    remap[hot] = n + torch.arange(K, dtype=torch.int32, device=dev)
    g1 = torch.where(valid, remap[g0.clamp(min=0).long()], g0)
    share = float(csum[K - 1] / tot)
    z1, t1, _ = run(xb, g1)
    print(json.dumps({"variant": "compact", "mb": mb, "hot_share": share, "tile_ms": t1,
                      "bitwise": bool(torch.equal(z1, z_ref))}), flush=True)
    for pmb in sorted({mb, min(mb + 16, maxp // 2**20), maxp // 2**20}):
        rc = set_window(xb.data_ptr() + n * dim * 2, K * dim * 2, pmb)
        z2, t2, ts = run(xb, g1)
        print(json.dumps({"variant": "compact+persist", "mb": mb, "persist_mb": pmb, "rc": rc, "tile_ms": t2,
                          "all": ts, "bitwise": bool(torch.equal(z2, z_ref))}), flush=True)
        set_window(0, 0, 0)
    del xb, g1, z1
