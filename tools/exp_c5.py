"""Experiment (not product): C5 (R-MAT scale 24) hybrid SpMM split into its tile and scalar
launches (CUDA events), with the scalar windows' nnz / row statistics."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import graphgen, _lib
from paper_2412_08902_b200.gnn import normalize_adj
from paper_2412_08902_b200.executors import DeviceOperand, get_plan

scale = int(os.environ.get("C5_SCALE", "24"))
dim = int(os.environ.get("C5_DIM", "128"))
torch.cuda.set_device(0)
if os.environ.get("C5_PAIRING"):
    from paper_2412_08902_b200 import _lib as _l
    _l.call("hcs_set_tile_pairing", int(os.environ["C5_PAIRING"]))
if os.environ.get("C5_TILE_SLICE"):
    from paper_2412_08902_b200 import _lib as _l
    _l.call("hcs_set_tile_slice", int(os.environ["C5_TILE_SLICE"]))
if os.environ.get("C5_SCALAR_VARIANT"):
    from paper_2412_08902_b200.executors import set_scalar_variant
    set_scalar_variant(os.environ["C5_SCALAR_VARIANT"])
adj = graphgen.rmat(scale, 33, seed=0); adj.symmetric = True
a = normalize_adj(adj, "gcn")
del adj
ws = hc.partition(a)
asg = hc.classify_windows(hc.default_model(), ws)
plan = get_plan(ws, asg, "bf16")
nnz_w = ws.nnz_per_window()
sl = plan.scalar_list.long()
snnz = int(nnz_w[sl].sum().item())
print(json.dumps({"n": a.num_rows, "nnz": a.nnz, "windows": len(ws), "tile": plan.n_tile,
                  "scalar_or_empty": int(sl.numel()), "scalar_nnz": snnz,
                  "empty": int((nnz_w == 0).sum().item())}), flush=True)
wn = nnz_w[sl]
rp = a.row_ptr
rl = (rp[1:] - rp[:-1])
wh = ws.window_height
rows_s = (sl[:, None] * wh + torch.arange(wh, device=sl.device)[None, :]).flatten()
rows_s = rows_s[rows_s < a.num_rows]
rls = rl[rows_s]
print(json.dumps({"scalar_win_nnz_max": int(wn.max()), "win_gt256": int((wn > 256).sum()), "win_gt4096": int((wn > 4096).sum()),
                  "nnz_in_gt256": int(wn[wn > 256].sum()), "row_nnz_max": int(rls.max()), "rows_gt1000": int((rls > 1000).sum()),
                  "rows_gt10000": int((rls > 10000).sum())}), flush=True)
ept = (plan.ent_ptr[1:] - plan.ent_ptr[:-1]).float()
print(json.dumps({"chunks": plan.nchunks, "ent_per_chunk": float(ept.mean()), "chunks_gt128": int((ept > 128).sum()),
                  "ent_in_gt128": int(ept[ept > 128].sum()), "ent_max": int(ept.max())}), flush=True)
if os.environ.get("C5_STATS_ONLY"):
    sys.exit(0)
x = graphgen.dense_features(a.num_rows, dim, seed=1)
xop = DeviceOperand(x, dim, dim, _lib.DTYPE_BF16)
z = torch.empty((a.num_rows, dim), dtype=torch.float32, device="cuda")
W = len(ws)
nt, ns = plan.n_tile, int(sl.numel())
parts = {"tile": (0, W, 0, nt, 0, 0), "scalar": (0, W, 0, 0, 0, ns), "all": None}
res = {}
for name, part in parts.items():
    for _ in range(2):
        plan.run(xop, z, dim, part=part)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(5):
        plan.run(xop, z, dim, part=part)
    e.record(); torch.cuda.synchronize()
    res[name] = s.elapsed_time(e) / 5
    print(name, f"{res[name]:.3f} ms", flush=True)
res["scalar_gather_GBps"] = snnz * dim * 2 / (res["scalar"] * 1e-3) / 1e9
print(json.dumps(res))
