"""compute-sanitizer workload (memcheck / racecheck / synccheck / initcheck): every product kernel
once on small inputs -- C1 (Cora-shaped) and the 8,192-node power-law graph (mixed TILE/SCALAR
windows): K1 partition + selector, K2 tile plan, K4 tile (bf16 + tf32), K3 scalar, the fused GCN
epilogues (bf16 + tf32, tile + scalar), grad_W, the dense update, normalisation, LOA + permute, and
the cost-weighted tile ranges (k_tile_bounds + the WB kernel) on a hub-window plan with a 4-CTA grid.
Run: compute-sanitizer --tool memcheck python tools/sanitize.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200 import gnn, graphgen, layout  # noqa: E402
from paper_2412_08902_b200.executors import Assignment, Path  # noqa: E402
from paper_2412_08902_b200.fused import dense_matmul, grad_weight  # noqa: E402
from paper_2412_08902_b200.matrices import Graph  # noqa: E402


def run(a, name):
    ws = hc.partition(a)
    for asg in (hc.classify_windows(hc.default_model(), ws), Assignment.uniform(len(ws), Path.TILE),
                Assignment.uniform(len(ws), Path.SCALAR)):
        for prec in ("bf16", "tf32"):
            for dim in (32, 64, 128, 41):
                x = torch.rand(a.num_rows, dim, device="cuda") * 2 - 1
                hc.spmm_hybrid(ws, asg, x, precision=prec)
            layer = gnn.GnnLayer.random(128, 64, seed=0)
            x = torch.rand(a.num_rows, 128, device="cuda") * 2 - 1
            xn, z, _ = gnn.forward(layer, a, x, mode="fused", assignment=asg, windows=ws, precision=prec)
            gnn.backward(layer, a, z, xn, mode="fused", assignment=asg, precision=prec)
    g = torch.rand(a.num_rows, 41, device="cuda")
    grad_weight(torch.rand(a.num_rows, 64, device="cuda"), g)
    dense_matmul(torch.rand(a.num_rows, 64, device="cuda"), torch.rand(64, 41, device="cuda"))
    torch.cuda.synchronize()
    print(name, "ok", flush=True)


def skewed():
    """Hub windows (chunks of up to 1,024 entries) -> HybridPlan.tile_alpha > 0; a 4-CTA tile grid
    makes the weighted split apply to a small plan (>= 8 tile windows per warp group)."""
    from oracle import rowwin_oracle as orc
    from paper_2412_08902_b200 import _lib
    from paper_2412_08902_b200.executors import get_plan

    rng = np.random.default_rng(5)
    n, m = 16 * 400, 4000
    hub = rng.choice(m, size=200, replace=False)
    rows, cols = [], []
    for r in range(n):
        c = hub if (r // 16) % 25 == 0 else rng.choice(m, size=int(rng.integers(4, 30)), replace=False)
        rows += [r] * len(c)
        cols += list(c)
    a = orc.from_coo(n, m, rows, cols, rng.uniform(-1, 1, len(rows)))
    ws = hc.partition(hc.SparseCsr(n, m, a.row_ptr, a.col_idx, a.values))
    asg = Assignment.uniform(len(ws), Path.TILE)
    assert get_plan(ws, asg, "bf16").tile_alpha > 0
    _lib.call("hcs_set_tile_grid", 4)
    try:
        for dim in (128, 64):
            hc.spmm_hybrid(ws, asg, torch.rand(m, dim, device="cuda") * 2 - 1)
    finally:
        _lib.call("hcs_set_tile_grid", 0)
    torch.cuda.synchronize()
    print("skewed ok", flush=True)


def main():
    torch.cuda.set_device(0)
    skewed()
    adj = graphgen.cora_shaped(seed=0)
    adj.symmetric = True
    run(gnn.normalize_adj(adj, "gcn"), "c1")
    import gen_graphs as gg
    from oracle import rowwin_oracle as orc

    n, r, c = gg.power_law(8192, 40.0, seed=7)
    raw = orc.from_coo(n, n, r, c, np.ones(len(r)))
    g = Graph(n, hc.SparseCsr(n, n, raw.row_ptr, raw.col_idx, raw.values), True)
    run(gnn.normalize_adj(g, "gcn"), "plaw8k")
    grouping = layout.build_windows_optimized(g, vw=128)
    layout.reorder(g, grouping)
    torch.cuda.synchronize()
    print("loa ok", flush=True)


if __name__ == "__main__":
    main()
