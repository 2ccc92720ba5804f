"""Debug: the K3 rows kernel on tiny inputs, one launch at a time (run under `timeout`)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200.executors import Assignment, Path, set_scalar_variant  # noqa: E402
from oracle import rowwin_oracle as orc  # noqa: E402

set_scalar_variant("rows")
rng = np.random.default_rng(0)
for n, deg in ((16, 3), (40, 5), (300, 60)):
    rows, cols = [], []
    for r in range(n):
        k = int(rng.integers(0, deg))
        cs = rng.choice(n, size=min(k, n), replace=False)
        rows += [r] * len(cs)
        cols += list(cs)
    a = orc.from_coo(n, n, rows, cols, rng.uniform(-1, 1, len(rows)))
    ws = hc.partition(hc.SparseCsr(n, n, a.row_ptr, a.col_idx, a.values))
    asg = Assignment.uniform(len(ws), Path.SCALAR)
    for dim in (8, 32, 128):
        x = orc.random_dense(n, dim, seed=1)
        print("launch", n, deg, dim, flush=True)
        r = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x), precision="bf16")
        torch.cuda.synchronize()
        print("  err", orc.max_rel_err(r.z.data, orc.spmm_exact(a, x)), flush=True)
