"""Debug: async (3 in flight) vs sync hybrid products, bisecting the fork and the piece kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen_graphs as gg  # noqa: E402
import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200 import executors as ex  # noqa: E402
from oracle import rowwin_oracle as orc  # noqa: E402

n, rr, cc = gg.power_law(3000, 24.0, seed=5)
adj = orc.from_coo(n, n, rr, cc, np.ones(len(rr)))
a = orc.normalize_adj(adj, "gcn")
codes = None
xs = [orc.random_dense(n, d, seed=10 + i) for i, d in enumerate((64, 128, 40))]
ins = [hc.DenseMatrix(xs[0]), torch.from_numpy(xs[1]).to(torch.bfloat16).pin_memory(), torch.from_numpy(xs[2]).float()]
for fork_max, pieces_max in ((8192, 1024),) * 1 + ((0, 1024), (8192, 0)):
    ex.CONCURRENT_MAX_WINDOWS, ex.SCALAR_PIECES_MAX_WINDOWS = fork_max, pieces_max
    for trial in range(int(os.environ.get('TRIALS', '30'))):
        ws = hc.partition(hc.SparseCsr(n, n, a.row_ptr, a.col_idx, a.values))
        asg = hc.classify_windows(hc.default_model(), ws)
        rows_tile = np.repeat(asg.codes, 16)[:n] == 1
        reqs = [hc.spmm_hybrid_async(ws, asg, x) for x in ins]
        got = [r.result() for r in reqs]
        out = []
        for i, (x, g) in enumerate(zip(ins, got)):
            want = hc.spmm_hybrid(ws, asg, x).z.data
            gz = np.asarray(g.z.data)
            wz = np.asarray(want)
            diff = np.abs(gz - wz).max(1)
            bad = np.nonzero(diff)[0]
            out.append((i, bad.size, int(rows_tile[bad].sum()), float(diff.max())))
        if any(o[1] for o in out) or trial == 0:
            print("fork", fork_max, "pieces", pieces_max, "trial", trial, out, flush=True)
