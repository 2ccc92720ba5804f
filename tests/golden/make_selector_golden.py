"""Golden fixture for the selector-training restatement (paper_2412_08902_b200/selector_train.py):
runs the REFERENCE's generate_synthetic / default_grid / analytic_samples / train / holdout_split
(/root/reference/pkg/src/rowwin/selector.py:67-242) in this container and stores inputs + outputs.
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_selector_golden.py
"""
import os
import numpy as np
from rowwin import selector as S
from rowwin.costmodel import default_cost_params

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "selector_train.npz")
grid = S.default_grid()
syn = {}
for ncols, nnz, seed in grid[::37]:
    w = S.generate_synthetic(ncols, nnz, seed)
    syn[f"syn_{ncols}_{nnz}_{seed}_ptr"] = w.local_ptr
    syn[f"syn_{ncols}_{nnz}_{seed}_cols"] = w.cond_cols
samples = S.analytic_samples(default_cost_params(), [1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 256, 512, 1024],
                             S._density_levels(), dim=32)
tr, ho = S.holdout_split(samples, frac=0.25, seed=0)
m = S.train(tr, seed=0)
np.savez_compressed(
    OUT,
    grid=np.array(grid, dtype=np.int64),
    s_ncols=np.array([s.ncols for s in samples], dtype=np.int64),
    s_density=np.array([s.density for s in samples]),
    s_ts=np.array([s.t_scalar for s in samples]),
    s_tt=np.array([s.t_tile for s in samples]),
    s_label=np.array([s.label for s in samples], dtype=np.int64),
    train_idx=np.array([samples.index(s) for s in tr], dtype=np.int64),
    model=np.array([m.w_ncols, m.w_density, m.bias, *m.feature_means, *m.feature_scales]),
    acc=np.array([S.accuracy(m, tr), S.accuracy(m, ho)]),
    **syn,
)
print("wrote", OUT, len(samples), "samples", m)
