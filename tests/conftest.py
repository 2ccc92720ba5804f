"""Shared test fixtures: golden vectors (tests/golden, generated from the reference by
tests/golden/make_golden.py), the CPU oracle (oracle/), and the `gpu` marker."""

from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, GOLDEN)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def golden_names(prefix: str) -> list[str]:
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_csr(g: dict, prefix: str = ""):
    from oracle.rowwin_oracle import Csr

    return Csr(int(g[prefix + "n_rows"]), int(g[prefix + "n_cols"]), g[prefix + "row_ptr"].astype(np.int64),
               g[prefix + "col_idx"].astype(np.int64), g[prefix + "values"].astype(np.float64))


def plaw8k_csr():
    """Regenerate the windows_plaw8k graph (generator params stored in the fixture)."""
    import gen_graphs as gg
    from oracle import rowwin_oracle as orc

    n, r, c = gg.power_law(8192, 40.0, seed=7)
    adj = orc.from_coo(n, n, r, c, np.ones(len(r)))
    return orc.normalize_adj(adj, "gcn")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device: the product has no CPU fallback")
    return True
