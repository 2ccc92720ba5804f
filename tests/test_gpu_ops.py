"""torch.ops.hcspmm custom operators (the north_star's "PyTorch custom op over a thin C-ABI"):
forward == the package entry points bit for bit, autograd against exact fp64 products within
the bf16 tolerance (north_star 1e-2), and torch.library.opcheck's schema / fake-tensor /
autograd-registration checks."""

import numpy as np
import pytest
import torch

from oracle import rowwin_oracle as orc

import paper_2412_08902_b200 as hc
from conftest import plaw8k_csr

pytestmark = pytest.mark.gpu
BF16_TOL = 1e-2


def to_hc(csr):
    return hc.SparseCsr(csr.num_rows, csr.num_cols, csr.row_ptr, csr.col_idx, csr.values)


def _tensors(a):
    d = hc.to_device_csr(to_hc(a))
    return d, (d.row_ptr, d.col_idx, d.values, a.num_cols)


def _dense_t(a):
    m = np.zeros((a.num_rows, a.num_cols))
    for r in range(a.num_rows):
        lo, hi = a.row_ptr[r], a.row_ptr[r + 1]
        m[r, a.col_idx[lo:hi]] += a.values[lo:hi]
    return m


def test_spmm_op_matches_entry_point(cuda_ok):
    a = plaw8k_csr()
    d, csr = _tensors(a)
    x = torch.from_numpy(orc.random_dense(a.num_cols, 64, seed=3)).float().cuda()
    z = torch.ops.hcspmm.spmm(*csr, x, "bf16")
    ws = hc.partition(d)
    want = hc.spmm_hybrid(ws, hc.classify_windows(hc.default_model(), ws), x).z.data
    assert torch.equal(z, want)
    assert torch.equal(torch.ops.hcspmm.spmm(*csr, x, "bf16"), z)  # cached operator, deterministic


def test_spmm_op_autograd(cuda_ok):
    rng = np.random.default_rng(1)
    n_r, n_c = 3000, 2500  # rectangular, so A^T is really used
    rows = rng.integers(0, n_r, 60000)
    cols = rng.integers(0, n_c, 60000)
    a = orc.from_coo(n_r, n_c, rows, cols, rng.uniform(-1, 1, rows.size))
    _, csr = _tensors(a)
    x = torch.from_numpy(orc.random_dense(n_c, 32, seed=4)).float().cuda().requires_grad_()
    z = torch.ops.hcspmm.spmm(*csr, x, "bf16")
    r = torch.from_numpy(orc.random_dense(n_r, 32, seed=5)).float().cuda()
    (z * r).sum().backward()
    m = _dense_t(a)
    want = m.T @ r.double().cpu().numpy()
    got = x.grad.double().cpu().numpy()
    assert np.abs(got - want).max() / np.abs(want).max() <= BF16_TOL
    assert np.abs(z.detach().double().cpu().numpy() - m @ x.detach().double().cpu().numpy()).max() / \
        np.abs(m @ x.detach().double().cpu().numpy()).max() <= BF16_TOL


def test_gcn_layer_op_autograd(cuda_ok):
    a = orc.normalize_adj(orc.from_coo(*_small_graph()), "gcn")
    _, csr = _tensors(a)
    x = torch.from_numpy(orc.random_dense(a.num_cols, 48, seed=6)).float().cuda().requires_grad_()
    w = (torch.from_numpy(orc.random_dense(48, 16, seed=7)).float() * 0.3).cuda().requires_grad_()
    out, z = torch.ops.hcspmm.gcn_layer(*csr, x, w, "bf16")
    g = torch.from_numpy(orc.random_dense(a.num_rows, 16, seed=8)).float().cuda()
    (out * g).sum().backward()
    m = _dense_t(a)
    xd, wd, gd = (t.detach().double().cpu().numpy() for t in (x, w, g))
    zd = m @ xd
    for got, want in ((z, zd), (out, zd @ wd), (x.grad, m.T @ (gd @ wd.T)), (w.grad, zd.T @ gd)):
        got = got.detach().double().cpu().numpy()
        assert np.abs(got - want).max() / np.abs(want).max() <= BF16_TOL


def _small_graph():
    rng = np.random.default_rng(2)
    n = 4000
    u = rng.integers(0, n, 40000)
    v = rng.integers(0, n, 40000)
    keep = u != v
    u, v = u[keep], v[keep]
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    return n, n, rows, cols, np.ones(rows.size)


def test_opcheck(cuda_ok):
    a = plaw8k_csr()
    _, csr = _tensors(a)
    x = torch.from_numpy(orc.random_dense(a.num_cols, 32, seed=9)).float().cuda().requires_grad_()
    w = torch.from_numpy(orc.random_dense(32, 8, seed=10)).float().cuda().requires_grad_()
    tests = ("test_schema", "test_faketensor", "test_autograd_registration")
    torch.library.opcheck(torch.ops.hcspmm.spmm.default, (*csr, x, "bf16"), test_utils=tests)
    torch.library.opcheck(torch.ops.hcspmm.gcn_layer.default, (*csr, x, w, "bf16"), test_utils=tests)


def test_operator_cache_follows_in_place_writes(cuda_ok):
    """Windows/plans are cached per operator; an in-place write to the values (version
    counter) gives a fresh operator: doubling every value doubles Z exactly."""
    a = plaw8k_csr()
    d, (rp, ci, v, nc) = _tensors(a)
    v = v.clone()
    x = torch.from_numpy(orc.random_dense(a.num_cols, 16, seed=11)).float().cuda()
    z1 = torch.ops.hcspmm.spmm(rp, ci, v, nc, x, "bf16")
    v.mul_(2)
    z2 = torch.ops.hcspmm.spmm(rp, ci, v, nc, x, "bf16")
    assert torch.equal(z2, 2 * z1)
