"""CPU: the C-ABI library loads and exports every symbol include/hcspmm.h declares;
host-side API logic (errors, selector KATs, Assignment/ExecStats) without a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2412_08902_b200 as hc
from paper_2412_08902_b200 import _lib
from paper_2412_08902_b200.executors import Assignment, ExecStats, Path


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hcspmm.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|size_t)\s+(hcs_[a-z0-9_]+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    h = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 10
    missing = [s for s in syms if not hasattr(h, s)]
    assert not missing, missing
    # every declared symbol is also bound by the Python layer
    assert not [s for s in syms if s not in _lib._SIGS]


def test_library_version_and_error_string():
    L = _lib.lib()
    assert L.hcs_version() >= 100
    assert isinstance(L.hcs_last_error(), bytes)


def test_abi_argument_validation_without_gpu():
    L = _lib.lib()
    # invalid window height is rejected before any device work
    rc = L.hcs_partition_count(None, None, 10, 10, 0, 0, None, None, None, None, None, None, 0, None)
    assert rc == _lib.HCS_EINVAL
    assert b"window_height" in L.hcs_last_error()
    with pytest.raises(ValueError, match="window_height"):
        _lib.check(rc)


def test_precision_rejected():
    with pytest.raises(ValueError, match="precision"):
        hc.spmm_scalar(hc.SparseCsr(2, 2, np.array([0, 1, 1]), np.array([0]), np.array([1.0])),
                       hc.DenseMatrix(np.ones((2, 2))), precision="f64")


def test_dimension_mismatch_message():
    csr = hc.SparseCsr(2, 3, np.array([0, 1, 1]), np.array([0]), np.array([1.0]))
    with pytest.raises(ValueError, match="mismatch"):
        hc.spmm_scalar(csr, hc.DenseMatrix(np.ones((2, 2))))


def test_partition_rejects_bad_height():
    with pytest.raises(ValueError, match="window_height"):
        hc.partition(hc.SparseCsr(1, 1, np.array([0, 0]), np.array([], dtype=np.int64), np.array([])),
                     window_height=0)


def test_selector_threshold_semantics():
    # reference tests/test_selector.py:160-174
    m = hc.SelectorModel(w_ncols=0.0, w_density=-1.0, bias=0.0, feature_means=(0.0, 0.5), feature_scales=(1.0, 1.0))
    assert m.decide(8, 0.4) is Path.SCALAR
    assert m.decide(8, 0.6) is Path.TILE
    assert m.decide(8, 0.5) is Path.TILE
    e = hc.SelectorModel(0.0, 0.0, -5.0, (0.0, 0.0), (1.0, 1.0))
    assert e.decide(0, 0.0) is Path.SCALAR


def test_default_model_constants():
    m = hc.default_model()
    assert (m.w_ncols, m.w_density, m.bias) == (-0.1454848214145233, -9.249873814861964, -15.105252482198011)
    assert m.feature_means == (140.38659793814432, 0.5)
    assert m.feature_scales == (123.08273985946481, 0.2570676399373035)


def test_default_model_monotone_in_density():
    # reference tests/test_selector.py:229-240
    m = hc.default_model()
    for nc in (16, 64, 128, 256):
        ds = [m.decide(nc, d) for d in np.linspace(0.01, 0.95, 60)]
        flips = sum(1 for a, b in zip(ds, ds[1:]) if a is not b)
        assert flips <= 1
        if flips:
            assert ds[0] is Path.SCALAR and ds[-1] is Path.TILE


def test_vectorised_host_decisions_match_scalar():
    from paper_2412_08902_b200.selector import decisions_host

    m = hc.default_model()
    rng = np.random.default_rng(0)
    nc = rng.integers(0, 3000, size=5000)
    d = rng.random(5000)
    want = [0 if n == 0 else (1 if m.decide(int(n), float(x)) is Path.TILE else 0) for n, x in zip(nc, d)]
    assert decisions_host(m, nc, d).tolist() == want


def test_assignment_semantics():
    a = Assignment(np.array([0, 1, 1, 0, 1], dtype=np.uint8))
    assert len(a) == 5 and a.count(Path.TILE) == 3 and a.count(Path.SCALAR) == 2
    assert a.path(0) is Path.SCALAR and a.path(1) is Path.TILE
    assert Assignment.from_paths([Path.SCALAR, Path.TILE]).codes.tolist() == [0, 1]
    with pytest.raises(ValueError):
        Assignment(np.array([0, 2], dtype=np.uint8))


def test_exec_stats_merge():
    s = ExecStats(1, 2, 3, 4, 5)
    s.merge(ExecStats(1, 1, 1, 1, 1))
    assert s.as_dict() == {"windows_scalar": 2, "windows_tile": 3, "entries_scalar": 4, "entries_tile": 5,
                           "tiles_processed": 6}


def test_sparse_csr_validate_and_from_coo():
    csr = hc.SparseCsr.from_coo(3, 3, np.array([0, 0, 2, 0]), np.array([1, 1, 0, 2]), np.array([2.0, 3.0, 1.0, 4.0]))
    assert csr.row_ptr.tolist() == [0, 2, 2, 3]
    assert csr.col_idx.tolist() == [1, 2, 0] and csr.values.tolist() == [5.0, 4.0, 1.0]
    csr.validate()
    bad = hc.SparseCsr(2, 3, np.array([0, 2, 2]), np.array([2, 1]), np.ones(2))
    with pytest.raises(ValueError, match="strictly ascending"):
        bad.validate()


def test_host_convert_f64_matches_torch_casts():
    """hcs_host_convert_f64 (the drop-in DenseMatrix staging, csrc/host_stage.cu) == torch's
    double -> bfloat16 cast bit for bit (infinities, overflow, subnormals, RNE ties, signed
    zeros; NaN stays NaN), == astype(float32) for fp32, and zeroes the padding columns; any
    thread count gives the same bytes."""
    import numpy as np
    import torch

    from paper_2412_08902_b200 import _lib

    rng = np.random.default_rng(0)
    a = rng.standard_normal((777, 77)) * np.exp(rng.uniform(-60, 60, (777, 77)))
    a[0, :6] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1e39]
    a[1, :4] = [1e-40, -1e-42, 3.4e38, -1e300]
    a[2, :3] = [1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8)]  # exact bf16 ties
    ref = torch.from_numpy(a).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    for ld, threads in ((77, 1), (80, 3), (96, 0)):
        out = np.full((777, ld), 0xAAAA, dtype=np.uint16)
        _lib.call("hcs_host_convert_f64", a.ctypes.data, 777, 77, 77, out.ctypes.data, ld, _lib.DTYPE_BF16, threads)
        nan = np.isnan(a)
        assert np.array_equal(out[:, :77][~nan], ref[~nan])
        assert ((out[:, :77][nan] & 0x7F80) == 0x7F80).all() and (out[:, :77][nan] & 0x7F).all()
        assert (out[:, 77:] == 0).all()
        o32 = np.full((777, ld), 7.0, dtype=np.float32)
        _lib.call("hcs_host_convert_f64", a.ctypes.data, 777, 77, 77, o32.ctypes.data, ld, _lib.DTYPE_F32, threads)
        with np.errstate(over="ignore"):
            assert np.array_equal(o32[:, :77], a.astype(np.float32), equal_nan=True)
        assert (o32[:, 77:] == 0).all()
    with pytest.raises(ValueError, match="leading dimensions"):
        _lib.call("hcs_host_convert_f64", a.ctypes.data, 777, 77, 70, out.ctypes.data, 96, _lib.DTYPE_BF16, 1)


def test_scalar_piece_list_host_logic():
    """executors.build_scalar_pieces (the small-plan K3's work list, host side, CPU tensors): every
    row of the listed windows is covered by consecutive pieces of <= 32 entries in entry order,
    empty rows get one empty piece, p_first/p_count name each row's piece range, window -> piece
    pointers are prefix sums, and rows past n_rows (a short last window) are skipped."""
    import torch

    from paper_2412_08902_b200.executors import build_scalar_pieces

    rng = np.random.default_rng(3)
    n, wh = 53, 7
    lens = rng.integers(0, 90, n)
    lens[[4, 11]] = 0
    lens[20] = 64  # exactly two pieces
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])

    class _Csr:  # the attributes build_scalar_pieces reads
        row_ptr = torch.from_numpy(rp)
        num_rows = n
        device = torch.device("cpu")

    W = -(-n // wh)
    wl = torch.tensor([1, 3, W - 1, 0], dtype=torch.int32)  # any order; the last window is short
    p_row, p_k, p_first, p_count, win_piece = build_scalar_pieces(_Csr, wl, wh)
    p_row, p_k, p_first, p_count = p_row.numpy(), p_k.numpy(), p_first.numpy(), p_count.numpy()
    assert (p_k[:, 1] - p_k[:, 0] <= 32).all() and (p_k[:, 1] >= p_k[:, 0]).all()
    q = 0
    for wi, w in enumerate(wl.tolist()):
        assert win_piece[wi] == q
        for r in range(w * wh, min(w * wh + wh, n)):
            k0, k1 = rp[r], rp[r + 1]
            cnt = max(1, -(-(k1 - k0) // 32))
            assert (p_row[q:q + cnt] == r).all()
            assert (p_first[q:q + cnt] == q).all() and (p_count[q:q + cnt] == cnt).all()
            assert p_k[q, 0] == k0 and p_k[q + cnt - 1, 1] == k1
            assert (p_k[q + 1:q + cnt, 0] == p_k[q:q + cnt - 1, 1]).all()  # consecutive
            q += cnt
    assert win_piece[len(wl)] == q == p_row.size
