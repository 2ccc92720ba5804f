"""CPU: pin the oracle (oracle/rowwin_oracle.py, oracle/loa_oracle.c) against golden
vectors produced by the reference itself (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

from conftest import golden_csr, golden_names, load_golden, plaw8k_csr
from oracle import rowwin_oracle as orc


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", [n for n in golden_names("windows_") if n != "windows_plaw8k"])
def test_partition_features_selector_exact(name):
    g = load_golden(name)
    csr = golden_csr(g)
    w = orc.partition(csr)
    nc, dens, ci = orc.features(w)
    assert np.array_equal(nc, g["ncols"])
    assert np.array_equal(dens.view(np.uint64), g["density"].view(np.uint64))
    assert np.array_equal(ci.view(np.uint64), g["ci"].view(np.uint64))
    assert np.array_equal(orc.classify(nc, dens), g["codes"])
    assert np.array_equal(w.nonzero_cols, g["nonzero_cols"])
    assert np.array_equal(w.cond_cols, g["cond_cols"])
    assert sha(w.nonzero_cols.astype(np.int64)) == str(g["nonzero_cols_sha"])
    stats = orc.exec_stats(w, g["codes"])
    for k, v in stats.items():
        assert v == int(g["stats_" + k]), k


@pytest.mark.parametrize("name", [n for n in golden_names("windows_") if n != "windows_plaw8k"])
def test_spmm_restatement_matches_reference(name):
    g = load_golden(name)
    csr = golden_csr(g)
    w = orc.partition(csr)
    x = orc.random_dense(csr.num_cols, int(g["dim"]), int(g["xseed"]))
    z32 = orc.spmm_hybrid(w, g["codes"], x, "f32")
    assert orc.max_rel_err(z32, g["z_f32"]) <= 1e-6
    exact = orc.spmm_exact(csr, x)
    assert orc.max_rel_err(exact, g["z_f64"]) <= 1e-12
    # the multi-threaded C restatement used for the full-size (C2/C3) checks
    exact_c = orc.spmm_exact_c(csr.row_ptr, csr.col_idx, csr.values, x, nthreads=3)
    assert orc.max_rel_err(exact_c, g["z_f64"]) <= 1e-12
    assert orc.max_rel_err(orc.spmm_hybrid(w, g["codes"], x, "f64"), g["z_f64"]) <= 1e-13


def test_plaw8k_hashes():
    g = load_golden("windows_plaw8k")
    a = plaw8k_csr()
    assert a.nnz == int(g["nnz"])
    assert sha(a.values) == str(g["values_sha"])
    w = orc.partition(a)
    nc, dens, ci = orc.features(w)
    assert np.array_equal(nc, g["ncols"])
    assert np.array_equal(dens.view(np.uint64), g["density"].view(np.uint64))
    assert np.array_equal(orc.classify(nc, dens), g["codes"])
    assert sha(w.nonzero_cols.astype(np.int64)) == str(g["nonzero_cols_sha"])
    assert sha(w.cond_cols.astype(np.int64)) == str(g["cond_cols_sha"])
    x = orc.random_dense(a.num_cols, 32, 1)
    assert orc.max_rel_err(orc.spmm_exact(a, x), g["z_f32"]) <= 1e-5


def test_kat_condensation():
    # tests/test_windows.py:23-32
    g = load_golden("windows_kat_condense")
    w = orc.partition(golden_csr(g))
    assert w.nonzero_cols.tolist() == [5, 9]
    assert w.cond_cols.tolist() == [0, 1, 1]
    assert w.values.tolist() == [2.0, 1.0, 3.0]


@pytest.mark.parametrize("kind", ["gcn", "row", "gin", "raw"])
def test_gnn_restatement(kind):
    g = load_golden(f"gnn_{kind}")
    n = len(g["adj_row_ptr"]) - 1
    adj = orc.Csr(n, n, g["adj_row_ptr"], g["adj_col_idx"], np.ones(len(g["adj_col_idx"])))
    a = orc.normalize_adj(adj, kind)
    assert np.array_equal(a.row_ptr, g["a_row_ptr"]) and np.array_equal(a.col_idx, g["a_col_idx"])
    assert np.max(np.abs(a.values - g["a_values"])) <= 1e-15
    xn, z = orc.gcn_forward(a, g["x"], g["w"])
    assert np.abs(xn - g["x_next"]).max() < 1e-12
    assert np.abs(z - g["z"]).max() < 1e-12
    gw, gx = orc.gcn_backward(a, g["z"], g["gout"], g["w"])
    assert np.abs(gw - g["grad_w"]).max() < 1e-12
    assert np.abs(gx - g["grad_x"]).max() < 1e-12


@pytest.mark.parametrize("name", golden_names("loa_"))
def test_loa_restatement_exact(name):
    g = load_golden(name)
    n = int(g["n"])
    adj = orc.Csr(n, n, g["row_ptr"], g["col_idx"], np.ones(len(g["col_idx"])))
    assert np.array_equal(orc.sort_by_min_neighbor(adj), g["order"])
    groups = orc.build_windows_optimized(adj, vw=int(g["vw"]))
    flat = np.array([v for grp in groups for v in grp], dtype=np.int64)
    gptr = np.cumsum([0] + [len(grp) for grp in groups])
    assert np.array_equal(flat, g["flat"])
    assert np.array_equal(gptr, g["gptr"])
    orc.validate_grouping(groups, n)
    assert np.array_equal(orc.induced_perm(groups, n), g["perm"])


@pytest.mark.parametrize("name", ["loa_corpus_path50", "loa_corpus_gnp128", "loa_corpus_block32", "loa_cora"])
def test_loa_python_loop_equals_c(name):
    g = load_golden(name)
    n = int(g["n"])
    adj = orc.Csr(n, n, g["row_ptr"], g["col_idx"], np.ones(len(g["col_idx"])))
    groups = orc._loa_py(adj, int(g["vw"]), 16)
    assert [v for grp in groups for v in grp] == g["flat"].tolist()


def test_loa_hand_examples():
    # tests/test_layout.py:28-33, 71-77, 87-92
    adj = orc.graph_from_edges(6, [(0, 5), (1, 3), (2, 3)])
    assert orc.sort_by_min_neighbor(adj).tolist() == [5, 3, 1, 2, 0, 4]
    path4 = orc.graph_from_edges(4, [(0, 1), (1, 2), (2, 3)])
    assert orc.build_windows_optimized(path4, vw=4, group_size=2) == [[1, 3], [0, 2]]
    assert orc._loa_py(path4, 4, 2) == [[1, 3], [0, 2]]
    assert orc.induced_perm([[2, 0], [1]], 3).tolist() == [1, 2, 0]


def test_permute_symmetric_roundtrip():
    a = orc.random_csr(40, 40, 0.1, seed=3)
    perm = np.random.default_rng(1).permutation(40)
    b = orc.permute_symmetric(a, perm)
    inv = np.argsort(perm)
    c = orc.permute_symmetric(b, inv)
    assert np.array_equal(c.row_ptr, a.row_ptr) and np.array_equal(c.col_idx, a.col_idx)
    assert np.array_equal(c.values, a.values)
