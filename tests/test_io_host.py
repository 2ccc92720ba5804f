"""CPU: the C++ entry parser (csrc/io_parse.cu, hcs_io_count / hcs_io_parse) behind
io.load_matrix_market / parse_edge_list / load_edge_list gives exactly the arrays of the
reference-rules path, and every irregular file still raises the reference's FormatError
(message and line) through that path (reference matrices.py:175-307)."""

import os

import numpy as np
import pytest

from paper_2412_08902_b200 import io
from paper_2412_08902_b200.errors import FormatError

MTX_CASES = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n% c\n\n3 4 4\n1 1 1.5\n2 3 -2e-3\n3 4 7\n1 2 0.1\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 3\n1 1 2\n3 1 -1.25\n4 2 3.0e+1\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 3\n3 1\n",
    "integer_crlf": "%%MatrixMarket matrix coordinate integer general\r\n2 2 2\r\n1 1 4\r\n2 2 -5\r\n",
    "comments_inside": "%%MatrixMarket matrix coordinate real general\n2 2 2\n% mid\n1 1 1\n\n   2 2    2.5  \n",
    "float_indices": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.0 2 3\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n1 1 2\n2 1 3\n",
}
MTX_BAD = {
    "bad_token": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 3\n",
    "too_many": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 2\n",
    "too_few": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n",
    "bounds": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "fields": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "header": "%%MatrixMarket matrix array real general\n2 2\n1\n",
}
EDGE_CASES = {
    "one_based": "# c\n1 2\n2 3\n\n3 1\n",
    "zero_based_commas": "0,1\n1 , 2\n% x\n2\t0\n",
    "dups": "5 6\n6 5\n5 6\n",
}
EDGE_BAD = {"three": "1 2 3\n", "neg": "1 -2\n", "word": "a b\n", "empty": "# only\n"}


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def lib_available():
    try:
        from paper_2412_08902_b200 import _lib

        return hasattr(_lib.lib(), "hcs_io_parse")
    except Exception:
        return False


needs_lib = pytest.mark.skipif(not lib_available(), reason="libhcspmm.so not built")


@needs_lib
@pytest.mark.parametrize("name", sorted(MTX_CASES))
def test_mtx_cpp_equals_reference_rules(tmp_path, name):
    path = write(tmp_path, name + ".mtx", MTX_CASES[name])
    fast = io._load_matrix_market_cpp(path)
    assert fast is not None  # the strict parser takes these files
    ref = io._load_matrix_market_py(path)
    for f in ("num_rows", "num_cols"):
        assert getattr(fast, f) == getattr(ref, f)
    assert np.array_equal(fast.row_ptr, ref.row_ptr)
    assert np.array_equal(fast.col_idx, ref.col_idx)
    assert np.array_equal(fast.values, ref.values)  # bit-identical doubles
    assert io.load_matrix_market(path).nnz == ref.nnz


@needs_lib
@pytest.mark.parametrize("name", sorted(MTX_BAD))
def test_mtx_irregular_raises_reference_error(tmp_path, name):
    path = write(tmp_path, name + ".mtx", MTX_BAD[name])
    assert io._load_matrix_market_cpp(path) is None
    with pytest.raises(FormatError) as e1:
        io._load_matrix_market_py(path)
    with pytest.raises(FormatError) as e2:
        io.load_matrix_market(path)
    assert str(e1.value) == str(e2.value)


@needs_lib
@pytest.mark.parametrize("name", sorted(EDGE_CASES))
def test_edges_cpp_equals_reference_rules(tmp_path, name):
    path = write(tmp_path, name + ".txt", EDGE_CASES[name])
    edges_py, ob_py = io._parse_edge_list_py(path)
    u, v, ob = io.parse_edge_arrays(path)
    assert ob == ob_py and list(zip(u.tolist(), v.tolist())) == edges_py
    g = io.load_edge_list(path)
    # same CSR as the reference's set-based graph_from_edges
    from paper_2412_08902_b200.matrices import graph_from_edges

    ref = graph_from_edges(max(max(e) for e in edges_py) + 1, edges_py, undirected=True)
    assert np.array_equal(g.adjacency.row_ptr, ref.adjacency.row_ptr)
    assert np.array_equal(g.adjacency.col_idx, ref.adjacency.col_idx)
    assert np.array_equal(g.adjacency.values, ref.adjacency.values)


@pytest.mark.parametrize("name", sorted(EDGE_BAD))
def test_edges_irregular_raises_reference_error(tmp_path, name):
    path = write(tmp_path, name + ".txt", EDGE_BAD[name])
    with pytest.raises(FormatError) as e1:
        io._parse_edge_list_py(path)
    with pytest.raises(FormatError) as e2:
        io.parse_edge_list(path)
    assert str(e1.value) == str(e2.value)


@needs_lib
def test_large_random_files_match(tmp_path):
    rng = np.random.default_rng(0)
    n, k = 5000, 200_000
    i = rng.integers(1, n + 1, k)
    j = rng.integers(1, n + 1, k)
    x = rng.standard_normal(k) * 10.0 ** rng.integers(-8, 8, k)
    body = "".join(f"{a} {b} {float(c)!r}\n" for a, b, c in zip(i, j, x))
    path = write(tmp_path, "big.mtx", f"%%MatrixMarket matrix coordinate real general\n{n} {n} {k}\n" + body)
    fast, ref = io._load_matrix_market_cpp(path), io._load_matrix_market_py(path)
    assert np.array_equal(fast.col_idx, ref.col_idx) and np.array_equal(fast.values, ref.values)
    epath = write(tmp_path, "big.txt", "".join(f"{a} {b}\n" for a, b in zip(i, j)))
    u, v, _ = io.parse_edge_arrays(epath)
    assert np.array_equal(u, i - 1) and np.array_equal(v, j - 1)

