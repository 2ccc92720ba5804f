"""CPU tests of the CLI front end and the I/O module (no GPU needed): argument handling,
exit codes (reference cli.py:627-650), Matrix Market / edge-list parsing with the
reference's semantics and messages (matrices.py:175-307)."""

import numpy as np
import pytest

from oracle import rowwin_oracle as orc

from paper_2412_08902_b200 import cli, io
from paper_2412_08902_b200.errors import FormatError


def test_usage_errors_exit_1(capsys):
    assert cli.main(["no-such-command"]) == 1
    assert cli.main(["spmm", "--matrix"]) == 1
    assert cli.main(["--precision", "f64", "spmm", "--matrix", "a.mtx", "--dense", "random:dim=2"]) == 1


def test_bad_input_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    assert cli.main(["partition-report", "--matrix", str(bad)]) == 2
    assert "outside declared" in capsys.readouterr().err
    assert cli.main(["classify", "--matrix", str(tmp_path / "missing.mtx")]) == 2
    assert cli.main(["pipeline", "--graph", str(tmp_path / "missing.edges")]) == 2


def test_matrix_market_roundtrip_and_symmetric(tmp_path):
    p = tmp_path / "s.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n% comment\n3 3 3\n1 1 2.0\n2 1 1.5\n3 2 -1\n")
    a = io.load_matrix_market(str(p))
    assert a.row_ptr.tolist() == [0, 2, 4, 5]
    assert a.col_idx.tolist() == [0, 1, 0, 2, 1]
    assert a.values.tolist() == [2.0, 1.5, 1.5, -1.0, -1.0]
    q = tmp_path / "g.mtx"
    io.write_matrix_market(a, str(q))
    b = io.load_matrix_market(str(q))
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values, b.values)
    pat = tmp_path / "p.mtx"
    pat.write_text("%%MatrixMarket matrix coordinate pattern general\n2 3 2\n1 3\n2 1\n")
    c = io.load_matrix_market(str(pat))
    assert c.num_cols == 3 and c.values.tolist() == [1.0, 1.0]


@pytest.mark.parametrize("text,msg", [
    ("", "empty file"),
    ("hello\n", "header"),
    ("%%MatrixMarket matrix array real general\n", "unsupported object/format"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n", "field type"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n", "symmetry"),
    ("%%MatrixMarket matrix coordinate real general\n1 1\n", "size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "declared 2 entries but found 1"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n", "more than the declared"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", "non-numeric"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", "expected 3 tokens"),
])
def test_matrix_market_errors(tmp_path, text, msg):
    p = tmp_path / "e.mtx"
    p.write_text(text)
    with pytest.raises(FormatError, match=msg):
        io.load_matrix_market(str(p))


def test_edge_list_matches_oracle(tmp_path):
    p = tmp_path / "g.edges"
    p.write_text("# c\n1 2\n2 3\n3,1\n% c\n4 1\n")
    g = io.load_edge_list(str(p))
    ref = orc.graph_from_edges(4, [(0, 1), (1, 2), (2, 0), (3, 0)])
    assert g.num_vertices == 4 and g.undirected
    assert np.array_equal(g.adjacency.row_ptr, ref.row_ptr) and np.array_equal(g.adjacency.col_idx, ref.col_idx)
    bad = tmp_path / "b.edges"
    bad.write_text("0 1 2\n")
    with pytest.raises(FormatError, match="two integer ids"):
        io.load_edge_list(str(bad))
