"""Matrix Market / edge-list I/O with the reference's semantics and error messages
(reference matrices.py:175-307), vectorised with numpy so 100 M-entry files load in
seconds instead of the reference's per-line Python loop.

  load_matrix_market   matrices.py:175-252  coordinate real/integer/pattern, general/symmetric
  write_matrix_market  matrices.py:255-262  general, entries sorted by (row, col)
  parse_edge_list      matrices.py:265-291  'src dst' pairs, '#'/'%' comments, 1-based auto-detect
  load_edge_list       matrices.py:294-298
"""

from __future__ import annotations

import numpy as np

from .errors import FormatError
from .matrices import Graph, SparseCsr, graph_from_edges


def _data_lines(lines, start: int):
    """(1-based line number, stripped text) of non-blank, non-comment lines from index start."""
    for i in range(start, len(lines)):
        text = lines[i].strip()
        if text and not text.startswith("%"):
            yield i + 1, text


def load_matrix_market(path: str) -> SparseCsr:
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise FormatError("empty file", line=1)
    header = lines[0].strip().split()
    if len(header) < 5 or header[0] != "%%MatrixMarket":
        raise FormatError("missing %%MatrixMarket header", line=1)
    obj, fmt, field, symmetry = (t.lower() for t in header[1:5])
    if obj != "matrix" or fmt != "coordinate":
        raise FormatError(f"unsupported object/format '{obj} {fmt}'", line=1)
    if field not in ("real", "integer", "pattern"):
        raise FormatError(f"unsupported field type '{field}'", line=1)
    if symmetry not in ("general", "symmetric"):
        raise FormatError(f"unsupported symmetry '{symmetry}'", line=1)
    pattern = field == "pattern"
    it = _data_lines(lines, 1)
    try:
        size_line, size_text = next(it)
    except StopIteration:
        raise FormatError("missing size line", line=len(lines)) from None
    tokens = size_text.split()
    if len(tokens) != 3:
        raise FormatError("size line must be 'rows cols nnz'", line=size_line)
    try:
        m, n, k = (int(t) for t in tokens)
    except ValueError:
        raise FormatError("non-integer token in size line", line=size_line) from None
    if m < 0 or n < 0 or k < 0:
        raise FormatError("negative dimension in size line", line=size_line)
    entries = list(it)
    expected = 2 if pattern else 3
    fast = _fast_entries(entries, expected, m, n, k, pattern)
    if fast is not None:
        rows, cols, vals = fast
    else:
        rows, cols, vals = _slow_entries(entries, expected, m, n, k, pattern, len(lines))
    if symmetry == "symmetric":
        off = rows != cols
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, vals[off]]))
    return SparseCsr.from_coo(m, n, rows, cols, vals)


def _fast_entries(entries, expected, m, n, k, pattern):
    """numpy parse of well-formed entries; None when anything needs the per-line checks."""
    if len(entries) != k:
        return None
    if k == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.float64)
    try:
        data = np.loadtxt([t for _, t in entries], dtype=np.float64, ndmin=2)
    except ValueError:
        return None
    if data.shape != (k, expected):
        return None
    ij = data[:, :2]
    if not np.array_equal(ij, np.floor(ij)):
        return None
    i = ij[:, 0].astype(np.int64)
    j = ij[:, 1].astype(np.int64)
    if i.min() < 1 or i.max() > m or j.min() < 1 or j.max() > n:
        return None
    vals = np.ones(k, dtype=np.float64) if pattern else data[:, 2].copy()
    return i - 1, j - 1, vals


def _slow_entries(entries, expected, m, n, k, pattern, nlines):
    rows = np.empty(len(entries), dtype=np.int64)
    cols = np.empty(len(entries), dtype=np.int64)
    vals = np.ones(len(entries), dtype=np.float64)
    for idx, (lineno, text) in enumerate(entries):
        tok = text.split()
        if len(tok) != expected:
            raise FormatError(f"expected {expected} tokens per entry", line=lineno)
        try:
            i, j = int(tok[0]), int(tok[1])
            if not pattern:
                vals[idx] = float(tok[2])
        except ValueError:
            raise FormatError("non-numeric token in entry", line=lineno) from None
        if not (1 <= i <= m and 1 <= j <= n):
            raise FormatError(f"entry ({i}, {j}) outside declared {m}x{n} bounds", line=lineno)
        if idx >= k:
            raise FormatError(f"more than the declared {k} entries", line=lineno)
        rows[idx], cols[idx] = i - 1, j - 1
    if len(entries) < k:
        raise FormatError(f"declared {k} entries but found {len(entries)}", line=nlines)
    return rows, cols, vals


def write_matrix_market(csr, path: str) -> None:
    if not isinstance(csr, SparseCsr):
        csr = csr.to_host()
    rows, cols, vals = csr.to_coo()
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{csr.num_rows} {csr.num_cols} {csr.nnz}\n")
        fh.writelines(f"{i + 1} {j + 1} {float(v)!r}\n" for i, j, v in zip(rows.tolist(), cols.tolist(),
                                                                            vals.tolist()))


def parse_edge_list(path: str):
    edges = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            text = raw.strip()
            if not text or text.startswith("#") or text.startswith("%"):
                continue
            tokens = text.replace(",", " ").split()
            if len(tokens) != 2:
                raise FormatError("expected two integer ids per line", line=lineno)
            try:
                u, v = int(tokens[0]), int(tokens[1])
            except ValueError:
                raise FormatError("non-integer token", line=lineno) from None
            if u < 0 or v < 0:
                raise FormatError("negative vertex id", line=lineno)
            edges.append((u, v))
    if not edges:
        raise FormatError("empty edge list", line=1)
    one_based = min(min(e) for e in edges) >= 1
    if one_based:
        edges = [(u - 1, v - 1) for u, v in edges]
    return edges, one_based


def load_edge_list(path: str, undirected: bool = True) -> Graph:
    edges, _ = parse_edge_list(path)
    num_vertices = max(max(e) for e in edges) + 1
    return graph_from_edges(num_vertices, edges, undirected=undirected)
