"""Matrix Market / edge-list I/O with the reference's semantics and error messages
(reference matrices.py:175-307).  Entry lines are parsed by the library's multi-threaded
C++ parser (csrc/io_parse.cu: hcs_io_count / hcs_io_parse) and the CSR is built with
vectorised numpy; a file the strict parser calls irregular (or a missing library) is
re-parsed with the per-line restatement below, which raises the reference's exact
FormatError.  The parsed arrays are identical either way (tests/test_io_host.py).

  load_matrix_market   matrices.py:175-252  coordinate real/integer/pattern, general/symmetric
  write_matrix_market  matrices.py:255-262  general, entries sorted by (row, col)
  parse_edge_list      matrices.py:265-291  'src dst' pairs, '#'/'%' comments, 1-based auto-detect
  load_edge_list       matrices.py:294-298
"""

from __future__ import annotations

import numpy as np

from .errors import FormatError
from .matrices import Graph, SparseCsr, graph_from_edges

_KIND_MTX, _KIND_EDGES = 0, 1


def _cpp_entries(path: str, offset: int, kind: int, expected: int):
    """(a, b, v) int64/int64/float64 arrays of the data lines from byte `offset`, or None
    when the library is absent or the strict parser defers to the reference rules."""
    try:
        from . import _lib

        L = _lib.lib()
        if not hasattr(L, "hcs_io_parse"):
            return None
    except Exception:
        return None
    import ctypes

    cnt, irr = ctypes.c_int64(0), ctypes.c_int(0)
    bpath = path.encode()
    _lib.check(L.hcs_io_count(bpath, offset, kind, 0, ctypes.byref(cnt), ctypes.byref(irr)))
    if irr.value:
        return None
    k = int(cnt.value)
    a = np.empty(k, dtype=np.int64)
    b = np.empty(k, dtype=np.int64)
    v = np.empty(k, dtype=np.float64) if kind == _KIND_MTX else None
    if k:
        _lib.check(L.hcs_io_parse(bpath, offset, kind, expected, k, 0, a.ctypes.data, b.ctypes.data,
                                  v.ctypes.data if v is not None else None, ctypes.byref(irr)))
        if irr.value:
            return None
    return a, b, v


def _mtx_header(path: str):
    """Header line, size line and the byte offset where the entries start (the reference's
    checks on those lines run in load_matrix_market either way); None if not well formed."""
    with open(path, "rb") as fh:
        first = fh.readline()
        off = len(first)
        while True:
            raw = fh.readline()
            if not raw:
                return None
            off += len(raw)
            text = raw.decode("utf-8", errors="strict").strip()
            if text and not text.startswith("%"):
                return first.decode("utf-8").strip(), text, off


def _data_lines(lines, start: int):
    """(1-based line number, stripped text) of non-blank, non-comment lines from index start."""
    for i in range(start, len(lines)):
        text = lines[i].strip()
        if text and not text.startswith("%"):
            yield i + 1, text


def load_matrix_market(path: str) -> SparseCsr:
    fast = _load_matrix_market_cpp(path)
    if fast is not None:
        return fast
    return _load_matrix_market_py(path)


def _check_mtx_header(header_text: str):
    header = header_text.split()
    if len(header) < 5 or header[0] != "%%MatrixMarket":
        raise FormatError("missing %%MatrixMarket header", line=1)
    obj, fmt, field, symmetry = (t.lower() for t in header[1:5])
    if obj != "matrix" or fmt != "coordinate":
        raise FormatError(f"unsupported object/format '{obj} {fmt}'", line=1)
    if field not in ("real", "integer", "pattern"):
        raise FormatError(f"unsupported field type '{field}'", line=1)
    if symmetry not in ("general", "symmetric"):
        raise FormatError(f"unsupported symmetry '{symmetry}'", line=1)
    return field, symmetry


def _finish_mtx(m, n, rows, cols, vals, symmetry):
    if symmetry == "symmetric":
        off = rows != cols
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, vals[off]]))
    return SparseCsr.from_coo(m, n, rows, cols, vals)


def _load_matrix_market_cpp(path: str):
    """Well-formed files through the C++ entry parser; None -> the reference-rules path."""
    try:
        hdr = _mtx_header(path)
    except (OSError, UnicodeDecodeError):
        return None
    if hdr is None:
        return None
    header_text, size_text, offset = hdr
    try:
        field, symmetry = _check_mtx_header(header_text)
        m, n, k = (int(t) for t in size_text.split())
    except (FormatError, ValueError):
        return None
    if m < 0 or n < 0 or k < 0:
        return None
    pattern = field == "pattern"
    parsed = _cpp_entries(path, offset, _KIND_MTX, 2 if pattern else 3)
    if parsed is None:
        return None
    i, j, vals = parsed
    if i.size != k or (k and (i.min() < 1 or i.max() > m or j.min() < 1 or j.max() > n)):
        return None  # the reference path reports the count / bounds error with its line
    return _finish_mtx(m, n, i - 1, j - 1, vals, symmetry)


def _load_matrix_market_py(path: str) -> SparseCsr:
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise FormatError("empty file", line=1)
    field, symmetry = _check_mtx_header(lines[0].strip())
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
    return _finish_mtx(m, n, rows, cols, vals, symmetry)


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
    """matrices.py:265-291: (edges as a list of (u, v), one_based)."""
    u, v, one_based = parse_edge_arrays(path)
    return list(zip(u.tolist(), v.tolist())), one_based


def parse_edge_arrays(path: str):
    """parse_edge_list as (u int64[], v int64[], one_based): the C++ parser for regular
    files, the reference's per-line rules (exact FormatError) otherwise."""
    parsed = _cpp_entries(path, 0, _KIND_EDGES, 2)
    if parsed is not None and parsed[0].size:
        u, v, _ = parsed
        one_based = bool(min(int(u.min()), int(v.min())) >= 1)
        if one_based:
            u, v = u - 1, v - 1
        return u, v, one_based
    edges, one_based = _parse_edge_list_py(path)
    arr = np.array(edges, dtype=np.int64).reshape(-1, 2)
    return arr[:, 0].copy(), arr[:, 1].copy(), one_based


def _parse_edge_list_py(path: str):
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
    """matrices.py:294-298 with graph_from_edges (292-307) vectorised: deduplicated unit
    (u, v) pairs (+ (v, u) when undirected) -> CSR."""
    u, v, _ = parse_edge_arrays(path)
    num_vertices = int(max(u.max(), v.max())) + 1
    if undirected:
        u, v = np.concatenate([u, v]), np.concatenate([v, u])
    keys = np.sort(u * num_vertices + v)  # sorted, deduplicated (row, col) pairs
    if keys.size:  # (np.unique hashes first: 13 s at 10 M keys)
        keys = keys[np.concatenate(([True], keys[1:] != keys[:-1]))]
    rows, cols = keys // num_vertices, keys % num_vertices
    row_ptr = np.zeros(num_vertices + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=num_vertices), out=row_ptr[1:])
    adj = SparseCsr(num_vertices, num_vertices, row_ptr, cols, np.ones(rows.size))
    return Graph(num_vertices, adj, undirected)


def load_edge_list_device(path: str, undirected: bool = True, device=None):
    """load_edge_list straight into HBM: the parsed (u, v) arrays go to the GPU once and are
    symmetrised, deduplicated and sorted there (one radix sort of 64-bit keys), giving the
    DeviceCsr the kernels consume -- the same CSR as load_edge_list(...).adjacency."""
    import torch

    from . import _lib
    from .graphgen import csr_from_keys

    dev = device if device is not None else _lib.require_cuda()
    u, v, _ = parse_edge_arrays(path)
    num_vertices = int(max(u.max(), v.max())) + 1
    tu = torch.from_numpy(u).to(dev, non_blocking=True)
    tv = torch.from_numpy(v).to(dev, non_blocking=True)
    keys = tu * num_vertices + tv
    if undirected:
        keys = torch.cat([keys, tv * num_vertices + tu])
    keys = torch.unique(keys, sorted=True)
    csr = csr_from_keys(num_vertices, keys)
    csr.symmetric = bool(undirected)
    return csr
