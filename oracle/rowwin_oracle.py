"""CPU oracle for the HC-SpMM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package `rowwin`
(/root/reference/pkg/src/rowwin, arXiv 2412.08902 CPU reference).  It exists
so the GPU product can be checked on the GPU box, where /root/reference does
not exist.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it, and only as the
checker or the timed CPU baseline -- never as a product code path.

Parity of this restatement is pinned against golden vectors generated from
the reference itself (tests/golden/make_golden.py, fixtures in tests/golden/,
checked by tests/test_oracle_golden.py).

Every function cites the reference file:line it restates.  Paths are relative
to /root/reference/pkg/src/rowwin/.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

import numpy as np

WINDOW_HEIGHT = 16  # windows.py:12
TILE_COLS = 8       # windows.py:13
TILE_DIM = 16       # windows.py:14

# data/default_selector.json:2-25 -- the 7 doubles of the shipped selector.
# Stored in the product package as paper_2412_08902_b200/data/selector_default.json;
# duplicated here so the oracle has no product import.
DEFAULT_SELECTOR = dict(
    w_ncols=-0.1454848214145233,
    w_density=-9.249873814861964,
    bias=-15.105252482198011,
    feature_means=(140.38659793814432, 0.5),
    feature_scales=(123.08273985946481, 0.2570676399373035),
)


# --------------------------------------------------------------------------- L0
@dataclass(frozen=True)
class Csr:
    """matrices.py:24-40 SparseCsr (row_ptr int64, col_idx int64, values float64)."""

    num_rows: int
    num_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


def from_coo(num_rows, num_cols, rows, cols, vals) -> Csr:
    """matrices.py:64-97: lexsort by (row, col); duplicates summed with np.add.at."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if not (rows.shape == cols.shape == vals.shape):
        raise ValueError("coordinate arrays must have equal length")
    if rows.size:
        if rows.min() < 0 or rows.max() >= num_rows:
            raise ValueError("row index out of range")
        if cols.min() < 0 or cols.max() >= num_cols:
            raise ValueError("column index out of range")
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        head = np.empty(rows.size, dtype=bool)
        head[0] = True
        head[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        group = np.cumsum(head) - 1
        summed = np.zeros(int(group[-1]) + 1, dtype=np.float64)
        np.add.at(summed, group, vals)  # sequential left-to-right sum, matrices.py:92
        rows, cols, vals = rows[head], cols[head], summed
    counts = np.bincount(rows, minlength=num_rows) if num_rows else np.zeros(0, np.int64)
    row_ptr = np.zeros(num_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return Csr(num_rows, num_cols, row_ptr, cols, vals)


def to_coo(csr: Csr):
    """matrices.py:99-101."""
    rows = np.repeat(np.arange(csr.num_rows, dtype=np.int64), np.diff(csr.row_ptr))
    return rows, csr.col_idx.copy(), csr.values.copy()


def to_dense(csr: Csr) -> np.ndarray:
    """matrices.py:103-107."""
    d = np.zeros((csr.num_rows, csr.num_cols))
    r, c, v = to_coo(csr)
    d[r, c] = v
    return d


def graph_from_edges(n: int, edges, undirected: bool = True) -> Csr:
    """matrices.py:292-307: dedup (u,v) pairs (+ mirror), unit values."""
    pairs = set()
    for u, v in edges:
        pairs.add((u, v))
        if undirected:
            pairs.add((v, u))
    if pairs:
        rows, cols = (np.array(a, dtype=np.int64) for a in zip(*sorted(pairs)))
    else:
        rows = cols = np.zeros(0, dtype=np.int64)
    return from_coo(n, n, rows, cols, np.ones(rows.size))


def permute_symmetric(csr: Csr, perm) -> Csr:
    """matrices.py:310-318: entry (i, j) moves to (perm[i], perm[j]); rows re-sorted."""
    if csr.num_rows != csr.num_cols:
        raise ValueError("symmetric permutation requires a square matrix")
    perm = np.asarray(perm, dtype=np.int64)
    if perm.shape != (csr.num_rows,) or not np.array_equal(np.sort(perm), np.arange(csr.num_rows)):
        raise ValueError("perm must be a bijection on 0..n-1")
    r, c, v = to_coo(csr)
    return from_coo(csr.num_rows, csr.num_cols, perm[r], perm[c], v)


def random_dense(rows: int, dim: int, seed: int, low=-1.0, high=1.0) -> np.ndarray:
    """matrices.py:146-149 DenseMatrix.random."""
    return np.random.default_rng(seed).uniform(low, high, size=(rows, dim))


def random_csr(num_rows, num_cols, density, seed) -> Csr:
    """tests/conftest.py:31-39 random_csr (exact cell sampling, values U[-1,1])."""
    rng = np.random.default_rng(seed)
    total = num_rows * num_cols
    nnz = min(total, max(0, int(round(density * total))))
    cells = rng.choice(total, size=nnz, replace=False)
    rows, cols = cells // num_cols, cells % num_cols
    vals = rng.uniform(-1.0, 1.0, size=nnz)
    return from_coo(num_rows, num_cols, rows, cols, vals)


def max_rel_err(actual, oracle) -> float:
    """tests/conftest.py:42-47: max|a-o| / max|o| (max|a| if the oracle is all zero)."""
    oracle = np.asarray(oracle, dtype=np.float64)
    actual = np.asarray(actual, dtype=np.float64)
    scale = float(np.abs(oracle).max()) if oracle.size else 0.0
    if scale == 0.0:
        return float(np.abs(actual).max()) if actual.size else 0.0
    return float(np.abs(actual - oracle).max()) / scale


# --------------------------------------------------------------------------- L1
@dataclass(frozen=True)
class Windows:
    """Structure-of-arrays form of windows.py:17-69 RowWindow list.

    Window w covers rows [w*wh, min((w+1)*wh, n)).  Its nonzero_cols are
    nonzero_cols[win_col_ptr[w]:win_col_ptr[w+1]]; entry e (CSR order) has
    condensed id cond_cols[e]; local_ptr is row_ptr sliced (windows.py:101).
    """

    num_rows: int
    window_height: int
    row_ptr: np.ndarray
    win_col_ptr: np.ndarray
    nonzero_cols: np.ndarray
    cond_cols: np.ndarray
    values: np.ndarray

    @property
    def num_windows(self) -> int:
        return len(self.win_col_ptr) - 1

    def ncols(self) -> np.ndarray:
        return np.diff(self.win_col_ptr)

    def row_start(self) -> np.ndarray:
        return np.arange(self.num_windows, dtype=np.int64) * self.window_height

    def row_count(self) -> np.ndarray:
        rs = self.row_start()
        return np.minimum(rs + self.window_height, self.num_rows) - rs

    def nnz(self) -> np.ndarray:
        rs = self.row_start()
        re = np.minimum(rs + self.window_height, self.num_rows)
        return self.row_ptr[re] - self.row_ptr[rs]


def partition(csr: Csr, window_height: int = WINDOW_HEIGHT) -> Windows:
    """windows.py:81-106 vectorised.

    The reference calls np.unique(cols, return_inverse=True) per window
    (windows.py:94).  Sorting (window, col) keys globally yields the same
    ascending unique columns and inverse indices per window, because every
    key of window w sorts before every key of window w+1.
    """
    if window_height <= 0:
        raise ValueError("window_height must be positive")
    n = csr.num_rows
    nwin = -(-n // window_height)
    row_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(csr.row_ptr))
    win_of = row_of // window_height
    keys = win_of * np.int64(max(csr.num_cols, 1)) + csr.col_idx.astype(np.int64)
    uniq, inv = np.unique(keys, return_inverse=True)
    uwin = uniq // np.int64(max(csr.num_cols, 1))
    ncols = np.bincount(uwin, minlength=nwin) if nwin else np.zeros(0, np.int64)
    win_col_ptr = np.zeros(nwin + 1, dtype=np.int64)
    np.cumsum(ncols, out=win_col_ptr[1:])
    nonzero_cols = uniq - uwin * np.int64(max(csr.num_cols, 1))
    cond = inv.astype(np.int64) - win_col_ptr[win_of]
    return Windows(n, window_height, csr.row_ptr, win_col_ptr, nonzero_cols, cond, csr.values)


def features(w: Windows):
    """windows.py:109-123: (ncols, density, computing_intensity), zeros for empty windows.

    density = nnz / (row_count * ncols) is Python int/int true division, i.e. a
    correctly rounded IEEE division of two exact doubles (values < 2**53).
    """
    nc = w.ncols().astype(np.int64)
    nnz = w.nnz().astype(np.int64)
    rc = w.row_count().astype(np.int64)
    dens = np.zeros(len(nc))
    ci = np.zeros(len(nc))
    live = nc > 0
    dens[live] = nnz[live].astype(np.float64) / (rc[live] * nc[live]).astype(np.float64)
    ci[live] = nnz[live].astype(np.float64) / nc[live].astype(np.float64)
    return nc, dens, ci


def tile_count(ncols, tile_cols: int = TILE_COLS):
    """windows.py:126-128: ceil(ncols / tile_cols)."""
    ncols = np.asarray(ncols, dtype=np.int64)
    return -(-ncols // tile_cols)


def classify(ncols, density, model: dict = DEFAULT_SELECTOR) -> np.ndarray:
    """selector.py:48-56 + 59-64 vectorised; returns Assignment codes (executors.py:30: 0 scalar, 1 tile).

    score = w_ncols*zn + w_density*zd + bias evaluated left to right in float64
    (numpy elementwise ops are individually IEEE-rounded, no contraction).
    """
    nc = np.asarray(ncols, dtype=np.int64)
    d = np.asarray(density, dtype=np.float64)
    zn = (nc.astype(np.float64) - model["feature_means"][0]) / model["feature_scales"][0]
    zd = (d - model["feature_means"][1]) / model["feature_scales"][1]
    score = model["w_ncols"] * zn + model["w_density"] * zd
    score = score + model["bias"]
    codes = np.where(score > 0, 0, 1).astype(np.uint8)
    codes[nc == 0] = 0  # selector.py:54-55 empty -> SCALAR
    return codes


def load_selector(path: str) -> dict:
    """selector.py:260-281 _model_from_doc / load_model."""
    with open(path, "r", encoding="utf-8") as fh:
        doc = json.load(fh)
    return dict(
        w_ncols=float(doc["w_ncols"]),
        w_density=float(doc["w_density"]),
        bias=float(doc["bias"]),
        feature_means=(float(doc["feature_means"][0]), float(doc["feature_means"][1])),
        feature_scales=(float(doc["feature_scales"][0]), float(doc["feature_scales"][1])),
    )


# --------------------------------------------------------------------------- L3
def exec_stats(w: Windows, codes) -> dict:
    """executors.py:148-157 + 185-187: counters over non-empty windows only."""
    codes = np.asarray(codes, dtype=np.uint8)
    nnz = w.nnz()
    live = nnz > 0
    tile = live & (codes == 1)
    scal = live & (codes == 0)
    return dict(
        windows_scalar=int(scal.sum()),
        windows_tile=int(tile.sum()),
        entries_scalar=int(nnz[scal].sum()),
        entries_tile=int(nnz[tile].sum()),
        tiles_processed=int(tile_count(w.ncols()[tile]).sum()),
    )


def spmm_exact(csr: Csr, x: np.ndarray) -> np.ndarray:
    """Exact float64 Z = A X (the role of matrices.py:321-325 spmm_dense_oracle,
    without densifying).  Rows are reduced with np.add.reduceat."""
    x = np.asarray(x, dtype=np.float64)
    z = np.zeros((csr.num_rows, x.shape[1]))
    if csr.nnz == 0:
        return z
    prod = csr.values[:, None] * x[csr.col_idx]
    lens = np.diff(csr.row_ptr)
    nz = np.flatnonzero(lens > 0)
    z[nz] = np.add.reduceat(prod, csr.row_ptr[nz], axis=0)
    return z


def scalar_window(w: Windows, wid: int, x: np.ndarray) -> np.ndarray:
    """executors.py:100-108: per-row values @ X[nonzero_cols[cond_cols]]."""
    rs = wid * w.window_height
    rc = min(rs + w.window_height, w.num_rows) - rs
    nzc = w.nonzero_cols[w.win_col_ptr[wid]:w.win_col_ptr[wid + 1]]
    out = np.zeros((rc, x.shape[1]), dtype=x.dtype)
    for r in range(rc):
        lo, hi = int(w.row_ptr[rs + r]), int(w.row_ptr[rs + r + 1])
        if hi > lo:
            out[r] = w.values[lo:hi].astype(x.dtype, copy=False) @ x[nzc[w.cond_cols[lo:hi]]]
    return out


def tile_window(w: Windows, wid: int, x: np.ndarray, tile_cols=TILE_COLS, dim_tile=TILE_DIM) -> np.ndarray:
    """executors.py:111-141: zero-padded slab x gathered X, 8-col blocks x 16-dim chunks."""
    rs = wid * w.window_height
    rc = min(rs + w.window_height, w.num_rows) - rs
    e0, e1 = int(w.row_ptr[rs]), int(w.row_ptr[rs + rc])
    nzc = w.nonzero_cols[w.win_col_ptr[wid]:w.win_col_ptr[wid + 1]]
    dim = x.shape[1]
    out = np.zeros((rc, dim), dtype=x.dtype)
    if e1 == e0:
        return out
    nb = int(tile_count(len(nzc), tile_cols))
    padded = nb * tile_cols
    slab = np.zeros((rc, padded), dtype=x.dtype)
    local_rows = np.repeat(np.arange(rc), np.diff(w.row_ptr[rs:rs + rc + 1]))
    slab[local_rows, w.cond_cols[e0:e1]] = w.values[e0:e1].astype(x.dtype, copy=False)
    gathered = np.zeros((padded, dim), dtype=x.dtype)
    gathered[: len(nzc)] = x[nzc]
    for d0 in range(0, dim, dim_tile):
        d1 = min(d0 + dim_tile, dim)
        for b in range(nb):
            c0 = b * tile_cols
            out[:, d0:d1] += slab[:, c0:c0 + tile_cols] @ gathered[c0:c0 + tile_cols, d0:d1]
    return out


def spmm_hybrid(w: Windows, codes, x: np.ndarray, precision="f32", window_ids=None) -> np.ndarray:
    """executors.py:160-188 + 234-251: per non-empty window, tile or scalar path.

    `window_ids` restricts execution to a subset (used for bounded CPU-baseline
    samples); other rows stay zero.  Returns Z (total_rows x dim).
    """
    dt = {"f64": np.float64, "f32": np.float32}[precision]
    xd = np.asarray(x).astype(dt, copy=False)
    z = np.zeros((w.num_rows, xd.shape[1]), dtype=dt)
    nnz = w.nnz()
    ids = range(w.num_windows) if window_ids is None else window_ids
    for wid in ids:
        if nnz[wid] == 0:
            continue
        rs = wid * w.window_height
        rc = min(rs + w.window_height, w.num_rows) - rs
        kern = tile_window if codes[wid] else scalar_window
        z[rs:rs + rc] = kern(w, wid, xd)
    return z


# --------------------------------------------------------------------------- L4 gnn
def normalize_adj(adj: Csr, kind: str = "gcn") -> Csr:
    """gnn.py:68-95: gcn D^-1/2 (A+I) D^-1/2, row D^-1 A, raw A, gin A+I."""
    kinds = ("gcn", "row", "raw", "gin")
    if kind not in kinds:
        raise ValueError(f"kind must be one of {kinds}, got {kind!r}")
    if kind == "raw":
        return adj
    r, c, v = to_coo(adj)
    if kind == "row":
        deg = np.diff(adj.row_ptr).astype(np.float64)
        scale = np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0)
        return from_coo(adj.num_rows, adj.num_cols, r, c, v * scale[r])
    n = adj.num_rows
    eye = np.arange(n, dtype=np.int64)
    loops = from_coo(n, n, np.concatenate([r, eye]), np.concatenate([c, eye]), np.concatenate([v, np.ones(n)]))
    if kind == "gin":
        return loops
    r2, c2, v2 = to_coo(loops)
    deg = np.zeros(n)
    np.add.at(deg, r2, v2)
    inv_sqrt = 1.0 / np.sqrt(deg)
    return from_coo(n, n, r2, c2, v2 * inv_sqrt[r2] * inv_sqrt[c2])


def glorot(d_in: int, d_out: int, seed: int) -> np.ndarray:
    """gnn.py:40-46 GnnLayer.random."""
    rng = np.random.default_rng(seed)
    bound = np.sqrt(6.0 / (d_in + d_out))
    return rng.uniform(-bound, bound, size=(d_in, d_out))


def transpose(csr: Csr) -> Csr:
    """gnn.py:181-182: A^T via to_coo + from_coo(cols, rows)."""
    r, c, v = to_coo(csr)
    return from_coo(csr.num_cols, csr.num_rows, c, r, v)


def gcn_forward(a_norm: Csr, x: np.ndarray, w: np.ndarray):
    """gnn.py:121-159: returns (x_next = (A X) W, z_cache = A X) in float64."""
    if x.shape[1] != w.shape[0]:
        raise ValueError(f"X has {x.shape[1]} features, layer expects {w.shape[0]}")
    z = spmm_exact(a_norm, x)
    return z @ w, z


def gcn_backward(a_norm: Csr, z_cache: np.ndarray, grad_out: np.ndarray, w: np.ndarray):
    """gnn.py:162-205: grad_w = Z^T G, grad_x = A^T (G W^T), float64."""
    if a_norm.num_rows != a_norm.num_cols:
        raise ValueError("backward requires a square aggregation operator")
    grad_w = z_cache.T @ grad_out
    grad_x = spmm_exact(transpose(a_norm), grad_out @ w.T)
    return grad_w, grad_x


# --------------------------------------------------------------------------- L4 layout (LOA)
def sort_by_min_neighbor(adj: Csr) -> np.ndarray:
    """layout.py:99-109: lexsort by (min neighbour, id); isolated vertices key n."""
    n = adj.num_rows
    key = np.full(n, n, dtype=np.int64)
    starts = adj.row_ptr[:-1]
    nonempty = np.flatnonzero(np.diff(adj.row_ptr) > 0)
    key[nonempty] = adj.col_idx[starts[nonempty]]
    return np.lexsort((np.arange(n), key)).astype(np.int64)


def build_windows_optimized(adj: Csr, vw: int = 128, group_size: int = WINDOW_HEIGHT) -> list[list[int]]:
    """layout.py:186-263 (Algorithm 6), restated with the same integer semantics.

    Uses the C restatement (oracle/loa_oracle.c) when its shared library has been
    built, else this pure-Python loop.  Candidates are the first `vw` unvisited
    sorted positions at or after the seed position (layout.py:112-115, 234);
    fraction (cur_eles+deg)/(cur_cols+deg-cns) with den 0 -> (0,1) (80-91);
    argmax by exact cross-multiplication, then strictly higher degree, then
    earliest scan index (118-130).
    """
    if vw < 1:
        raise ValueError("vw must be >= 1")
    lib = _loa_lib()
    if lib is not None:
        return _loa_c(lib, adj, vw, group_size)
    return _loa_py(adj, vw, group_size)


def _loa_py(adj: Csr, vw: int, group_size: int) -> list[list[int]]:
    n = adj.num_rows
    order = sort_by_min_neighbor(adj)
    rp, ci = adj.row_ptr, adj.col_idx
    deg = np.diff(rp).astype(np.int64)
    unvisited = np.ones(n, dtype=bool)
    cns = np.zeros(n, dtype=np.int64)
    groups = []
    seed = 0
    while seed < n:
        if not unvisited[seed]:
            seed += 1
            continue
        touched = []
        in_cols = set()
        cur_eles = 0
        cur_cols = 0

        def admit(v):
            nonlocal cur_eles, cur_cols
            for c in ci[rp[v]:rp[v + 1]].tolist():
                if c in in_cols:
                    continue
                in_cols.add(c)
                cur_cols += 1
                for u in ci[rp[c]:rp[c + 1]].tolist():
                    cns[u] += 1
                    touched.append(u)
            cur_eles += int(deg[v])

        v0 = int(order[seed])
        unvisited[seed] = False
        group = [v0]
        admit(v0)
        while len(group) < group_size:
            hits = np.flatnonzero(unvisited[seed:])[:vw] + seed
            if hits.size == 0:
                break
            best = None
            for k, p in enumerate(hits.tolist()):
                v = int(order[p])
                d = int(deg[v])
                num = cur_eles + d
                den = cur_cols + d - int(cns[v])
                if den == 0:
                    num, den = 0, 1
                if best is None:
                    best = (num, den, d, p)
                    continue
                bn, bd, bdeg, _ = best
                lhs, rhs = num * bd, bn * den
                if lhs > rhs or (lhs == rhs and d > bdeg):
                    best = (num, den, d, p)
            p_best = best[3]
            unvisited[p_best] = False
            vb = int(order[p_best])
            group.append(vb)
            admit(vb)
        groups.append(group)
        for u in touched:
            cns[u] = 0
    return groups


_LOA_LIB = None


def _loa_lib():
    global _LOA_LIB
    if _LOA_LIB is None:
        import ctypes

        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle.so")
        if not os.path.exists(path):
            _LOA_LIB = False
        else:
            lib = ctypes.CDLL(path)
            lib.oracle_loa.restype = ctypes.c_int
            lib.oracle_loa.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            _LOA_LIB = lib
    return _LOA_LIB or None


def spmm_exact_c(row_ptr, col_idx, values, x: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    """Exact float64 Z = A X through oracle/spmm_oracle.c (same math as spmm_exact: float64
    products summed per row in CSR order), multi-threaded for BASELINE-size checks (C2: 115 M
    entries x 128 features).  Raises if liboracle.so is not built."""
    import ctypes

    lib = _loa_lib()
    if not lib:
        raise RuntimeError("oracle/liboracle.so is not built (make -C oracle)")
    if not hasattr(lib, "_spmm_typed"):
        lib.oracle_spmm_f64.restype = ctypes.c_int
        lib.oracle_spmm_f64.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_int32]
        lib._spmm_typed = True
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    va = np.ascontiguousarray(values, dtype=np.float64)
    xd = np.ascontiguousarray(x, dtype=np.float64)
    n = rp.size - 1
    z = np.empty((n, xd.shape[1]), dtype=np.float64)
    nt = nthreads or max(1, min(64, os.cpu_count() or 1))
    lib.oracle_spmm_f64(rp.ctypes.data, ci.ctypes.data, va.ctypes.data, n, xd.ctypes.data, xd.shape[1],
                        xd.shape[1], z.ctypes.data, z.shape[1], nt)
    return z


def _loa_c(lib, adj: Csr, vw: int, group_size: int) -> list[list[int]]:
    n = adj.num_rows
    rp = np.ascontiguousarray(adj.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(adj.col_idx, dtype=np.int32)
    order = sort_by_min_neighbor(adj)
    out_order = np.zeros(n, dtype=np.int64)
    ngroups = max(1, -(-n // group_size) + 1)
    gptr = np.zeros(ngroups + 1, dtype=np.int64)
    rc = lib.oracle_loa(rp.ctypes.data, ci.ctypes.data, n, vw, group_size, order.ctypes.data,
                        out_order.ctypes.data, gptr.ctypes.data)
    if rc < 0:
        raise RuntimeError("oracle_loa failed")
    return [out_order[gptr[i]:gptr[i + 1]].tolist() for i in range(rc)]


def induced_perm(groups: list[list[int]], n: int) -> np.ndarray:
    """layout.py:32-41: perm[old_id] = new_id in concatenation order."""
    perm = np.empty(n, dtype=np.int64)
    flat = [v for g in groups for v in g]
    perm[np.asarray(flat, dtype=np.int64)] = np.arange(len(flat), dtype=np.int64)
    return perm


def validate_grouping(groups, n, group_size=WINDOW_HEIGHT) -> None:
    """layout.py:43-61 WindowGrouping.validate."""
    seen = np.zeros(n, dtype=bool)
    total = 0
    for gi, group in enumerate(groups):
        if not 0 < len(group) <= group_size:
            raise ValueError(f"group size must be in 1..{group_size}")
        if len(group) < group_size and gi != len(groups) - 1:
            raise ValueError(f"group {gi} is short but not last")
        for v in group:
            if not 0 <= v < n:
                raise ValueError(f"vertex id {v} out of range")
            if seen[v]:
                raise ValueError(f"vertex {v} appears twice")
            seen[v] = True
        total += len(group)
    if total != n:
        raise ValueError("groups must cover every vertex exactly once")
