"""Host and device matrix types.

Host types mirror the reference's (rowwin matrices.py:24-172: SparseCsr,
DenseMatrix, Graph) so user code constructing them keeps working; every
compute entry point also accepts the reference's own objects (duck-typed on
num_rows/num_cols/row_ptr/col_idx/values).  `DeviceCsr` is the HBM-resident
form the kernels consume: int64 row_ptr, int32 col_idx, fp32 values (plus a
lazily materialised bf16 copy).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import FormatError, InvariantError  # noqa: F401  (re-export, reference names)


@dataclass(frozen=True)
class SparseCsr:
    """Host CSR (reference matrices.py:24-123)."""

    num_rows: int
    num_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def validate(self) -> None:
        """matrices.py:42-62 (vectorised strict-ascending check)."""
        if self.num_rows < 0 or self.num_cols < 0:
            raise ValueError("negative dimensions")
        if self.row_ptr.shape != (self.num_rows + 1,):
            raise ValueError("row_ptr length must be num_rows+1")
        if self.row_ptr[0] != 0:
            raise ValueError("row_ptr must start at 0")
        if np.any(np.diff(self.row_ptr) < 0):
            raise ValueError("row_ptr must be non-decreasing")
        nnz = int(self.row_ptr[-1])
        if self.col_idx.shape != (nnz,) or self.values.shape != (nnz,):
            raise ValueError("col_idx/values length must equal row_ptr[-1]")
        if nnz:
            if self.col_idx.min() < 0 or self.col_idx.max() >= self.num_cols:
                raise ValueError("column index out of range")
            d = np.diff(self.col_idx.astype(np.int64))
            same_row = np.ones(nnz - 1, dtype=bool)
            starts = self.row_ptr[1:-1]
            starts = starts[(starts > 0) & (starts < nnz)]
            same_row[starts - 1] = False
            bad = np.flatnonzero(same_row & (d <= 0))
            if bad.size:
                row = int(np.searchsorted(self.row_ptr, bad[0], side="right") - 1)
                raise ValueError(f"row {row}: column indices not strictly ascending")

    @classmethod
    def from_coo(cls, num_rows, num_cols, rows, cols, vals) -> "SparseCsr":
        """matrices.py:64-97: lexsort by (row, col), duplicates summed."""
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
        if num_rows * max(num_cols, 1) < (1 << 62):
            # one stable key sort == lexsort((cols, rows)) (equal keys keep input order)
            order = np.argsort(rows * max(num_cols, 1) + cols, kind="stable")
        else:
            order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        if rows.size:
            head = np.empty(rows.size, dtype=bool)
            head[0] = True
            head[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
            if head.all():  # no duplicates: np.add.at into zeros is 0.0 + v (maps -0.0 to +0.0)
                vals = vals + 0.0
            else:
                group = np.cumsum(head) - 1
                summed = np.zeros(int(group[-1]) + 1, dtype=np.float64)
                np.add.at(summed, group, vals)
                rows, cols, vals = rows[head], cols[head], summed
        counts = np.bincount(rows, minlength=num_rows) if num_rows else np.zeros(0, np.int64)
        row_ptr = np.zeros(num_rows + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        return cls(num_rows, num_cols, row_ptr, cols, vals)

    def to_coo(self):
        rows = np.repeat(np.arange(self.num_rows, dtype=np.int64), np.diff(self.row_ptr))
        return rows, self.col_idx.copy(), self.values.copy()

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.num_rows, self.num_cols), dtype=np.float64)
        r, c, v = self.to_coo()
        dense[r, c] = v
        return dense

    def row_slice(self, i: int):
        lo, hi = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        return self.col_idx[lo:hi], self.values[lo:hi]

    def is_symmetric(self) -> bool:
        if self.num_rows != self.num_cols:
            return False
        r, c, v = self.to_coo()
        m = SparseCsr.from_coo(self.num_rows, self.num_cols, c, r, v)
        return (np.array_equal(m.row_ptr, self.row_ptr) and np.array_equal(m.col_idx, self.col_idx)
                and np.array_equal(m.values, self.values))


@dataclass(frozen=True)
class DenseMatrix:
    """Row-major dense matrix (reference matrices.py:126-149); `data` may be a numpy
    array (host) or a torch tensor (device)."""

    data: object

    def __post_init__(self):
        d = self.data
        if isinstance(d, torch.Tensor):
            if d.dim() != 2:
                raise ValueError("dense matrix must be 2-dimensional")
            object.__setattr__(self, "data", d.contiguous())
        else:
            arr = np.ascontiguousarray(d)
            if arr.ndim != 2:
                raise ValueError("dense matrix must be 2-dimensional")
            object.__setattr__(self, "data", arr)

    @property
    def rows(self) -> int:
        return int(self.data.shape[0])

    @property
    def dim(self) -> int:
        return int(self.data.shape[1])

    @classmethod
    def random(cls, rows: int, dim: int, seed: int, low: float = -1.0, high: float = 1.0) -> "DenseMatrix":
        rng = np.random.default_rng(seed)
        return cls(rng.uniform(low, high, size=(rows, dim)))


@dataclass(frozen=True)
class Graph:
    """Adjacency wrapper (reference matrices.py:152-172)."""

    num_vertices: int
    adjacency: object
    undirected: bool

    def validate(self) -> None:
        adj = self.adjacency
        if isinstance(adj, DeviceCsr):
            adj = adj.to_host()
        adj.validate()
        if adj.num_rows != self.num_vertices or adj.num_cols != self.num_vertices:
            raise ValueError("adjacency must be num_vertices x num_vertices")
        if self.undirected and not adj.is_symmetric():
            raise ValueError("undirected graph requires a symmetric adjacency")

    def neighbors(self, v: int):
        adj = self.adjacency if not isinstance(self.adjacency, DeviceCsr) else self.adjacency.to_host()
        return adj.row_slice(v)[0]

    def degree(self, v: int) -> int:
        rp = self.adjacency.row_ptr
        return int(rp[v + 1] - rp[v])


def graph_from_edges(num_vertices: int, edges, undirected: bool = True) -> Graph:
    """matrices.py:292-307: unit-valued, deduplicated (u, v) pairs."""
    pairs = set()
    for u, v in edges:
        if u >= num_vertices or v >= num_vertices:
            raise ValueError(f"edge ({u}, {v}) exceeds num_vertices={num_vertices}")
        pairs.add((u, v))
        if undirected:
            pairs.add((v, u))
    if pairs:
        rows, cols = (np.array(a, dtype=np.int64) for a in zip(*sorted(pairs)))
    else:
        rows = cols = np.zeros(0, dtype=np.int64)
    adj = SparseCsr.from_coo(num_vertices, num_vertices, rows, cols, np.ones(rows.size))
    return Graph(num_vertices, adj, undirected)


@dataclass
class DeviceCsr:
    """HBM-resident CSR consumed by the kernels."""

    num_rows: int
    num_cols: int
    row_ptr: torch.Tensor  # int64 [n+1]
    col_idx: torch.Tensor  # int32 [nnz]
    values: torch.Tensor   # float32 [nnz]
    _bf16: torch.Tensor | None = field(default=None, repr=False)
    host_values_f64: np.ndarray | None = field(default=None, repr=False)
    values_f64: torch.Tensor | None = field(default=None, repr=False)  # exact operator values (device)
    symmetric: bool = False  # A == A^T known by construction (e.g. gcn-normalised undirected graph)
    # derived device structures cached per operator (partitions keyed by (height, selector), A^T)
    _derived: dict = field(default_factory=dict, repr=False)

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @property
    def device(self) -> torch.device:
        return self.row_ptr.device

    def values_bf16(self) -> torch.Tensor:
        if self._bf16 is None:
            self._bf16 = self.values.to(torch.bfloat16)
        return self._bf16

    def to_host(self) -> SparseCsr:
        if self.host_values_f64 is not None:
            vals = self.host_values_f64
        elif self.values_f64 is not None:
            vals = self.values_f64.cpu().numpy()
        else:
            vals = self.values.double().cpu().numpy()
        return SparseCsr(self.num_rows, self.num_cols, self.row_ptr.cpu().numpy(),
                         self.col_idx.long().cpu().numpy(), vals)


def to_device_csr(csr, device=None) -> DeviceCsr:
    """Upload a host CSR (ours or the reference's) to the GPU; DeviceCsr passes through."""
    if isinstance(csr, DeviceCsr):
        return csr
    if device is None:
        from ._lib import require_cuda

        device = require_cuda()
    rp = np.asarray(csr.row_ptr, dtype=np.int64)
    ci = np.asarray(csr.col_idx)
    if csr.num_cols >= 2 ** 31 or (ci.size and int(ci.max()) >= 2 ** 31):
        raise ValueError("column ids must fit in int32")
    vals = np.asarray(csr.values, dtype=np.float64)
    return DeviceCsr(
        int(csr.num_rows), int(csr.num_cols),
        torch.from_numpy(rp).to(device),
        torch.from_numpy(ci.astype(np.int32, copy=False)).to(device),
        torch.from_numpy(vals.astype(np.float32)).to(device),
        host_values_f64=vals,
    )


def permute_symmetric(csr, perm):
    """matrices.py:310-318 -- P A P^T; dispatched to the GPU kernel (layout.permute_symmetric)."""
    from .layout import permute_symmetric as _ps

    return _ps(csr, perm)


def _device_csr_host_api(name):
    def f(self, *a, **k):
        return getattr(self.to_host(), name)(*a, **k)
    f.__name__ = name
    return f


for _n in ("to_dense", "to_coo", "is_symmetric", "row_slice", "validate"):
    setattr(DeviceCsr, _n, _device_csr_host_api(_n))
