"""Row windows with column condensation (reference windows.py), computed on the GPU.

`partition(csr)` runs K1 (csrc/partition.cu): per 16-row window the ascending
distinct columns (`nonzero_cols`), the inverse index of every entry
(`cond_cols`), the features (ncols, density, CI) and the default selector's
decision -- all bit-identical to the reference's per-window
np.unique(return_inverse=True) (windows.py:81-106), features (109-123) and
SelectorModel.decide (selector.py:48-56).

The result is a `WindowSet`: structure-of-arrays in HBM that also behaves as
the reference's `list[RowWindow]` (len / iteration / indexing materialise
host `RowWindow` objects lazily), so code written against the reference keeps
working.
"""

from __future__ import annotations

import math
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .matrices import DeviceCsr, to_device_csr

WINDOW_HEIGHT = 16  # windows.py:12
TILE_COLS = 8       # windows.py:13
TILE_DIM = 16       # windows.py:14


@dataclass(frozen=True)
class RowWindow:
    """Host view of one window (reference windows.py:17-69)."""

    window_id: int
    row_start: int
    row_count: int
    nonzero_cols: np.ndarray
    local_ptr: np.ndarray
    cond_cols: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.local_ptr[-1])

    @property
    def ncols(self) -> int:
        return int(self.nonzero_cols.size)

    def row_entries(self, r: int):
        lo, hi = int(self.local_ptr[r]), int(self.local_ptr[r + 1])
        return self.cond_cols[lo:hi], self.values[lo:hi]

    def decondense(self):
        local_rows = np.repeat(np.arange(self.row_count, dtype=np.int64), np.diff(self.local_ptr))
        return local_rows + self.row_start, self.nonzero_cols[self.cond_cols], self.values.copy()

    def validate(self) -> None:
        """windows.py:53-69."""
        if self.row_count <= 0:
            raise ValueError("window must span at least one row")
        if self.local_ptr.shape != (self.row_count + 1,) or self.local_ptr[0] != 0:
            raise ValueError("local_ptr must have row_count+1 entries starting at 0")
        if np.any(np.diff(self.local_ptr) < 0):
            raise ValueError("local_ptr must be non-decreasing")
        if self.nonzero_cols.size > 1 and np.any(np.diff(self.nonzero_cols) <= 0):
            raise ValueError("nonzero_cols must be strictly ascending")
        if self.cond_cols.size:
            if self.cond_cols.min() < 0 or self.cond_cols.max() >= self.ncols:
                raise ValueError("condensed column id out of range")
        if self.nnz and self.ncols == 0:
            raise ValueError("entries present but no nonzero columns recorded")
        if np.unique(self.cond_cols).size != self.ncols:
            raise ValueError("every condensed column must be used by some entry")


@dataclass(frozen=True)
class WindowFeatures:
    """windows.py:72-78."""

    ncols: int
    density: float
    computing_intensity: float


class WindowSet(Sequence):
    """Device-resident windows of one CSR (SoA); a Sequence[RowWindow] on the host side."""

    def __init__(self, csr: DeviceCsr, window_height: int, win_col_ptr: torch.Tensor, nonzero_cols: torch.Tensor,
                 cond_cols: torch.Tensor, density: torch.Tensor, ci: torch.Tensor, codes: torch.Tensor | None,
                 selector: tuple | None):
        self.csr = csr
        self.window_height = int(window_height)
        self.win_col_ptr = win_col_ptr
        self.nonzero_cols = nonzero_cols
        self.cond_cols = cond_cols
        self.density = density
        self.ci = ci
        self.codes = codes          # decisions of `selector` (uint8, 0 scalar / 1 tile)
        self.selector = selector    # the 7 doubles the codes were computed with
        self._host = None
        self._plans = {}

    def assignment(self):
        """The selector's decisions (codes) as an executors.Assignment, made once per WindowSet with
        its host copy and plan key, so per-call users (model.Gcn2's explicit epoch) neither copy the
        codes to the host nor synchronise -- the epoch can be captured in a CUDA graph."""
        a = getattr(self, "_assignment", None)
        if a is None:
            from .executors import Assignment

            a = Assignment(self.codes)
            _ = a.codes  # host copy now, not inside a later call
            self._assignment = a
        return a

    # ---------------------------------------------------------------- sizes
    @property
    def num_windows(self) -> int:
        return int(self.win_col_ptr.numel()) - 1

    @property
    def num_rows(self) -> int:
        return self.csr.num_rows

    def __len__(self) -> int:
        return self.num_windows

    def ncols(self) -> torch.Tensor:
        return self.win_col_ptr[1:] - self.win_col_ptr[:-1]

    def nnz_per_window(self) -> torch.Tensor:
        wh, n = self.window_height, self.csr.num_rows
        W = self.num_windows
        rs = torch.arange(W, device=self.csr.device, dtype=torch.int64) * wh
        re = torch.clamp(rs + wh, max=n)
        return self.csr.row_ptr[re] - self.csr.row_ptr[rs]

    def total_rows(self) -> int:
        return self.csr.num_rows

    # ---------------------------------------------------------------- host views
    def host_arrays(self) -> dict:
        if self._host is None:
            csr = self.csr
            vals = csr.host_values_f64 if csr.host_values_f64 is not None else csr.values.double().cpu().numpy()
            self._host = dict(
                row_ptr=csr.row_ptr.cpu().numpy(),
                win_col_ptr=self.win_col_ptr.cpu().numpy(),
                nonzero_cols=self.nonzero_cols.long().cpu().numpy(),
                cond_cols=self.cond_cols.long().cpu().numpy(),
                values=vals,
            )
        return self._host

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        W = len(self)
        if i < 0:
            i += W
        if not 0 <= i < W:
            raise IndexError("window index out of range")
        h = self.host_arrays()
        wh, n = self.window_height, self.csr.num_rows
        lo = i * wh
        hi = min(lo + wh, n)
        e0, e1 = int(h["row_ptr"][lo]), int(h["row_ptr"][hi])
        c0, c1 = int(h["win_col_ptr"][i]), int(h["win_col_ptr"][i + 1])
        return RowWindow(
            window_id=i, row_start=lo, row_count=hi - lo,
            nonzero_cols=h["nonzero_cols"][c0:c1].copy(),
            local_ptr=(h["row_ptr"][lo:hi + 1] - e0).astype(np.int64),
            cond_cols=h["cond_cols"][e0:e1].copy(),
            values=h["values"][e0:e1].copy(),
        )

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]

    def __eq__(self, other):
        if isinstance(other, list):
            return len(other) == len(self) and all(a == b for a, b in zip(self, other))
        return self is other

    __hash__ = object.__hash__

    def features_host(self):
        """(ncols int64, density f64, ci f64) numpy arrays, bit-exact with windows.py:109-123."""
        return (self.ncols().cpu().numpy(), self.density.cpu().numpy(), self.ci.cpu().numpy())


def _selector_doubles(model) -> tuple:
    return (float(model.w_ncols), float(model.w_density), float(model.bias),
            float(model.feature_means[0]), float(model.feature_means[1]),
            float(model.feature_scales[0]), float(model.feature_scales[1]))


@_lib.nvtx("hcs.partition")
def partition(csr, window_height: int = WINDOW_HEIGHT, model=None) -> WindowSet:
    """GPU K1: windows.py:81-106 partition (+ features + selector decisions).

    `model` defaults to the shipped selector (selector.default_model()); the
    decisions are stored on the WindowSet and reused by classify_windows.
    """
    if window_height <= 0:
        raise ValueError("window_height must be positive")
    from .selector import default_model

    dev = _lib.require_cuda()
    cached = isinstance(csr, DeviceCsr)
    d = to_device_csr(csr, dev)
    n, nnz = d.num_rows, d.nnz
    W = -(-n // window_height)
    sel = _selector_doubles(model if model is not None else default_model())
    key = ("windows", window_height, sel)
    if cached and key in d._derived:  # same device operator: windows are a pure function of it
        return d._derived[key]
    sel_c = (_lib.ctypes.c_double * 7)(*sel)  # host array (read on the host by the ABI)
    ws_bytes = _lib.ctypes.c_size_t(0)
    L = _lib.lib()
    _lib.check(L.hcs_partition_workspace_bytes(n, d.num_cols, nnz, window_height, _lib.ctypes.byref(ws_bytes)))
    ws = torch.empty(max(int(ws_bytes.value), 1), dtype=torch.uint8, device=dev)
    wcp = torch.empty(W + 1, dtype=torch.int64, device=dev)
    dens = torch.empty(W, dtype=torch.float64, device=dev)
    ci = torch.empty(W, dtype=torch.float64, device=dev)
    codes = torch.empty(W, dtype=torch.uint8, device=dev)
    s = _lib.stream()
    _lib.check(L.hcs_partition_count(d.row_ptr.data_ptr(), d.col_idx.data_ptr() if nnz else None, n, d.num_cols, nnz,
                                     window_height, _lib.ctypes.addressof(sel_c), wcp.data_ptr(), dens.data_ptr(), ci.data_ptr(),
                                     codes.data_ptr(), ws.data_ptr(), ws.numel(), s))
    total = int(wcp[-1].item()) if W else 0
    nzc = torch.empty(max(total, 1), dtype=torch.int32, device=dev)[:total]
    cond = torch.empty(nnz, dtype=torch.int32, device=dev)
    if nnz:
        _lib.check(L.hcs_partition_fill(d.row_ptr.data_ptr(), d.col_idx.data_ptr(), n, d.num_cols, nnz, window_height,
                                        wcp.data_ptr(), nzc.data_ptr(), cond.data_ptr(), ws.data_ptr(), ws.numel(), s))
    out = WindowSet(d, window_height, wcp, nzc, cond, dens, ci, codes, sel)
    if cached:
        d._derived[key] = out
    return out


def features(window) -> WindowFeatures:
    """windows.py:109-123 for one host RowWindow."""
    nc = window.ncols
    if nc == 0:
        return WindowFeatures(ncols=0, density=0.0, computing_intensity=0.0)
    nnz = window.nnz
    return WindowFeatures(ncols=nc, density=nnz / (window.row_count * nc), computing_intensity=nnz / nc)


def tile_count(window, tile_cols: int = TILE_COLS) -> int:
    """windows.py:126-128."""
    return math.ceil(window.ncols / tile_cols)


def total_rows(windows) -> int:
    """windows.py:131-136."""
    if isinstance(windows, WindowSet):
        return windows.total_rows()
    if not windows:
        return 0
    last = windows[-1]
    return last.row_start + last.row_count


def as_windowset(windows, window_height: int = WINDOW_HEIGHT) -> WindowSet:
    """Accept a WindowSet, or a host list of RowWindow objects (ours or the reference's):
    the entries are decondensed into a CSR and re-partitioned on the GPU (bit-identical)."""
    if isinstance(windows, WindowSet):
        return windows
    windows = list(windows)
    if not windows:
        raise ValueError("no windows")
    wh = windows[0].row_count if len(windows) > 1 else max(windows[0].row_count, 1)
    for i, w in enumerate(windows[:-1]):
        if w.row_count != wh or w.row_start != i * wh:
            raise ValueError("windows must be consecutive equal-height row windows")
    n_rows = windows[-1].row_start + windows[-1].row_count
    rows, cols, vals = [], [], []
    for w in windows:
        r, c, v = w.decondense()
        rows.append(r); cols.append(c); vals.append(v)
    rows = np.concatenate(rows).astype(np.int64)
    cols = np.concatenate(cols).astype(np.int64)
    vals = np.concatenate(vals).astype(np.float64)
    counts = np.bincount(rows, minlength=n_rows)
    row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    n_cols = int(cols.max()) + 1 if cols.size else 1
    from .matrices import SparseCsr

    return partition(SparseCsr(n_rows, n_cols, row_ptr, cols, vals), window_height=wh)
