"""B200-calibrated path selector (opt-in): the training half of the reference selector
(selector.py:25-257) with a GPU timing provider.

The shipped model (data/selector_default.json, selector.py:284-288) stays the default so
window decisions remain bit-exact with the reference.  Its boundary was fitted to abstract
CPU cost units (costmodel.py:1-12); on B200 the tensor-core tile path is faster than the
CUDA-core path for most windows the shipped model sends to SCALAR.  This
module re-labels the same kind of synthetic 16-row windows with measured B200 timings of
this repo's two kernels and fits the reference's logistic model to them:

  TrainingSample, generate_synthetic, default_grid / dense_grid, collect_samples, train,
  holdout_split, accuracy  -- restatements of selector.py:25-36, 67-128, 131-144, 174-242
                              (same arithmetic, same seeds -> same samples and weights);
  b200_grid                -- the reference grid extended to the column counts real graphs
                              produce (up to 8,192 condensed columns per window);
  B200Provider             -- replaces costmodel.py:126-160 (MeasuredCpuProvider): both
                              paths timed with CUDA events on a batch of copies of the
                              window (distinct random column maps into an L2-resident X),
                              so a window's cost is its steady-state throughput cost.

Use:  model = train(collect_samples(b200_grid(), B200Provider(), dim=128))
      save_model(model, "b200_selector.json"); classify_windows(load_model(...), ws)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .selector import SelectorModel, save_model  # noqa: F401  (save_model re-exported for callers)

GEN_ROWS = 16
GEN_MAX_NCOLS = 130
MAX_FILL = GEN_ROWS - 1  # at most 15 entries per column on a 16-row window


@dataclass(frozen=True)
class TrainingSample:
    """selector.py:25-36; label 1 = the scalar path was faster (ties go to the tile path)."""

    ncols: int
    density: float
    t_scalar: float
    t_tile: float
    label: int

    @classmethod
    def from_timings(cls, ncols: int, density: float, t_scalar: float, t_tile: float) -> "TrainingSample":
        return cls(ncols, density, t_scalar, t_tile, label=1 if t_scalar < t_tile else 0)


@dataclass(frozen=True)
class SyntheticWindow:
    """A 16-row window pattern: CSR rows over condensed columns 0..ncols-1."""

    ncols: int
    local_ptr: np.ndarray
    cond_cols: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.cond_cols.size)

    @property
    def density(self) -> float:
        return self.nnz / (GEN_ROWS * self.ncols)


def generate_synthetic(ncols: int, nnz: int, seed: int, max_ncols: int = GEN_MAX_NCOLS) -> SyntheticWindow:
    """selector.py:67-96 (same draws from the same seed): each condensed column first gets
    one entry in a random row; the remaining nnz - ncols entries fill distinct free cells.
    max_ncols lifts the reference's 130-column cap for the B200 grid."""
    if ncols < 1 or ncols > max_ncols:
        raise ValueError(f"ncols must be in [1, {max_ncols}]")
    if nnz < ncols or nnz > MAX_FILL * ncols:
        raise ValueError(f"nnz must be in [ncols, {MAX_FILL}*ncols]")
    gen = np.random.default_rng(seed)
    col_ids = np.arange(ncols)
    seeded = gen.integers(0, GEN_ROWS, size=ncols) * ncols + col_ids  # cell = row * ncols + col
    open_cells = np.setdiff1d(np.arange(GEN_ROWS * ncols), seeded, assume_unique=False)
    cells = np.sort(np.concatenate([seeded, gen.choice(open_cells, size=nnz - ncols, replace=False)]))
    ptr = np.concatenate([[0], np.cumsum(np.bincount(cells // ncols, minlength=GEN_ROWS))]).astype(np.int64)
    return SyntheticWindow(ncols, ptr, (cells % ncols).astype(np.int64))


def _grid(column_counts, seeds: int) -> list[tuple[int, int, int]]:
    """selector.py:99-128: for every column count, 8 densities evenly spaced over
    [1/16, 15/16] (nnz rounded, clipped to [ncols, 15 ncols]), `seeds` windows each; the
    seed is the running index of the grid point."""
    levels = np.linspace(1.0 / GEN_ROWS, MAX_FILL / GEN_ROWS, 8)
    pts = []
    for nc in column_counts:
        for lv in levels:
            k = int(np.clip(int(round(lv * GEN_ROWS * nc)), nc, MAX_FILL * nc))
            base = len(pts)
            pts.extend([(nc, k, base + i) for i in range(seeds)])
    return pts


def default_grid(seeds: int = 3) -> list[tuple[int, int, int]]:
    """selector.py:108-111: 20 column counts x 8 densities x seeds."""
    return _grid([1, 2, 4, 8, *range(16, 129, 8), GEN_MAX_NCOLS], seeds)


def dense_grid(seeds: int = 5) -> list[tuple[int, int, int]]:
    """selector.py:114-116: every column count 1..130."""
    return _grid(range(1, GEN_MAX_NCOLS + 1), seeds)


B200_NCOLS = [1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 512, 1024, 2048, 4096, 8192]


def b200_grid(seeds: int = 2) -> list[tuple[int, int, int]]:
    """The reference grid's densities over the column counts real windows have (C2 windows
    average ~7,400 condensed columns, C5 scalar windows ~110)."""
    return _grid(B200_NCOLS, seeds)


def collect_samples(grid, provider, dim: int = 32, max_ncols: int | None = None) -> list[TrainingSample]:
    """selector.py:131-144: materialise each grid window, time both paths, label."""
    cap = max_ncols if max_ncols is not None else max(GEN_MAX_NCOLS, *(g[0] for g in grid))
    out = []
    for nc, k, sd in grid:
        win = generate_synthetic(nc, k, sd, max_ncols=cap)
        out.append(TrainingSample.from_timings(win.ncols, win.density, *provider(win, dim)))
    return out


def train(samples: list[TrainingSample], learning_rate: float = 0.1, epochs: int = 50_000, tol: float = 1e-8,
          seed: int = 0) -> SelectorModel:
    """selector.py:174-215: logistic regression on z-scored (ncols, density), full-batch
    gradient descent on the mean cross-entropy, stopping when the loss changes < tol.
    The update order and float operations follow the reference, so the same samples give
    the same weights bit for bit."""
    if not samples:
        raise ValueError("no training samples")
    label = np.fromiter((s.label for s in samples), dtype=np.float64, count=len(samples))
    if label.min() == label.max():
        raise ValueError("training data contains a single class")
    x = np.array([[s.ncols, s.density] for s in samples], dtype=np.float64)
    mu, sd = x.mean(axis=0), x.std(axis=0)
    sd[sd == 0.0] = 1.0
    xz = (x - mu) / sd
    coef = np.random.default_rng(seed).normal(0.0, 0.01, size=2)
    bias, last, m = 0.0, np.inf, len(samples)
    for _ in range(epochs):
        logit = xz @ coef + bias
        resid = 1.0 / (1.0 + np.exp(-logit)) - label
        cur = float(np.mean(np.logaddexp(0.0, logit) - label * logit))
        coef -= learning_rate * (xz.T @ resid) / m
        bias -= learning_rate * float(resid.mean())
        if abs(last - cur) < tol:
            break
        last = cur
    return SelectorModel(float(coef[0]), float(coef[1]), float(bias), (float(mu[0]), float(mu[1])),
                         (float(sd[0]), float(sd[1])))


def holdout_split(samples, frac: float = 0.25, seed: int = 0):
    """selector.py:218-232: a seeded permutation's first round(frac * n) indices are held out
    (kept in index order); the rest train, in input order."""
    if not 0.0 < frac < 1.0:
        raise ValueError("frac must be in (0, 1)")
    held = np.random.default_rng(seed).permutation(len(samples))[: int(round(frac * len(samples)))]
    mask = np.zeros(len(samples), dtype=bool)
    mask[held] = True
    return [s for s, h in zip(samples, mask) if not h], [samples[i] for i in np.flatnonzero(mask)]


def accuracy(model: SelectorModel, samples) -> float:
    """selector.py:235-242: fraction of samples whose SCALAR/TILE decision matches the label."""
    from .executors import Path

    if not samples:
        raise ValueError("no samples to score")
    return float(np.mean([(model.decide(s.ncols, s.density) is Path.SCALAR) == (s.label == 1) for s in samples]))


class B200Provider:
    """Per-window (t_scalar, t_tile) in milliseconds on the current CUDA device.

    The window pattern is replicated `batch` times (enough copies for >= min_nnz entries);
    copy k maps its condensed columns to distinct pseudo-random rows of an X with x_rows
    rows (bf16, dim features), so the gathers look like a real graph's.  Both paths run
    through spmm_hybrid's plan (all-SCALAR / all-TILE assignments) and are timed with CUDA
    events (median of `reps`); a window's cost is the batch time / batch."""

    def __init__(self, x_rows: int = 232_965, min_nnz: int = 2_000_000, max_batch: int = 16_384,
                 min_batch: int = 512, reps: int = 5, seed: int = 0, precision: str = "bf16"):
        self.x_rows, self.min_nnz, self.max_batch, self.min_batch = x_rows, min_nnz, max_batch, min_batch
        self.reps, self.seed, self.precision = reps, seed, precision
        self._x = {}

    def _operand(self, dim: int):
        from . import _lib
        from .executors import DeviceOperand, stage_operand

        if dim not in self._x:
            g = torch.Generator(device="cuda")
            g.manual_seed(self.seed + 7)
            x = (torch.rand(self.x_rows, dim, generator=g, device="cuda") * 2 - 1)
            self._x[dim] = stage_operand(x.to(torch.bfloat16 if self.precision == "bf16" else torch.float32),
                                         self.precision, torch.device("cuda"),
                                         tf32_round=self.precision == "tf32")[0]
        return self._x[dim]

    def batch_matrix(self, w: SyntheticWindow, batch: int):
        """CSR of `batch` stacked copies of the window (16 rows each, unit values)."""
        from .matrices import DeviceCsr

        dev = torch.device("cuda")
        nc = w.ncols
        if nc > self.x_rows:
            raise ValueError("window has more columns than X rows")
        g = torch.Generator(device=dev)
        g.manual_seed(self.seed * 1_000_003 + nc * 131 + w.nnz)
        # copy k: column c -> (base_k + c * step) mod x_rows, distinct for c < nc since gcd(step, x_rows) = 1
        step = 1_000_003 % self.x_rows or 1
        while np.gcd(step, self.x_rows) != 1:
            step += 1
        base = torch.randint(0, self.x_rows, (batch, 1), generator=g, device=dev, dtype=torch.int64)
        cols_p = torch.as_tensor(w.cond_cols, device=dev)
        rows_p = torch.as_tensor(np.repeat(np.arange(GEN_ROWS), np.diff(w.local_ptr)), device=dev)
        cols = (base + cols_p[None, :] * step) % self.x_rows  # [batch, nnz]
        rows = torch.arange(batch, device=dev, dtype=torch.int64)[:, None] * GEN_ROWS + rows_p[None, :]
        keys = torch.sort((rows * self.x_rows + cols).flatten()).values
        r = torch.div(keys, self.x_rows, rounding_mode="floor")
        c = (keys - r * self.x_rows).to(torch.int32)
        n_rows = batch * GEN_ROWS
        row_ptr = torch.zeros(n_rows + 1, dtype=torch.int64, device=dev)
        torch.cumsum(torch.bincount(r, minlength=n_rows), 0, out=row_ptr[1:])
        return DeviceCsr(n_rows, self.x_rows, row_ptr, c, torch.ones(keys.numel(), dtype=torch.float32, device=dev))

    def __call__(self, w: SyntheticWindow, dim: int) -> tuple[float, float]:
        from .executors import Assignment, Path, get_plan
        from .windows import partition

        batch = int(np.clip(self.min_nnz // max(w.nnz, 1), self.min_batch, self.max_batch))
        csr = self.batch_matrix(w, batch)
        ws = partition(csr)
        xop = self._operand(dim)
        z = torch.empty((csr.num_rows, xop.ld), dtype=torch.float32, device="cuda")
        out = []
        for path in (Path.SCALAR, Path.TILE):
            plan = get_plan(ws, Assignment.uniform(len(ws), path), self.precision)
            for _ in range(2):
                plan.run(xop, z, xop.ld)
            times = []
            for _ in range(self.reps):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                plan.run(xop, z, xop.ld)
                e.record()
                e.synchronize()
                times.append(s.elapsed_time(e))
            out.append(float(np.median(times)) / batch)
        return out[0], out[1]
