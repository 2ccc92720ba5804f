"""The UNMODIFIED reference, timed on a window sample -- BENCH INFRASTRUCTURE ONLY.

Imports the reference package `rowwin` from baseline/_ref (installed offline from
/root/reference/pkg with `pip install --no-index --no-deps --target baseline/_ref`, see
DESIGN.md §8; git-ignored, it travels to the GPU box with the snapshot) and times its own
public API on the host cores:

    windows = rowwin.windows.partition(csr)                        (windows.py:81-106)
    asg     = rowwin.selector.classify_windows(default_model(), windows)   (selector.py:63-64)
    rowwin.executors.spmm_hybrid(windows, asg, x, precision="f32", threads=1)   (executors.py:234-251)

Only spmm_hybrid is timed (the GPU arm also excludes preprocessing from GFLOP/s).  threads=1
is the reference's fastest setting: its executor is GIL-bound (threads=8 was
slower), so one call uses one core.  To use every host core the sample -- the stratified
every-73rd window set of SURVEY §8d -- is cut into one interleaved group per CPU and each timed
step runs all groups at once in forked processes (one step = the whole sample once); the
single-process rate is reported beside it.
Windows are row-local (windows.py:90-105): the rows of the sampled windows stacked into one
CSR partition into exactly those windows (a short last window is stacked last).

Used only by bench.py (the cpu_baseline leg and --impl reference).  Never imported by the
product package.
"""

from __future__ import annotations

import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PATH = os.path.join(ROOT, "baseline", "_ref")
STRIDE = 73


def load_reference():
    """The installed reference package, or None when baseline/_ref is absent."""
    if not os.path.isdir(os.path.join(REF_PATH, "rowwin")):
        return None
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import rowwin  # noqa: F401
    import rowwin.executors
    import rowwin.matrices
    import rowwin.selector
    import rowwin.windows

    return rowwin


def host_info() -> dict:
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "numpy": np.__version__}


class ReferenceSample:
    """Reference windows of the sampled rows, split into `groups` interleaved step workloads."""

    def __init__(self, rowwin, row_ptr, col_idx, values, n: int, groups: int, stride: int = STRIDE):
        W = -(-n // 16)
        sample = list(range(0, W, stride))
        self.groups = []
        self.windows_total = 0
        self.nnz_total = 0
        for g in range(groups):
            wids = sample[g::groups]
            if not wids:
                continue
            wids.sort(key=lambda w: (min(16 * w + 16, n) - 16 * w < 16, w))  # a short window goes last
            rows = [np.arange(16 * w, min(16 * w + 16, n)) for w in wids]
            rr = np.concatenate(rows)
            lens = row_ptr[rr + 1] - row_ptr[rr]
            rp = np.zeros(rr.size + 1, dtype=np.int64)
            np.cumsum(lens, out=rp[1:])
            idx = np.concatenate([np.arange(row_ptr[r], row_ptr[r + 1]) for r in rr])
            csr = rowwin.matrices.SparseCsr(int(rr.size), n, rp, col_idx[idx].astype(np.int64),
                                            values[idx].astype(np.float64))
            ws = rowwin.windows.partition(csr)
            asg = rowwin.selector.classify_windows(rowwin.selector.default_model(), ws)
            self.groups.append((ws, asg, int(rp[-1])))
            self.windows_total += len(ws)
            self.nnz_total += int(rp[-1])

    def run_group(self, rowwin, g: int, x) -> tuple[float, int, int]:
        """Times the reference's spmm_hybrid on group g; returns (seconds, nnz, windows)."""
        ws, asg, nnz = self.groups[g % len(self.groups)]
        t0 = time.perf_counter()
        rowwin.executors.spmm_hybrid(ws, asg, x, precision="f32", threads=1)
        return time.perf_counter() - t0, nnz, len(ws)


# ----------------------------------------------------------------------------- parallel timing
_STATE: dict = {}


def _run_one(g: int):
    rowwin, sample, x = _STATE["rowwin"], _STATE["sample"], _STATE["x"]
    return sample.run_group(rowwin, g, x)


def timed_steps(row_ptr, col_idx, values, n: int, x: np.ndarray, steps: int, warmup: int,
                processes: int | None = None) -> dict:
    """Runs the reference's spmm_hybrid on the stratified sample: every step, `processes` forked
    workers (default: every host CPU) each run one group concurrently (all host cores in use,
    threads=1 inside each process, the executor's fastest setting), so one step covers the whole
    sample once.  Returns per-step seconds and GFLOP/s (2 * nnz * dim / t, sampled nnz)."""
    import multiprocessing as mp

    rowwin = load_reference()
    if rowwin is None:
        raise RuntimeError(f"the reference is not installed under {REF_PATH}")
    procs = processes or max(1, os.cpu_count() or 1)
    W = -(-n // 16)
    stride = STRIDE if W >= 4 * STRIDE else 1  # C1 (170 windows): every window
    sample = ReferenceSample(rowwin, row_ptr, col_idx, values, n, groups=procs, stride=stride)
    procs = len(sample.groups)
    xm = rowwin.matrices.DenseMatrix(np.ascontiguousarray(x, dtype=np.float32))
    _STATE.update(rowwin=rowwin, sample=sample, x=xm)
    ctx = mp.get_context("fork")
    per_step = []
    with ctx.Pool(procs) as pool:
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            res = pool.map(_run_one, range(procs))
            wall = time.perf_counter() - t0
            if i >= warmup:
                per_step.append((wall, sum(r[1] for r in res), max(r[0] for r in res)))
    dim = x.shape[1]
    tot_t = sum(p[0] for p in per_step)
    tot_nnz = sum(p[1] for p in per_step)
    # the same window groups once more on one core: the single-threaded reference rate
    t1, nnz1, win1 = sample.run_group(rowwin, 0, xm)
    return {"gflops": 2.0 * tot_nnz * dim / tot_t / 1e9, "ms_per_step": tot_t / max(len(per_step), 1) * 1e3,
            "windows_per_step": sample.windows_total, "nnz_per_step": sample.nnz_total, "stride": stride,
            "processes": procs, "steps": len(per_step),
            "single_core_gflops": 2.0 * nnz1 * dim / t1 / 1e9, "single_core_sample": f"{win1} windows, {nnz1} nnz",
            **host_info()}
