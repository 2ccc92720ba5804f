"""Hybrid SpMM executors (reference executors.py) on the B200.

  spmm_scalar  -> K3 CUDA-core warp-per-row kernel over every row (executors.py:191-213)
  spmm_tile    -> K4 tcgen05 tile kernel over every non-empty window (216-231)
  spmm_hybrid  -> K2 plan + K4 for TILE windows + K3 for SCALAR windows (234-251)
  spmm_auto    -> K1 partition/select, then spmm_hybrid (263-272)

Precision: "bf16" (bf16 X and A values, fp32 accumulate; default) or "tf32"
(fp32 X and values, tf32 tensor-core inputs rounded to nearest, fp32 scalar
path).  The reference's "f64"/"f32" host precisions are rejected (no CPU path).
Outputs are fp32.  `threads` is accepted for signature compatibility and ignored.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .matrices import DenseMatrix, DeviceCsr, to_device_csr

_PRECISIONS = ("bf16", "tf32")
TILE_CHUNK = 64  # condensed columns per tensor-core K step group


class Path(Enum):
    """executors.py:23-25."""

    SCALAR = "scalar"
    TILE = "tile"


class Assignment:
    """Per-window path codes, 0 = scalar, 1 = tile (executors.py:28-57).

    Holds host codes (numpy uint8) and/or a device copy; each is materialised on demand.
    """

    def __init__(self, codes):
        if isinstance(codes, torch.Tensor):
            self._dev = codes.to(torch.uint8)
            self._host = None
        else:
            c = np.asarray(codes, dtype=np.uint8)
            if c.ndim != 1 or (c.size and c.max() > 1):
                raise ValueError("assignment codes must be a 1-D array of 0/1")
            self._host = c
            self._dev = None

    @classmethod
    def from_device(cls, codes: torch.Tensor) -> "Assignment":
        return cls(codes)

    @property
    def codes(self) -> np.ndarray:
        if self._host is None:
            self._host = self._dev.cpu().numpy()
        return self._host

    def device_codes(self, device) -> torch.Tensor:
        if self._dev is None or self._dev.device != device:
            self._dev = torch.from_numpy(self.codes).to(device)
        return self._dev

    def __len__(self) -> int:
        return int(self._dev.numel()) if self._dev is not None else int(self._host.size)

    def path(self, window_id: int) -> Path:
        return Path.TILE if self.codes[window_id] else Path.SCALAR

    def count(self, path: Path) -> int:
        tiles = int(self.codes.sum())
        return tiles if path is Path.TILE else len(self) - tiles

    @classmethod
    def from_paths(cls, paths) -> "Assignment":
        return cls(np.array([1 if p is Path.TILE else 0 for p in paths], dtype=np.uint8))

    @classmethod
    def uniform(cls, n: int, path: Path) -> "Assignment":
        return cls(np.full(n, 1 if path is Path.TILE else 0, dtype=np.uint8))

    def __eq__(self, other):
        return isinstance(other, Assignment) and np.array_equal(self.codes, other.codes)

    __hash__ = object.__hash__


@dataclass
class ExecStats:
    """executors.py:60-84."""

    windows_scalar: int = 0
    windows_tile: int = 0
    entries_scalar: int = 0
    entries_tile: int = 0
    tiles_processed: int = 0

    def merge(self, other: "ExecStats") -> None:
        self.windows_scalar += other.windows_scalar
        self.windows_tile += other.windows_tile
        self.entries_scalar += other.entries_scalar
        self.entries_tile += other.entries_tile
        self.tiles_processed += other.tiles_processed

    def as_dict(self) -> dict:
        return {"windows_scalar": self.windows_scalar, "windows_tile": self.windows_tile,
                "entries_scalar": self.entries_scalar, "entries_tile": self.entries_tile,
                "tiles_processed": self.tiles_processed}


@dataclass(frozen=True)
class SpmmResult:
    """executors.py:87-90."""

    z: DenseMatrix
    stats: ExecStats


def _resolve_precision(precision: str) -> str:
    if precision not in _PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(_PRECISIONS)}, got {precision!r}")
    return precision


# --------------------------------------------------------------------------- operands
def _round_up(v: int, m: int) -> int:
    return -(-v // m) * m


class DeviceOperand:
    """X staged for the kernels: compute dtype, rows padded to a 16-byte multiple."""

    def __init__(self, t: torch.Tensor, dim: int, ld: int, dtype_code: int):
        self.t, self.dim, self.ld, self.dtype_code = t, dim, ld, dtype_code

    @property
    def rows(self) -> int:
        return int(self.t.shape[0])


# Pad X rows to whole gather slices (32 / 64 bf16 features, 32 fp32) whenever the feature width is
# not a multiple of the slice, even when no padding would otherwise be needed: unpadded 48-B rows
# (N = 24) straddle sectors and lines and took the tile kernel from 0.79 to 1.22 ms
# (tools/exp_tile_dims.py).
PAD_TO_SLICE = True


def stage_operand(x, precision: str, device, tf32_round: bool = False) -> tuple[DeviceOperand, bool]:
    """Returns (operand, was_host).  Host numpy / DenseMatrix inputs are copied to HBM."""
    data = x.data if isinstance(x, DenseMatrix) else x
    was_host = (not isinstance(data, torch.Tensor)) or data.device.type == "cpu"
    t = data if isinstance(data, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(data))
    if t.dim() != 2:
        raise ValueError("dense matrix must be 2-dimensional")
    rows, dim = int(t.shape[0]), int(t.shape[1])
    if precision == "bf16":
        want, elems, code = torch.bfloat16, 8, _lib.DTYPE_BF16
    else:
        want, elems, code = torch.float32, 4, _lib.DTYPE_F32
    ld = max(_round_up(dim, elems), elems)
    slice_elems = (32 if dim <= 32 else 64) if want == torch.bfloat16 else 32
    if PAD_TO_SLICE and dim % slice_elems:
        ld = _round_up(dim, slice_elems)  # whole gather slices per row (see below)
    direct = (not was_host and t.device == device and t.dtype == want and t.is_contiguous() and ld == dim
              and t.data_ptr() % 16 == 0 and not tf32_round)
    if direct:
        return DeviceOperand(t, dim, ld, code), was_host
    if ld != dim:
        # a padded copy is made anyway: pad rows to whole gather slices (64 or 128 B for bf16,
        # 128 B for fp32) so every gathered row slice starts on a cache-line boundary (C3's
        # 41-wide gradient: 96-B rows straddle lines; the fused backward took 1.52 ms)
        ld = _round_up(dim, slice_elems)
    if (was_host and t.dtype == torch.float64 and rows * dim >= HOST_STAGE_MIN_ELEMS and dim
            and t.stride(1) == 1):
        # the drop-in operand (a reference DenseMatrix: float64, pageable): converted on the host
        # cores straight into pinned blocks of the compute dtype, each block's H2D copy overlapping
        # the conversion of the next (csrc/host_stage.cu)
        return DeviceOperand(_stage_host_f64(t, rows, dim, ld, want, device, tf32_round), dim, ld, code), was_host
    if was_host and t.dtype == want and ld == dim and t.is_contiguous() and not tf32_round:
        # host operand already in the compute dtype: one (async when pinned) H2D copy
        buf = torch.empty((rows, ld), dtype=want, device=device)
        buf.copy_(t, non_blocking=True)
        return DeviceOperand(buf, dim, ld, code), was_host
    if ld == dim and not tf32_round:  # no padding: one conversion copy, no zero fill
        buf = torch.empty((rows, ld), dtype=want, device=device)
        buf.copy_(t, non_blocking=True)
        return DeviceOperand(buf, dim, ld, code), was_host
    buf = torch.zeros((rows, ld), dtype=want, device=device)
    if rows and dim:
        src = t.to(device=device, non_blocking=True)
        if tf32_round:
            src32 = src.to(torch.float32).contiguous()
            tmp = torch.empty_like(src32)
            _lib.call("hcs_convert", src32.data_ptr(), tmp.data_ptr(), src32.numel(), 0, _lib.stream())
            buf[:, :dim] = tmp
        else:
            buf[:, :dim] = src.to(want)
    return DeviceOperand(buf, dim, ld, code), was_host


HOST_STAGE_MIN_ELEMS = 1 << 20   # float64 host operands from 8 MB take the pipelined staging path
HOST_STAGE_BLOCK_BYTES = 16 << 20  # bytes (compute dtype) per staged block
HOST_STAGE_THREADS = None         # None: every CPU this process may run on
_STAGE_RINGS: dict = {}


class _StageRing:
    """Two pinned staging blocks per device, reused across calls; `busy[i]` is the event of the
    last H2D copy out of block i (it must complete before the block is rewritten)."""

    def __init__(self, nbytes: int):
        self.blocks = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.busy = [None, None]


def _stage_host_f64(t: torch.Tensor, rows: int, dim: int, ld: int, want, device, tf32_round: bool) -> torch.Tensor:
    import os

    elem = 2 if want == torch.bfloat16 else 4
    out_code = _lib.DTYPE_BF16 if want == torch.bfloat16 else _lib.DTYPE_F32
    block_rows = max(1, HOST_STAGE_BLOCK_BYTES // (ld * elem))
    nbytes = block_rows * ld * elem
    ring = _STAGE_RINGS.get(device)
    if ring is None or ring.blocks[0].numel() < nbytes:
        if ring is not None:
            for ev in ring.busy:
                if ev is not None:
                    ev.synchronize()
        ring = _STAGE_RINGS[device] = _StageRing(nbytes)
    h2d = _H2D_STREAMS.get(device)
    if h2d is None:
        h2d = _H2D_STREAMS[device] = torch.cuda.Stream(device=device)
    cur = torch.cuda.current_stream(device)
    buf = torch.empty((rows, ld), dtype=want, device=device)
    h2d.wait_stream(cur)  # buf's memory may still be in use by earlier work on this stream
    threads = HOST_STAGE_THREADS or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                                     else (os.cpu_count() or 1))
    src = t.data_ptr()
    ld_src = t.stride(0)
    for i, r0 in enumerate(range(0, rows, block_rows)):
        r1 = min(rows, r0 + block_rows)
        slot = i & 1
        if ring.busy[slot] is not None:
            ring.busy[slot].synchronize()
        blk = ring.blocks[slot][: (r1 - r0) * ld * elem].view(want).view(r1 - r0, ld)
        _lib.call("hcs_host_convert_f64", src + r0 * ld_src * 8, r1 - r0, dim, ld_src, blk.data_ptr(), ld, out_code,
                  threads)
        with torch.cuda.stream(h2d):
            buf[r0:r1].copy_(blk, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
        ring.busy[slot] = ev
    cur.wait_stream(h2d)
    if tf32_round:  # tf32 tensor-core inputs: RNA-rounded on the device
        rnd = torch.empty_like(buf)
        _lib.call("hcs_convert", buf.data_ptr(), rnd.data_ptr(), buf.numel(), 0, _lib.stream())
        return rnd
    return buf


# --------------------------------------------------------------------------- hybrid plan
class HybridPlan:
    """K2 execution plan for (windows, assignment, precision): TILE window list with
    packed 64-column chunks, SCALAR/empty window list, and the ExecStats."""

    @_lib.nvtx("hcs.tile_plan")
    def __init__(self, windows, codes: torch.Tensor, precision: str):
        dev = windows.csr.device
        self.windows = windows
        self.precision = precision
        csr = windows.csr
        nnz_w = windows.nnz_per_window()
        ncols = windows.ncols()
        tile_mask = (codes.to(torch.bool)) & (nnz_w > 0)
        self.tile_list = torch.nonzero(tile_mask).flatten().to(torch.int32)
        self.scalar_list = torch.nonzero(~tile_mask).flatten().to(torch.int32)
        nc_t = ncols[self.tile_list.long()]
        chunks = (nc_t + TILE_CHUNK - 1) // TILE_CHUNK
        self.chunk_ptr = torch.zeros(self.tile_list.numel() + 1, dtype=torch.int64, device=dev)
        torch.cumsum(chunks, 0, out=self.chunk_ptr[1:])
        scal_live = (~codes.to(torch.bool)) & (nnz_w > 0)
        tot = torch.stack([
            scal_live.sum(), tile_mask.sum(), nnz_w[scal_live].sum(), nnz_w[tile_mask].sum(),
            ((nc_t + 7) // 8).sum(), self.chunk_ptr[-1]]).cpu().tolist()
        self.stats = ExecStats(int(tot[0]), int(tot[1]), int(tot[2]), int(tot[3]), int(tot[4]))
        self.nchunks = int(tot[5])
        self.chunk_ptr_host = self.chunk_ptr.cpu().numpy()
        self.n_tile = int(self.tile_list.numel())
        self.nnz_tile = int(tot[3])
        ent_dtype = _lib.DTYPE_BF16 if precision == "bf16" else _lib.DTYPE_F32
        self.ent_dtype = ent_dtype
        self.gidx = torch.empty(max(self.nchunks * TILE_CHUNK, 1), dtype=torch.int32, device=dev)
        self.ent_ptr = torch.zeros(self.nchunks + 1, dtype=torch.int64, device=dev)
        ent_words = self.nnz_tile if ent_dtype == _lib.DTYPE_BF16 else 2 * self.nnz_tile
        # +8 words: the tile kernel stages entries with 16-byte aligned bulk copies
        self.ent = torch.zeros(max(ent_words, 1) + 8, dtype=torch.int32, device=dev)
        if self.n_tile:
            wsb = _lib.ctypes.c_size_t(0)
            _lib.check(_lib.lib().hcs_tile_plan_workspace_bytes(self.nnz_tile, self.nchunks, _lib.ctypes.byref(wsb)))
            ws = torch.empty(max(int(wsb.value), 1), dtype=torch.uint8, device=dev)
            _lib.call("hcs_tile_plan", csr.row_ptr.data_ptr(), windows.cond_cols.data_ptr(), csr.values.data_ptr(),
                      _lib.DTYPE_F32, windows.win_col_ptr.data_ptr(), windows.nonzero_cols.data_ptr(), csr.num_rows,
                      csr.num_cols, windows.window_height, self.tile_list.data_ptr(), self.n_tile,
                      self.chunk_ptr.data_ptr(), self.nchunks, self.gidx.data_ptr(), self.ent_ptr.data_ptr(),
                      self.ent.data_ptr(), ent_dtype, self.nnz_tile, ws.data_ptr(), ws.numel(), _lib.stream())
            del ws
        # skewed plans (a chunk with more entries than the kernel holds in registers: hub windows,
        # e.g. R-MAT) run with cost-weighted warp ranges (hcs_spmm_tile_balanced; C5 tile launch
        # 28.7 -> 27.9 ms at alpha 256, tools/exp_tile_alpha.py); balanced plans keep equal chunk
        # counts (C2: the weighted split only adds its bounds launch)
        self.tile_alpha = 0
        if self.n_tile and precision == "bf16" and self.nchunks:
            if int((self.ent_ptr[1:] - self.ent_ptr[:-1]).max().item()) > TILE_DENSE_CHUNK:
                self.tile_alpha = TILE_BALANCE_ALPHA
        if precision == "bf16":
            self.scalar_vals, self.scalar_vals_code = csr.values_bf16(), _lib.DTYPE_BF16
        else:
            self.scalar_vals, self.scalar_vals_code = csr.values, _lib.DTYPE_F32

    def range_chunks(self, t0: int, t1: int) -> int:
        """64-column chunks of tile windows [t0, t1) (host copy of chunk_ptr made with the plan, so
        no sync inside a captured graph): the tile launch sizes its grid to them."""
        cp = self.chunk_ptr_host
        return int(cp[t1] - cp[t0])

    @property
    def _cache(self) -> dict:
        if getattr(self, "_cache_d", None) is None:
            self._cache_d = {}
        return self._cache_d

    def new_scratch(self) -> torch.Tensor:
        """A fresh workspace for the tile kernel's split windows: completion counters (zero
        when first used; the kernels leave them zero) and partial-sum slots (include/hcspmm.h: a
        workspace must not be shared by launches that may run concurrently)."""
        n = _lib.ctypes.c_int64(0)
        _lib.check(_lib.lib().hcs_tile_scratch_floats(_lib.ctypes.byref(n)))
        return torch.zeros(max(int(n.value), 1), dtype=torch.float32, device=self.tile_list.device)

    def scratch(self, stream: int | None = None) -> torch.Tensor:
        """Partial-sum slots of the tile kernel, one buffer per CUDA stream: launches on one
        stream are ordered, so they may share it; launches on different streams (side streams,
        a replayed SpmmGraph -- which owns its own buffer -- next to eager calls) never do."""
        key = _lib.stream() if stream is None else int(stream)
        bufs = self.__dict__.setdefault("_scratch_by_stream", {})
        buf = bufs.get(key)
        if buf is None:
            buf = bufs[key] = self.new_scratch()
        return buf

    def scalar_pieces(self):
        """Small plans: the SCALAR windows' rows cut into <= 32-entry pieces (build_scalar_pieces)."""
        if "pieces" not in self._cache:
            self._cache["pieces"] = build_scalar_pieces(self.windows.csr, self.scalar_list,
                                                        self.windows.window_height)
        return self._cache["pieces"]

    def _run_scalar_pieces(self, xop, z, ldz, s0: int, s1: int, stream: int) -> None:
        run_scalar_pieces(self.windows.csr, self.scalar_vals, self.scalar_vals_code, self.scalar_pieces(), self._cache,
                          xop, z, ldz, s0, s1, stream)

    def launches_per_run(self, dim: int) -> int:
        """Kernels of one run(): the tile kernel (split windows finished in-kernel) plus the
        scalar kernel."""
        return (1 if self.n_tile else 0) + (1 if self.scalar_list.numel() else 0)

    def parts(self, k: int) -> list[tuple[int, int, int, int, int, int]]:
        """k contiguous window ranges of ~equal nnz: (w0, w1, tile t0, t1, scalar s0, s1) each."""
        key = ("parts", k)
        if key not in self._cache:
            ws = self.windows
            W, wh, n = len(ws), ws.window_height, ws.num_rows
            rp = ws.csr.row_ptr
            starts = rp[torch.clamp(torch.arange(W + 1, device=rp.device) * wh, max=n)].cpu().numpy()
            targets = (np.arange(1, k) * int(starts[-1])) // k
            bounds = [0] + [int(v) for v in np.searchsorted(starts, targets, side="left")] + [W]
            self._cache[key] = self.parts_from_bounds(bounds)
        return self._cache[key]

    def parts_from_bounds(self, bounds) -> list[tuple[int, int, int, int, int, int]]:
        """Window bounds b_0 <= ... <= b_k -> parts (w0, w1, t0, t1, s0, s1) for run(part=...)."""
        if "lists_host" not in self._cache:
            self._cache["lists_host"] = (self.tile_list.cpu().numpy(), self.scalar_list.cpu().numpy())
        tl, sl = self._cache["lists_host"]
        out = []
        for i in range(len(bounds) - 1):
            w0, w1 = int(bounds[i]), max(int(bounds[i]), int(bounds[i + 1]))
            out.append((w0, w1, int(np.searchsorted(tl, w0)), int(np.searchsorted(tl, w1)),
                        int(np.searchsorted(sl, w0)), int(np.searchsorted(sl, w1))))
        return out

    @_lib.nvtx("hcs.spmm")
    def run(self, xop: DeviceOperand, z: torch.Tensor, ldz: int, stream=None, tile_events=None, part=None,
            scratch: torch.Tensor | None = None) -> None:
        """Launch K4 (tile windows) then K3 (scalar + empty windows) on the current stream.
        tile_events: optional (start, end) torch.cuda.Event pair recorded around K4.
        part: optional (w0, w1, t0, t1, s0, s1) from parts(): only windows [w0, w1).
        scratch: the tile kernel's partial-sum buffer (default: this stream's, see scratch())."""
        csr = self.windows.csr
        s = _lib.stream() if stream is None else stream
        t0, t1 = (0, self.n_tile) if part is None else part[2:4]
        s0, s1 = (0, int(self.scalar_list.numel())) if part is None else part[4:6]
        # small hybrid plans are latency-bound: K3 runs on a side stream next to K4 (forked and
        # joined on the current stream, so a CUDA-graph capture gets two parallel branches)
        fork = (stream is None and tile_events is None and t1 > t0 and s1 > s0
                and len(self.windows) <= CONCURRENT_MAX_WINDOWS)
        pieces = s1 > s0 and int(self.scalar_list.numel()) <= SCALAR_PIECES_MAX_WINDOWS and _scalar_variant_auto()
        if fork:
            cur = torch.cuda.current_stream(csr.device)
            side = _side_stream(csr.device, cur)
        ss = side.cuda_stream if fork else s
        if pieces:  # first use allocates and zero-fills on the current stream: before the fork point
            pieces_workspace(self._cache, self.scalar_pieces(), ss, xop.dim, csr.device)
        if fork:
            side.wait_stream(cur)
        if tile_events is not None:
            tile_events[0].record()
        if t1 > t0:
            if scratch is None:
                scratch = self.scratch(s)
            _lib.call("hcs_spmm_tile_balanced", self.tile_list.data_ptr() + 4 * t0, t1 - t0,
                      self.chunk_ptr.data_ptr() + 8 * t0, self.gidx.data_ptr(), self.ent_ptr.data_ptr(),
                      self.ent.data_ptr(), self.ent_dtype, csr.num_rows, self.windows.window_height, xop.t.data_ptr(),
                      xop.dtype_code, xop.rows, xop.dim, xop.ld, z.data_ptr(), ldz, scratch.data_ptr(),
                      scratch.numel() * 4, self.tile_alpha, self.range_chunks(t0, t1), s)
        if tile_events is not None:
            tile_events[1].record()
        if s1 > s0:
            if pieces:
                self._run_scalar_pieces(xop, z, ldz, s0, s1, ss)
            else:
                _lib.call("hcs_spmm_scalar", csr.row_ptr.data_ptr(), csr.col_idx.data_ptr(),
                          self.scalar_vals.data_ptr(), self.scalar_vals_code, csr.num_rows, self.windows.window_height,
                          self.scalar_list.data_ptr() + 4 * s0, s1 - s0, xop.t.data_ptr(), xop.dtype_code,
                          xop.rows, xop.dim, xop.ld, z.data_ptr(), ldz, ss)
        if fork:
            cur.wait_stream(side)


CONCURRENT_MAX_WINDOWS = 8192
TILE_DENSE_CHUNK = 128   # entries the tile kernel holds in registers per chunk (kWarpEntRegs x 32)
TILE_BALANCE_ALPHA = 256  # cost of one chunk in entries for the weighted split (tools/exp_tile_alpha.py)
SCALAR_PIECES_MAX_WINDOWS = 1024  # scalar lists up to this length run hcs_spmm_scalar_pieces
_SIDE_STREAMS: dict = {}


def _side_stream(dev, cur: torch.cuda.Stream) -> torch.cuda.Stream:
    """One side stream per (device, caller stream): products issued from different streams or
    threads (or one of them being captured into a CUDA graph) never share a side stream."""
    key = (dev, cur.cuda_stream)
    st = _SIDE_STREAMS.get(key)
    if st is None:
        st = _SIDE_STREAMS[key] = torch.cuda.Stream(device=dev)
    return st


def build_scalar_pieces(csr, win_list: torch.Tensor, wh: int):
    """Every row of the listed windows cut into pieces of <= 32 entries, in list order, for
    hcs_spmm_scalar_pieces (one warp per piece; a hub row's pieces are summed in piece order by the
    last to finish).  Returns (p_row i32, p_k i64 [P, 2], p_first i32, p_count i32, window -> first
    piece as host int64 [len + 1])."""
    dev = csr.device
    sl = win_list.to(torch.int64)
    rows = sl[:, None] * wh + torch.arange(wh, device=dev)[None, :]
    valid = rows < csr.num_rows
    nrow_w = valid.sum(1)
    rows = rows[valid]
    k0, k1 = csr.row_ptr[rows], csr.row_ptr[rows + 1]
    npc = torch.clamp((k1 - k0 + 31) // 32, min=1)
    first = torch.cumsum(npc, 0) - npc
    r_of = torch.repeat_interleave(torch.arange(rows.numel(), device=dev), npc)
    q = torch.arange(r_of.numel(), device=dev) - first[r_of]
    pk0 = k0[r_of] + 32 * q
    pk = torch.stack([pk0, torch.minimum(pk0 + 32, k1[r_of])], 1).contiguous()
    row_first = torch.zeros(nrow_w.numel() + 1, dtype=torch.int64, device=dev)
    torch.cumsum(nrow_w, 0, out=row_first[1:])
    pc_ptr = torch.zeros(rows.numel() + 1, dtype=torch.int64, device=dev)
    torch.cumsum(npc, 0, out=pc_ptr[1:])
    return (rows[r_of].to(torch.int32), pk, first[r_of].to(torch.int32), npc[r_of].to(torch.int32),
            pc_ptr[row_first].cpu().numpy())


def pieces_workspace(cache: dict, pieces, stream: int, dim: int, device):
    """The (slots, counters) workspace of hcs_spmm_scalar_pieces for launches on `stream`, cached
    per (stream, row width).  A new one is allocated and its counters zero-filled on the CURRENT
    torch stream: a caller launching on another stream must order that stream after this call
    (HybridPlan.run creates it before its fork point); the kernel leaves the counters zero."""
    ld_slot = _round_up(dim, 4)
    wkey = ("pieces_ws", stream, ld_slot)
    ws = cache.get(wkey)
    if ws is None:
        P = max(int(pieces[0].numel()), 1)
        ws = cache[wkey] = (torch.empty((P, ld_slot), dtype=torch.float32, device=device),
                            torch.zeros(P, dtype=torch.int32, device=device), ld_slot)
    return ws


def run_scalar_pieces(csr, vals, vals_code, pieces, cache: dict, xop, z, ldz, s0: int, s1: int, stream: int) -> None:
    """Launch hcs_spmm_scalar_pieces for windows [s0, s1) of the piece list (see pieces_workspace)."""
    p_row, p_k, p_first, p_count, win_piece = pieces
    q0, q1 = int(win_piece[s0]), int(win_piece[s1])
    if q1 <= q0:
        return
    slots, cnt, ld_slot = pieces_workspace(cache, pieces, stream, xop.dim, z.device)
    _lib.call("hcs_spmm_scalar_pieces", csr.col_idx.data_ptr(), vals.data_ptr(), vals_code,
              p_row.data_ptr() + 4 * q0, p_k.data_ptr() + 16 * q0, p_first.data_ptr() + 4 * q0,
              p_count.data_ptr() + 4 * q0, q1 - q0, xop.t.data_ptr(), xop.dtype_code, xop.dim, xop.ld, z.data_ptr(),
              ldz, slots.data_ptr(), ld_slot, cnt.data_ptr(), stream)


def get_plan(windows, assignment: Assignment, precision: str) -> HybridPlan:
    """Plans are cached per WindowSet, keyed by the assignment's code CONTENT."""
    import hashlib

    dev = windows.csr.device
    h = getattr(assignment, "_sha1", None)
    if h is None:  # one host copy + hash per Assignment object
        h = assignment._sha1 = hashlib.sha1(assignment.codes.tobytes()).hexdigest()
    key = (precision, h)
    plan = windows._plans.get(key)
    if plan is None:
        plan = HybridPlan(windows, assignment.device_codes(dev), precision)
        windows._plans[key] = plan
    return plan


def _check_window_bounds(windows, x_rows: int) -> None:
    """executors.py:254-260: first window whose largest column is >= X rows.  The largest
    referenced column is computed once per WindowSet (one device sync), so repeated calls
    on the same windows add no device round trip."""
    max_col = getattr(windows, "_max_col", None)
    if max_col is None:
        if windows.nonzero_cols.numel() == 0:  # no entries at all
            max_col = -1
        else:
            live = windows.ncols() > 0
            last = windows.nonzero_cols[(windows.win_col_ptr[1:] - 1).clamp(min=0)].to(torch.int64)
            max_col = int(torch.where(live, last, torch.full_like(last, -1)).max().item())
        windows._max_col = max_col
    if max_col < x_rows:
        return
    live = windows.ncols() > 0
    last = windows.nonzero_cols[(windows.win_col_ptr[1:] - 1).clamp(min=0)].to(torch.int64)
    w = int(torch.nonzero(live & (last >= x_rows))[0].item())
    raise ValueError(f"window {w} references column {int(last[w].item())} but X has {x_rows} rows")


def _host_kind(x):
    data = x.data if isinstance(x, DenseMatrix) else x
    return "torch" if isinstance(data, torch.Tensor) else True


def _alloc_z(rows: int, dim: int, device) -> tuple[torch.Tensor, int]:
    ldz = max(_round_up(dim, 4), 4)
    return torch.empty((rows, ldz), dtype=torch.float32, device=device), ldz


def _wrap_result(z: torch.Tensor, dim: int, was_host, stats: ExecStats) -> SpmmResult:
    """Host inputs give host outputs (numpy for numpy/DenseMatrix input, a CPU tensor
    for a CPU tensor input), device inputs give device outputs."""
    out = z[:, :dim]
    if was_host:
        # D2H into pinned memory (torch's caching host allocator reuses the buffer)
        host = torch.empty(tuple(out.shape), dtype=out.dtype, pin_memory=True)
        host.copy_(out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return SpmmResult(DenseMatrix(host if was_host == "torch" else host.numpy()), stats)
    return SpmmResult(DenseMatrix(out if out.is_contiguous() else out.contiguous()), stats)


@_lib.nvtx("hcs.spmm_hybrid")
def spmm_hybrid(windows, assignment: Assignment, x, precision: str = "bf16", threads: int = 1,
                tile_cols: int = 8, dim_tile: int = 16) -> SpmmResult:
    """executors.py:234-251: TILE windows on tensor cores, SCALAR windows on CUDA cores."""
    from .windows import as_windowset

    if len(assignment) != len(windows):
        raise ValueError(f"assignment covers {len(assignment)} windows, expected {len(windows)}")
    precision = _resolve_precision(precision)
    ws = as_windowset(windows)
    xrows = x.rows if isinstance(x, DenseMatrix) else int(x.shape[0])
    _check_window_bounds(ws, xrows)
    dev = ws.csr.device
    plan = get_plan(ws, assignment, precision)
    xop, was_host = stage_operand(x, precision, dev, tf32_round=(precision == "tf32" and plan.n_tile > 0))
    z, ldz = _alloc_z(ws.num_rows, xop.dim, dev)
    if was_host and len(ws) >= HOST_PIPELINE_MIN_WINDOWS:
        return _run_host_pipelined(plan, xop, z, ldz, _host_kind(x), ExecStats(**plan.stats.as_dict()))
    plan.run(xop, z, ldz)
    return _wrap_result(z, xop.dim, _host_kind(x) if was_host else False, ExecStats(**plan.stats.as_dict()))


def spmm_staged(windows, assignment: Assignment, xop: DeviceOperand, precision: str = "bf16") -> torch.Tensor:
    """spmm_hybrid for an operand already staged on the device in the compute dtype (rows padded
    to whole gather slices, e.g. written by hcs_gemm_bf16 or hcs_softmax_xent): returns the fp32
    device product as a [rows, dim] view (model.Gcn2's explicit epoch)."""
    from .windows import as_windowset

    precision = _resolve_precision(precision)
    want = _lib.DTYPE_BF16 if precision == "bf16" else _lib.DTYPE_F32
    if xop.dtype_code != want:
        raise ValueError(f"operand dtype code {xop.dtype_code} does not match precision {precision!r}")
    if len(assignment) != len(windows):
        raise ValueError(f"assignment covers {len(assignment)} windows, expected {len(windows)}")
    ws = as_windowset(windows)
    _check_window_bounds(ws, xop.rows)
    plan = get_plan(ws, assignment, precision)
    z, ldz = _alloc_z(ws.num_rows, xop.dim, ws.csr.device)
    plan.run(xop, z, ldz)
    return z[:, :xop.dim]


HOST_PIPELINE_MIN_WINDOWS = 4096
HOST_PIPELINE_PARTS = 8  # measured on C2 (tools/exp_e2e_parts.py): 4 -> 4.36 ms, 8 -> 4.18, 16 -> 4.18, 32 -> 4.48
_COPY_STREAMS: dict = {}
# spmm_hybrid_async: requests overlap each other, so fewer, larger launches win (C2 N=128, two in
# flight, tools/exp_e2e_async.py PARTS_SWEEP: 1 -> 3.11-3.20 ms, 2 -> 2.61, 4 -> 2.64, 8 -> 2.72)
ASYNC_PIPELINE_PARTS = 2


def _run_host_pipelined(plan, xop, z, ldz, host_kind, stats) -> SpmmResult:
    """Host-memory result: the windows run in HOST_PIPELINE_PARTS nnz-balanced row ranges,
    and each range's Z rows are copied to pinned host memory on a copy stream while the
    next range computes (D2H overlapped with the SpMM)."""
    dev = z.device
    dim = xop.dim
    cs = _COPY_STREAMS.get(dev)
    if cs is None:
        cs = _COPY_STREAMS[dev] = torch.cuda.Stream(device=dev)
    host = torch.empty((z.shape[0], dim), dtype=torch.float32, pin_memory=True)
    wh, n = plan.windows.window_height, z.shape[0]
    cur = torch.cuda.current_stream(dev)
    for part in plan.parts(HOST_PIPELINE_PARTS):
        plan.run(xop, z, ldz, part=part)
        r0, r1 = min(part[0] * wh, n), min(part[1] * wh, n)
        if r1 > r0:
            ev = torch.cuda.Event()
            ev.record(cur)
            cs.wait_event(ev)
            with torch.cuda.stream(cs):
                host[r0:r1].copy_(z[r0:r1, :dim], non_blocking=True)
    cs.synchronize()
    z.record_stream(cs)
    return SpmmResult(DenseMatrix(host if host_kind == "torch" else host.numpy()), stats)


_H2D_STREAMS: dict = {}


class SpmmRequest:
    """A host-memory hybrid SpMM in flight (spmm_hybrid_async).  result() waits for the
    request's last D2H copy and returns what spmm_hybrid would have returned."""

    def __init__(self, host: torch.Tensor, done: torch.cuda.Event, host_kind, stats: ExecStats):
        self._host, self._done, self._kind, self._stats = host, done, host_kind, stats

    def done(self) -> bool:
        return self._done.query()

    def result(self) -> SpmmResult:
        self._done.synchronize()
        h = self._host
        return SpmmResult(DenseMatrix(h if self._kind == "torch" else h.numpy()), self._stats)


def spmm_hybrid_async(windows, assignment: Assignment, x, precision: str = "bf16",
                      out: torch.Tensor | None = None) -> SpmmRequest:
    """spmm_hybrid for a HOST operand, returning before the product is done, so consecutive
    requests overlap: request i+1's X upload (H2D stream) runs under request i's kernels, and
    each request's Z rows stream back (copy stream) while its later row ranges compute.  The
    kernels are those of spmm_hybrid; the product runs in ASYNC_PIPELINE_PARTS row ranges, so
    results equal spmm_hybrid's to fp32 summation order (bit for bit when unsplit).  Pinned host
    memory makes the copies asynchronous; a request's X must not be modified before result().
    `out`: optional pinned fp32 host tensor of at least (rows, dim) for Z (a caller-owned ring of
    result buffers avoids a pinned allocation per request)."""
    from .windows import as_windowset

    if len(assignment) != len(windows):
        raise ValueError(f"assignment covers {len(assignment)} windows, expected {len(windows)}")
    precision = _resolve_precision(precision)
    ws = as_windowset(windows)
    xrows = x.rows if isinstance(x, DenseMatrix) else int(x.shape[0])
    _check_window_bounds(ws, xrows)
    dev = ws.csr.device
    plan = get_plan(ws, assignment, precision)
    data = x.data if isinstance(x, DenseMatrix) else x
    if isinstance(data, torch.Tensor) and data.is_cuda:
        raise ValueError("spmm_hybrid_async takes a host operand; use spmm_hybrid for device tensors")
    h2d = _H2D_STREAMS.get(dev)
    if h2d is None:
        h2d = _H2D_STREAMS[dev] = torch.cuda.Stream(device=dev)
    cs = _COPY_STREAMS.get(dev)
    if cs is None:
        cs = _COPY_STREAMS[dev] = torch.cuda.Stream(device=dev)
    cur = torch.cuda.current_stream(dev)
    with torch.cuda.stream(h2d):  # the upload does not wait for earlier requests' kernels
        xop, _ = stage_operand(x, precision, dev, tf32_round=(precision == "tf32" and plan.n_tile > 0))
        up = torch.cuda.Event()
        up.record(h2d)
    cur.wait_event(up)
    xop.t.record_stream(cur)
    z, ldz = _alloc_z(ws.num_rows, xop.dim, dev)
    dim, wh, n = xop.dim, plan.windows.window_height, z.shape[0]
    if out is None:
        host = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
    else:
        if out.is_cuda or out.dtype != torch.float32 or out.shape[0] < n or out.shape[1] < dim:
            raise ValueError(f"out must be a host float32 tensor of at least ({n}, {dim})")
        host = out[:n, :dim]
    W = len(ws)
    parts = plan.parts(ASYNC_PIPELINE_PARTS) if W >= HOST_PIPELINE_MIN_WINDOWS else [None]
    for part in parts:
        plan.run(xop, z, ldz, part=part)
        r0, r1 = (min(part[0] * wh, n), min(part[1] * wh, n)) if part is not None else (0, n)
        if r1 > r0:
            ev = torch.cuda.Event()
            ev.record(cur)
            cs.wait_event(ev)
            with torch.cuda.stream(cs):
                host[r0:r1].copy_(z[r0:r1, :dim], non_blocking=True)
    done = torch.cuda.Event()
    done.record(cs)
    z.record_stream(cs)
    return SpmmRequest(host, done, _host_kind(x), ExecStats(**plan.stats.as_dict()))


class SpmmGraph:
    """A hybrid SpMM captured once as a CUDA graph and replayed: for repeated products with
    the same windows, assignment and X buffer (small graphs, where the 2-3 kernel launches of
    one product cost more than the kernels).  `x` must be a CUDA tensor; when it already is
    in the compute dtype with 16-byte rows it is used in place, so updating it in place and
    calling replay() recomputes Z.  Results are those of spmm_hybrid (same kernels)."""

    def __init__(self, windows, assignment: Assignment, x: torch.Tensor, precision: str = "bf16"):
        from .windows import as_windowset

        if len(assignment) != len(windows):
            raise ValueError(f"assignment covers {len(assignment)} windows, expected {len(windows)}")
        if not isinstance(x, torch.Tensor) or x.device.type != "cuda":
            raise ValueError("SpmmGraph needs a CUDA tensor operand")
        precision = _resolve_precision(precision)
        ws = as_windowset(windows)
        _check_window_bounds(ws, int(x.shape[0]))
        dev = ws.csr.device
        self.plan = get_plan(ws, assignment, precision)
        self.xop, _ = stage_operand(x, precision, dev, tf32_round=(precision == "tf32" and self.plan.n_tile > 0))
        self.z, self.ldz = _alloc_z(ws.num_rows, self.xop.dim, dev)
        self.stats = ExecStats(**self.plan.stats.as_dict())
        # the graph owns its partial-sum buffer (allocated before capture): a replay may run
        # next to eager products of the same plan on other streams
        self.scratch = self.plan.new_scratch() if self.plan.n_tile else None
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm-up outside the capture (module loading, attributes)
            self.plan.run(self.xop, self.z, self.ldz, scratch=self.scratch)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.plan.run(self.xop, self.z, self.ldz, scratch=self.scratch)
        self.launches = self.plan.launches_per_run(self.xop.dim)

    def replay(self) -> torch.Tensor:
        """Recompute Z = A X on the current stream; returns the [rows, dim] view of Z."""
        self.graph.replay()
        return self.z[:, : self.xop.dim]


def spmm_tile(windows, x, precision: str = "bf16", tile_cols: int = 8, dim_tile: int = 16,
              threads: int = 1) -> SpmmResult:
    """executors.py:216-231: every non-empty window on the tensor-core path."""
    from .windows import as_windowset

    ws = as_windowset(windows)
    asg = Assignment(torch.ones(len(ws), dtype=torch.uint8, device=ws.csr.device))
    return spmm_hybrid(ws, asg, x, precision=precision, threads=threads)


@_lib.nvtx("hcs.spmm_scalar")
def spmm_scalar(csr, x, precision: str = "bf16", window_height: int = 16) -> SpmmResult:
    """executors.py:191-213: every row on the CUDA-core path (no partition needed)."""
    xrows = x.rows if isinstance(x, DenseMatrix) else int(x.shape[0])
    if csr.num_cols != xrows:
        raise ValueError(f"dimension mismatch: matrix has {csr.num_cols} cols, X has {xrows} rows")
    precision = _resolve_precision(precision)
    dev = _lib.require_cuda()
    d = to_device_csr(csr, dev)
    xop, was_host = stage_operand(x, precision, dev)
    z, ldz = _alloc_z(d.num_rows, xop.dim, dev)
    W = -(-d.num_rows // window_height)
    wl = torch.arange(W, dtype=torch.int32, device=dev)
    vals, vcode = (d.values_bf16(), _lib.DTYPE_BF16) if precision == "bf16" else (d.values, _lib.DTYPE_F32)
    if W and W <= SCALAR_PIECES_MAX_WINDOWS and _scalar_variant_auto():  # the hybrid plan's small-list kernel
        run_scalar_pieces(d, vals, vcode, build_scalar_pieces(d, wl, window_height), {}, xop, z, ldz, 0, W,
                          _lib.stream())
    elif W:
        _lib.call("hcs_spmm_scalar", d.row_ptr.data_ptr(), d.col_idx.data_ptr(), vals.data_ptr(), vcode, d.num_rows,
                  window_height, wl.data_ptr(), W, xop.t.data_ptr(), xop.dtype_code, xop.rows, xop.dim, xop.ld,
                  z.data_ptr(), ldz, _lib.stream())
    rs = torch.arange(W, device=dev, dtype=torch.int64) * window_height
    re = torch.clamp(rs + window_height, max=d.num_rows)
    nonempty = int(((d.row_ptr[re] - d.row_ptr[rs]) > 0).sum().item()) if W else 0
    return _wrap_result(z, xop.dim, _host_kind(x) if was_host else False,
                        ExecStats(windows_scalar=nonempty, entries_scalar=d.nnz))


def spmm_auto(csr, x, assignment_for, precision: str = "bf16", threads: int = 1) -> SpmmResult:
    """executors.py:263-272."""
    from .windows import partition

    windows = partition(csr)
    return spmm_hybrid(windows, assignment_for(windows), x, precision=precision, threads=threads)


_SCALAR_VARIANTS = {"auto": 0, "block": 1, "warp16": 2, "rows": 3, "warp": 4}
_SCALAR_VARIANT = ["auto"]


def _scalar_variant_auto() -> bool:
    return _SCALAR_VARIANT[0] == "auto"


def set_scalar_variant(variant: str = "auto") -> None:
    """Select the CUDA-core (K3) kernel: "auto" (inside a hybrid plan: the piece kernel, one warp
    per <= 32-entry piece of a row, for lists of <= 1,024 windows; through hcs_spmm_scalar
    directly: "rows" for lists of <= 1,024 windows, else the warp-per-window kernel with 16-byte X
    vectors for bf16 X and 32-byte ones for fp32 X), "warp" (warp per window, col/val staged in
    shared memory, 32-byte X vectors when the operand allows), "rows" (warp per row, pairs broadcast by shuffles; small graphs), "block"
    (block per window, one warp per row with a fixed shuffle tree), "warp16" (warp per window,
    16-byte vectors)."""
    if variant not in _SCALAR_VARIANTS:
        raise ValueError(f"variant must be one of {sorted(_SCALAR_VARIANTS)}, got {variant!r}")
    _lib.call("hcs_set_scalar_variant", _SCALAR_VARIANTS[variant])
    _SCALAR_VARIANT[0] = variant
