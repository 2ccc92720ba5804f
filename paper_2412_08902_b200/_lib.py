"""ctypes binding of libhcspmm.so (include/hcspmm.h) and status -> exception mapping.

There is no fallback: if the shared library is missing or no CUDA device is
present, every compute entry point raises.  Build it with
`python -m paper_2412_08902_b200._build` (or __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import InvariantError

_HERE = os.path.dirname(os.path.abspath(__file__))
# HCS_LIB_PATH: load an experimental build of the same library instead (tools/ only)
LIB_PATH = os.environ.get("HCS_LIB_PATH") or os.path.join(_HERE, "libhcspmm.so")

HCS_OK, HCS_EINVAL, HCS_EDIM, HCS_EINVARIANT, HCS_ECUDA, HCS_ENCCL = range(6)
DTYPE_F32, DTYPE_BF16 = 0, 1

_lib = None
_lock = threading.Lock()

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
SZ = ctypes.c_size_t

_SIGS = {
    "hcs_version": (ctypes.c_int, []),
    "hcs_last_error": (ctypes.c_char_p, []),
    "hcs_device_sm_count": (ctypes.c_int, []),
    "hcs_partition_workspace_bytes": (ctypes.c_int, [I64, I64, I64, I32, ctypes.POINTER(SZ)]),
    "hcs_partition_count": (ctypes.c_int, [P, P, I64, I64, I64, I32, P, P, P, P, P, P, SZ, P]),
    "hcs_partition_fill": (ctypes.c_int, [P, P, I64, I64, I64, I32, P, P, P, P, SZ, P]),
    "hcs_classify": (ctypes.c_int, [P, P, I64, P, P, P]),
    "hcs_tile_plan_workspace_bytes": (ctypes.c_int, [I64, I64, ctypes.POINTER(SZ)]),
    "hcs_tile_plan": (ctypes.c_int, [P, P, P, ctypes.c_int, P, P, I64, I64, I32, P, I64, P, I64, P, P, P,
                                     ctypes.c_int, I64, P, SZ, P]),
    "hcs_spmm_scalar": (ctypes.c_int, [P, P, P, ctypes.c_int, I64, I32, P, I64, P, ctypes.c_int, I64, I32, I64, P,
                                       I64, P]),
    "hcs_spmm_scalar_pieces": (ctypes.c_int, [P, P, ctypes.c_int, P, P, P, P, I64, P, ctypes.c_int, I32, I64, P,
                                              I64, P, I64, P, P]),
    "hcs_spmm_tile": (ctypes.c_int, [P, I64, P, P, P, P, ctypes.c_int, I64, I32, P, ctypes.c_int, I64, I32, I64, P,
                                     I64, P, SZ, P]),
    "hcs_spmm_tile_balanced": (ctypes.c_int, [P, I64, P, P, P, P, ctypes.c_int, I64, I32, P, ctypes.c_int, I64, I32,
                                              I64, P, I64, P, SZ, ctypes.c_int, I64, P]),
    "hcs_tile_scratch_floats": (ctypes.c_int, [ctypes.POINTER(I64)]),
    "hcs_set_tile_slice": (ctypes.c_int, [ctypes.c_int]),
    "hcs_set_tile_npr3": (ctypes.c_int, [ctypes.c_int]),
    "hcs_set_scalar_variant": (ctypes.c_int, [ctypes.c_int]),
    "hcs_set_tile_pairing": (ctypes.c_int, [ctypes.c_int]),
    "hcs_set_tile_grid": (ctypes.c_int, [ctypes.c_int]),
    "hcs_set_tile_plan_builder": (ctypes.c_int, [ctypes.c_int]),
    "hcs_gcn_tile": (ctypes.c_int, [P, I64, P, P, P, P, ctypes.c_int, I64, I32, P, ctypes.c_int, I64, I32, I64, P,
                                     I64, P, I32, P, I64, P, SZ, P]),
    "hcs_gcn_scalar": (ctypes.c_int, [P, P, P, ctypes.c_int, I64, I32, P, I64, P, ctypes.c_int, I64, I32, I64, P,
                                       I64, P, I32, P, I64, P]),
    "hcs_grad_w_workspace_bytes": (ctypes.c_int, [I64, I32, I32, ctypes.POINTER(SZ)]),
    "hcs_grad_w": (ctypes.c_int, [P, I64, P, I64, I64, I32, I32, P, I64, P, SZ, P]),
    "hcs_gemm": (ctypes.c_int, [P, I64, P, I64, I64, I32, I32, P, I64, P]),
    "hcs_gemm_bf16": (ctypes.c_int, [P, I64, P, I64, I64, I32, I32, P, I64, I32, P, I64, P]),
    "hcs_softmax_xent_workspace_bytes": (ctypes.c_int, [I64, ctypes.POINTER(SZ)]),
    "hcs_softmax_xent": (ctypes.c_int, [P, I64, I64, I32, P, ctypes.c_float, P, P, ctypes.c_int, I64, I32, P, SZ,
                                        P]),
    "hcs_loa_workspace_bytes": (ctypes.c_int, [I64, ctypes.POINTER(SZ)]),
    "hcs_loa": (ctypes.c_int, [P, P, I64, I32, I32, P, P, P, P, P, SZ, P]),
    "hcs_convert": (ctypes.c_int, [P, P, I64, ctypes.c_int, P]),
    "hcs_normalize_values": (ctypes.c_int, [ctypes.c_int, P, P, P, I64, P, P, P, P]),
    "hcs_host_convert_f64": (ctypes.c_int, [P, I64, I64, I64, P, I64, ctypes.c_int, ctypes.c_int]),
    "hcs_io_count": (ctypes.c_int, [ctypes.c_char_p, I64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(I64),
                                    ctypes.POINTER(ctypes.c_int)]),
    "hcs_io_parse": (ctypes.c_int, [ctypes.c_char_p, I64, ctypes.c_int, ctypes.c_int, I64, ctypes.c_int, P, P, P,
                                    ctypes.POINTER(ctypes.c_int)]),
}


def lib():
    """Load (once) and return the ctypes handle; raises if the library is absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build the CUDA library with "
                        "`python -m paper_2412_08902_b200._build` (no CPU fallback exists)")
                h = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(h, name, None)
                    if fn is None:
                        continue
                    fn.restype = res
                    fn.argtypes = args
                _lib = h
    return _lib


def exported_symbols() -> list[str]:
    h = ctypes.CDLL(LIB_PATH)
    return [n for n in _SIGS if hasattr(h, n)]


def check(rc: int) -> None:
    if rc == HCS_OK:
        return
    msg = lib().hcs_last_error().decode(errors="replace")
    if rc in (HCS_EINVAL, HCS_EDIM):
        raise ValueError(msg)
    if rc == HCS_EINVARIANT:
        raise InvariantError(msg)
    raise RuntimeError(f"libhcspmm error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2412_08902_b200 requires a CUDA device (sm_100a); no CPU fallback exists")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


_NVTX = None


def nvtx(name: str):
    """Decorator: an NVTX range around each call (visible in nsys / ncu --nvtx timelines; a
    no-op cost of a few hundred ns without a profiler attached)."""
    import functools

    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*args, **kwargs):
            global _NVTX
            if _NVTX is None:
                _NVTX = torch.cuda.is_available()
            if not _NVTX:
                return fn(*args, **kwargs)
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.nvtx.range_pop()

        return wrapper

    return deco


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()
