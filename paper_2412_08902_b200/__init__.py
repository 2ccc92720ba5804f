"""B200-native HC-SpMM (arXiv 2412.08902): hybrid tensor-core / CUDA-core SpMM and
fused GCN layer behind the reference `rowwin` package's public entry points.

Modules mirror the reference layout: matrices, windows, selector, executors,
gnn, layout.  All compute runs in libhcspmm.so (sm_100a CUDA, C ABI in
include/hcspmm.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import FormatError, InvariantError  # noqa: F401
from .matrices import DenseMatrix, DeviceCsr, Graph, SparseCsr, graph_from_edges, to_device_csr  # noqa: F401
from .executors import (  # noqa: F401
    Assignment, ExecStats, Path, SpmmGraph, SpmmRequest, SpmmResult, spmm_auto, spmm_hybrid, spmm_hybrid_async,
    spmm_scalar, spmm_tile,
)
from .windows import (  # noqa: F401
    TILE_COLS, TILE_DIM, WINDOW_HEIGHT, RowWindow, WindowFeatures, WindowSet, features, partition,
    tile_count, total_rows,
)
from .selector import SelectorModel, b200_model, classify, classify_windows, default_model, load_model  # noqa: F401
from . import ops  # noqa: F401,E402  (registers torch.ops.hcspmm.spmm / gcn_layer)
