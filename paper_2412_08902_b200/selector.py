"""Per-window core selector (reference selector.py inference half, lines 38-64, 260-288).

Decisions for a device WindowSet are computed on the GPU in IEEE fp64 with
round-to-nearest intrinsics (csrc/partition.cu k_features / k_classify), so
they are bit-identical to the reference's Python-float evaluation of
((w_ncols*zn) + (w_density*zd)) + bias.  Training (selector.py:67-257) lives in
selector_train.py (B200 timing provider); b200_model() is the opt-in result.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from .executors import Assignment, Path
from .windows import WindowFeatures, WindowSet, _selector_doubles, features

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "selector_default.json")
_DATA_B200 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "selector_b200.json")


@dataclass(frozen=True)
class SelectorModel:
    """selector.py:38-56: positive score picks SCALAR; empty windows are SCALAR."""

    w_ncols: float
    w_density: float
    bias: float
    feature_means: tuple
    feature_scales: tuple

    def score(self, ncols: float, density: float) -> float:
        zn = (ncols - self.feature_means[0]) / self.feature_scales[0]
        zd = (density - self.feature_means[1]) / self.feature_scales[1]
        return self.w_ncols * zn + self.w_density * zd + self.bias

    def decide(self, ncols: int, density: float) -> Path:
        if ncols == 0:
            return Path.SCALAR
        return Path.SCALAR if self.score(ncols, density) > 0 else Path.TILE


def classify(model: SelectorModel, f: WindowFeatures) -> Path:
    """selector.py:59-60."""
    return model.decide(f.ncols, f.density)


def classify_windows(model, windows) -> Assignment:
    """selector.py:63-64.  GPU path for a WindowSet; host path for RowWindow lists."""
    if isinstance(windows, WindowSet):
        sel = _selector_doubles(model)
        if windows.codes is not None and windows.selector == sel:
            codes = windows.codes
        else:
            dev = windows.win_col_ptr.device
            W = windows.num_windows
            codes = torch.empty(W, dtype=torch.uint8, device=dev)
            sel_c = (_lib.ctypes.c_double * 7)(*sel)
            if W:
                _lib.call("hcs_classify", windows.win_col_ptr.data_ptr(), windows.density.data_ptr(), W,
                          _lib.ctypes.addressof(sel_c), codes.data_ptr(), _lib.stream())
        return Assignment.from_device(codes)
    return Assignment.from_paths(classify(model, features(w)) for w in windows)


def _model_from_doc(doc: dict) -> SelectorModel:
    """selector.py:260-275."""
    required = ("w_ncols", "w_density", "bias", "feature_means", "feature_scales")
    missing = [k for k in required if k not in doc]
    if missing:
        raise ValueError(f"selector model missing fields: {missing}")
    means, scales = doc["feature_means"], doc["feature_scales"]
    if len(means) != 2 or len(scales) != 2:
        raise ValueError("feature_means/feature_scales must have two entries")
    return SelectorModel(float(doc["w_ncols"]), float(doc["w_density"]), float(doc["bias"]),
                         (float(means[0]), float(means[1])), (float(scales[0]), float(scales[1])))


def load_model(path: str) -> SelectorModel:
    """selector.py:278-281."""
    with open(path, "r", encoding="utf-8") as fh:
        return _model_from_doc(json.load(fh))


@lru_cache(maxsize=1)
def default_model() -> SelectorModel:
    """selector.py:284-288: the shipped weights (data/selector_default.json)."""
    return load_model(_DATA)


@lru_cache(maxsize=1)
def b200_model() -> SelectorModel:
    """Opt-in model trained on measured B200 timings of this repo's kernels (cli
    train-selector --grid b200 --dim 128; selector_train.py).  Not the default: the
    reference's shipped model keeps window decisions bit-exact with rowwin."""
    return load_model(_DATA_B200)


def save_model(model: SelectorModel, path: str, provenance: dict | None = None) -> None:
    """selector.py:244-257 (JSON persistence of the 7 doubles)."""
    doc = {"w_ncols": model.w_ncols, "w_density": model.w_density, "bias": model.bias,
           "feature_means": list(model.feature_means), "feature_scales": list(model.feature_scales),
           "version": 1, "provenance": provenance or {}}
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=2, sort_keys=True)
        fh.write("\n")


def decisions_host(model: SelectorModel, ncols: np.ndarray, density: np.ndarray) -> np.ndarray:
    """Vectorised host restatement of decide() (used for RowWindow lists of any size)."""
    nc = np.asarray(ncols, dtype=np.int64)
    zn = (nc.astype(np.float64) - model.feature_means[0]) / model.feature_scales[0]
    zd = (np.asarray(density, dtype=np.float64) - model.feature_means[1]) / model.feature_scales[1]
    s = model.w_ncols * zn + model.w_density * zd
    s = s + model.bias
    out = np.where(s > 0, 0, 1).astype(np.uint8)
    out[nc == 0] = 0
    return out
