"""Operator boundary, drop-in for voltseg.kernels (kernels.py:89-108).

The reference dispatches mean_zncc_scores between a Cython kernel and a
float64 numpy fallback via VOLTSEG_BACKEND.  Here there is exactly one
implementation -- libvoltb200's sm_100a kernel (vb_mean_zncc_scores) -- and no
fallback: a missing library or device raises.
"""
from __future__ import annotations

import numpy as np

from . import _lib

HAVE_NATIVE = True
BACKEND = "b200"


def mean_zncc_scores(frame, reference, origins, patch, radius) -> np.ndarray:
    """(2r+1, 2r+1) float64 mean-ZNCC grid indexed [dy+r, dx+r]
    (_native.pyx:22-118 / kernels.py:23-75 semantics)."""
    f = np.ascontiguousarray(frame, dtype=np.float32)
    r = np.ascontiguousarray(reference, dtype=np.float32)
    if f.ndim != 2 or r.shape != f.shape:
        raise ValueError("frame and reference dimensions differ")
    o = np.ascontiguousarray(origins, dtype=np.int32).reshape(-1, 2)
    side = 2 * int(radius) + 1
    out = np.empty((side, side), dtype=np.float64)
    _lib.call("vb_mean_zncc_scores", f.ctypes.data, r.ctypes.data, f.shape[0], f.shape[1],
              o.ctypes.data, len(o), int(patch), int(radius), out.ctypes.data)
    return out


_backends = {BACKEND: mean_zncc_scores}
