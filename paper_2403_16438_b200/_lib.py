"""ctypes binding of libvoltb200.so (include/voltb200.h).

The CUDA library is the ONLY compute path: there is no CPU fallback.  If the
shared library is missing it is built with nvcc (build.py); if that fails, or
no CUDA device is visible when a compute entry point is called, the error is
raised -- never silently routed elsewhere.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from . import build as _build

VB_OK, VB_EINVAL, VB_ECUDA, VB_ENOMEM = 0, 1, 2, 3
VB_U16, VB_F32 = 0, 1

MOTION_DTYPE = np.dtype([("dx", "<i4"), ("dy", "<i4"), ("sub_dx", "<f8"), ("sub_dy", "<f8"),
                         ("confidence", "<f8")], align=True)
assert MOTION_DTYPE.itemsize == 32


class VbMotion(C.Structure):
    _fields_ = [("dx", C.c_int32), ("dy", C.c_int32), ("sub_dx", C.c_double), ("sub_dy", C.c_double),
                ("confidence", C.c_double)]


class VbStageConfig(C.Structure):
    _fields_ = [("height", C.c_int), ("width", C.c_int), ("patch", C.c_int), ("radius", C.c_int),
                ("subpixel", C.c_int), ("ref_frames", C.c_int), ("segment_length", C.c_int),
                ("sigma", C.c_double), ("device", C.c_int), ("chunk_frames", C.c_int64)]


class VbSummaryOpts(C.Structure):
    """vb_summary_opts (include/voltb200.h): recording context + A17 options."""
    _fields_ = [("t_global0", C.c_int64), ("t_total", C.c_int64), ("interior_off", C.c_int64),
                ("n_interior", C.c_int64), ("highpass_window", C.c_int), ("gain_dev", C.c_void_p)]


_vp = C.c_void_p
_i32, _i64, _dbl = C.c_int, C.c_int64, C.c_double

# name -> (restype, argtypes); every symbol declared in include/voltb200.h
SIGNATURES = {
    "vb_version": (C.c_char_p, []),
    "vb_last_error": (C.c_char_p, []),
    "vb_mean_zncc_scores": (_i32, [_vp, _vp, _i32, _i32, _vp, _i32, _i32, _i32, _vp]),
    "vb_patch_grid": (_i32, [_i32, _i32, _i32, _i32, _vp, C.POINTER(C.c_int)]),
    "vb_template_sum": (_i32, [_vp, _i32, _i64, _i32, _i32, _vp, _i32, _vp]),
    "vb_template_finish": (_i32, [_vp, _i64, _i64, _vp, _vp]),
    "vb_make_reference": (_i32, [_vp, _i32, _i64, _i32, _i32, _i32, _vp, _vp]),
    "vb_motion_plan_create": (_i32, [C.POINTER(_vp), _i32, _i32, _i32, _i32, _vp, _i32]),
    "vb_motion_plan_set_reference": (_i32, [_vp, _vp, _vp]),
    "vb_motion_estimate": (_i32, [_vp, _vp, _i32, _i64, _i32, _vp, _vp, _vp]),
    "vb_motion_plan_info": (_i32, [_vp] + [C.POINTER(C.c_int)] * 4),
    "vb_motion_plan_destroy": (_i32, [_vp]),
    "vb_correct_frames": (_i32, [_vp, _i32, _i64, _i32, _i32, _vp, _vp, _vp]),
    "vb_summarize": (_i32, [_vp, _i32, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _vp, _vp]),
    "vb_smooth_frames": (_i32, [_vp, _i32, _i64, _i32, _i32, _vp, _i32, _vp, _vp]),
    "vb_extract_traces": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp, _i32, _vp, _vp]),
    "vb_extract_traces_raw": (_i32, [_vp, _i32, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _i32, _vp, _vp]),
    "vb_summarize_ex": (_i32, [_vp, _i32, _vp, _i64, _i32, _i32, _i32, _vp, _i32, C.POINTER(VbSummaryOpts),
                               _vp, _vp, _vp, _vp]),
    "vb_block_piece": (_i32, [_vp, _i32, _vp, _i64, _i32, _i32, _vp, _i32, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "vb_block_finish": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "vb_ipc_alloc": (_i32, [_i64, C.POINTER(_vp), _vp]),
    "vb_ipc_open": (_i32, [_vp, C.POINTER(_vp)]),
    "vb_ipc_close": (_i32, [_vp]),
    "vb_ipc_free": (_i32, [_vp]),
    "vb_copy_async": (_i32, [_vp, _vp, _i64, _vp]),
    "vb_memset_async": (_i32, [_vp, _i32, _i64, _vp]),
    "vb_unet_param_count": (_i64, []),
    "vb_unet_create": (_i32, [C.POINTER(_vp), _vp, _i64]),
    "vb_unet_forward": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "vb_normalize_pair": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp]),
    "vb_unet_tile_merge": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "vb_unet_segment": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp]),
    "vb_unet_destroy": (_i32, [_vp]),
    "vb_shading_gain": (_i32, [_vp, _i32, _i32, _vp, _i32, _vp, _vp]),
    "vb_correct_frames_ex": (_i32, [_vp, _i32, _i64, _i32, _i32, _vp, _vp, _vp, _vp]),
    "vb_stage_set_highpass": (_i32, [_vp, _i32]),
    "vb_stage_set_shading": (_i32, [_vp, _vp, _i32]),
    "vb_stage_create": (_i32, [C.POINTER(_vp), C.POINTER(VbStageConfig)]),
    "vb_stage_set_weights": (_i32, [_vp, _vp, _i32]),
    "vb_stage_run_host": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp]),
    "vb_stage_last_launches": (_i64, [_vp]),
    "vb_stage_set_unet": (_i32, [_vp, _vp, _i32]),
    "vb_stage_run_host_segment": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "vb_stage_destroy": (_i32, [_vp]),
    "vb_stage_set_reference": (_i32, [_vp, _vp]),
    "vb_group_plan": (_i32, [_i64, _i32, _i32, _vp]),
    "vb_group_create": (_i32, [C.POINTER(_vp), _vp, _i32, C.POINTER(VbStageConfig)]),
    "vb_group_set_weights": (_i32, [_vp, _vp, _i32]),
    "vb_group_run_host": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp]),
    "vb_group_last_launches": (_i64, [_vp]),
    "vb_group_destroy": (_i32, [_vp]),
    "vb_host_alloc": (_i32, [_i64, C.POINTER(_vp)]),
    "vb_host_free": (_i32, [_vp]),
    "vb_host_copy": (_i32, [_vp, _vp, _i64, _i32]),
    "vb_launch_count": (_i64, []),
    "vb_prof_enable": (_i32, [_i32]),
    "vb_prof_collect": (_i32, [_vp, _vp, _i32]),
    "vb_fp32_peak_probe": (_i32, [C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

_lock = threading.Lock()
_lib = None


def lib_path() -> Path:
    # VB_LIBRARY selects the experiment build (build.py --experiments) for A/B runs
    return Path(os.environ["VB_LIBRARY"]) if os.environ.get("VB_LIBRARY") else _build.LIB


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if needed) the CUDA library.  Raises on failure."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if build_if_missing and path == _build.LIB:
            _build.build()
        if not path.exists():
            raise ImportError(f"{path} is missing; run `python -m paper_2403_16438_b200.build`")
        L = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def last_error() -> str:
    return load().vb_last_error().decode(errors="replace")


def check(rc: int) -> None:
    """Map a VB_* status to the reference's exception types."""
    if rc == VB_OK:
        return
    msg = last_error()
    if rc == VB_EINVAL:
        raise ValueError(msg)
    if rc == VB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def launch_count() -> int:
    return int(load().vb_launch_count())
