"""ctypes front-end for the C restatement in oracle.c -- TEST INFRASTRUCTURE ONLY.

Mirrors the reference's Python functions (file:line under
/root/reference/pkg/src/voltseg) with numpy in/out so tests read like the
reference's own tests.  Pinned against the reference's outputs by
tests/test_oracle_golden.py (fixtures in tests/golden/, made by
tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libvsoracle.so"

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_lib = None


def build() -> Path:
    """Compile libvsoracle.so (gcc, a few seconds)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.or_make_reference.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p]
        L.or_patch_grid.argtypes = [C.c_int] * 5 + [C.c_void_p]
        L.or_patch_grid.restype = C.c_int
        L.or_mean_zncc_scores.argtypes = [_f32p, _f32p, C.c_int, C.c_int, _i32p, C.c_int, C.c_int, C.c_int, _f64p]
        L.or_mean_zncc_scores.restype = C.c_int
        L.or_pick_motion.argtypes = [_f64p, C.c_int, C.c_int, _i32p, _f64p]
        L.or_translate.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_double, _f32p]
        L.or_correct_frame.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_double, _f32p]
        L.or_spatial_summary.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p]
        L.or_smooth_frame.argtypes = [_f32p, C.c_int, C.c_int, _f64p, C.c_int, _f32p, C.c_void_p]
        L.or_temporal_summary.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f64p, C.c_int, _f32p]
        L.or_temporal_summary.restype = C.c_int
        L.or_preprocess.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, _f64p, C.c_int, C.c_int, _i32p, _f64p, C.c_void_p,
                                    _f32p, _f32p]
        L.or_preprocess.restype = C.c_int
        L.or_extract_trace.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _f64p]
        L.or_shading_gain.argtypes = [_f32p, C.c_int, C.c_int, _f64p, C.c_int, _f32p]
        L.or_highpass_summary.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f64p, C.c_int, C.c_int, C.c_int,
                                          _f32p]
        L.or_highpass_summary.restype = C.c_int
        L.or_motion_frames.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p, _i32p, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, _i32p, _f64p, C.c_void_p, C.c_void_p]
        L.or_motion_frames.restype = C.c_int
        L.or_summaries.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f64p, C.c_int, C.c_int, _f32p, _f32p]
        L.or_summaries.restype = C.c_int
        _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def gaussian_weights(sigma: float = 3.0) -> tuple[np.ndarray, int]:
    """scipy.ndimage._filters._gaussian_kernel1d(sigma, 0, radius) with
    radius = ceil(3 sigma) (summarize.py:71): exp(-0.5/sigma^2 x^2), normalised."""
    radius = math.ceil(3 * sigma)
    sigma2 = sigma * sigma
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / sigma2 * x ** 2)
    phi = phi / phi.sum()
    return np.ascontiguousarray(phi[::-1], dtype=np.float64), radius


def make_reference(frames: np.ndarray, ref_frames: int = 50) -> np.ndarray:
    """motion.py:211-214 (REFERENCE_FRAMES passed explicitly)."""
    f = _f32(frames)
    n = min(f.shape[0], ref_frames)
    out = np.empty(f.shape[1:], np.float32)
    lib().or_make_reference(f, n, f.shape[1], f.shape[2], out)
    return out


def patch_grid(h: int, w: int, patch: int = 21, margin: int = 0) -> np.ndarray:
    """motion.py:52-75 PatchGrid.cover(...).origins."""
    n = lib().or_patch_grid(h, w, patch, patch, margin, None)
    if n < 0:
        raise ValueError(f"frame {h}x{w} too small for patch {patch} with margin {margin}")
    out = np.empty((n, 2), np.int32)
    lib().or_patch_grid(h, w, patch, patch, margin, out.ctypes.data)
    return out


def mean_zncc_scores(frame, reference, origins, patch: int, radius: int) -> np.ndarray:
    """kernels.py:23-75 (float64 backend semantics)."""
    f, r = _f32(frame), _f32(reference)
    if f.shape != r.shape:
        raise ValueError("frame and reference dimensions differ")
    o = np.ascontiguousarray(origins, dtype=np.int32)
    side = 2 * radius + 1
    out = np.empty((side, side), np.float64)
    if lib().or_mean_zncc_scores(f, r, f.shape[0], f.shape[1], o, len(o), patch, radius, out) != 0:
        raise ValueError("patch origin too close to border for search radius")
    return out


def pick_motion(scores: np.ndarray, radius: int, subpixel: bool = True):
    """motion.py:127-140 -> (dx, dy, sub_dx, sub_dy, confidence)."""
    dxdy = np.empty(2, np.int32)
    sc = np.empty(3, np.float64)
    lib().or_pick_motion(np.ascontiguousarray(scores, np.float64), radius, int(subpixel), dxdy, sc)
    return int(dxdy[0]), int(dxdy[1]), float(sc[0]), float(sc[1]), float(sc[2])


def estimate_motion(frame, reference, origins, patch, radius, subpixel=True):
    """motion.py:113-140."""
    if radius < 1:
        raise ValueError("search_radius must be >= 1")
    return pick_motion(mean_zncc_scores(frame, reference, origins, patch, radius), radius, subpixel)


def translate(frame, dx: float, dy: float) -> np.ndarray:
    """motion.py:163-200."""
    f = _f32(frame)
    out = np.empty_like(f)
    lib().or_translate(f, f.shape[0], f.shape[1], float(dx), float(dy), out)
    return out


def correct_frame(frame, vx: float, vy: float) -> np.ndarray:
    """motion.py:244-248 (vector given as x = dx + sub_dx, y = dy + sub_dy)."""
    f = _f32(frame)
    out = np.empty_like(f)
    lib().or_correct_frame(f, f.shape[0], f.shape[1], float(vx), float(vy), out)
    return out


def spatial_summary(frames) -> np.ndarray:
    """summarize.py:55-57."""
    f = _f32(frames)
    out = np.empty(f.shape[1:], np.float32)
    lib().or_spatial_summary(f, f.shape[0], f.shape[1], f.shape[2], out)
    return out


def smooth_frame(frame, sigma: float = 3.0) -> np.ndarray:
    """summarize.py:70-73 on one frame."""
    f = _f32(frame)
    w, r = gaussian_weights(sigma)
    out = np.empty_like(f)
    lib().or_smooth_frame(f, f.shape[0], f.shape[1], w, r, out, None)
    return out


def temporal_summary(frames, sigma: float = 3.0) -> np.ndarray:
    """summarize.py:76-92."""
    f = _f32(frames)
    if f.shape[0] < 2:
        raise ValueError("temporal summary needs at least 2 frames")
    w, r = gaussian_weights(sigma)
    out = np.empty(f.shape[1:], np.float32)
    lib().or_temporal_summary(f, f.shape[0], f.shape[1], f.shape[2], w, r, out)
    return out


def preprocess(frames, patch=21, radius=10, subpixel=True, ref_frames=50,
               segment_length=50, sigma=3.0, threads=None, want_corrected=True):
    """correct_motion (motion.py:217-241) then summarize (summarize.py:99-102).

    Returns dict(dxdy int32[T,2], sub_conf f64[T,3], corrected f32[T,H,W] | None,
    spatial f32[K,H,W], temporal f32[K,H,W])."""
    f = _f32(frames)
    t, h, w = f.shape
    k = -(-t // segment_length)
    wts, wr = gaussian_weights(sigma)
    dxdy = np.empty((t, 2), np.int32)
    sc = np.empty((t, 3), np.float64)
    corr = np.empty_like(f) if want_corrected else None
    sp = np.zeros((k, h, w), np.float32)
    tp = np.zeros((k, h, w), np.float32)
    threads = threads or os.cpu_count() or 1
    rc = lib().or_preprocess(f, t, h, w, patch, radius, int(subpixel), ref_frames, segment_length,
                             wts, wr, threads, dxdy, sc,
                             corr.ctypes.data if corr is not None else None, sp, tp)
    if rc != 0:
        raise ValueError("invalid preprocess geometry")
    return dict(dxdy=dxdy, sub_conf=sc, corrected=corr, spatial=sp, temporal=tp)


def motion_frames(frames, reference, origins, patch: int, radius: int, subpixel: bool = True,
                  threads: int | None = None, want_corrected: bool = True, want_scores: bool = False):
    """estimate_motion + correct_frame (motion.py:113-160, :235-240) of every
    frame against a given template, frames split over threads.

    Returns dict(dxdy int32[T,2], sub_conf f64[T,3], corrected f32[T,H,W] | None,
    scores f64[T,2r+1,2r+1] | None)."""
    f = _f32(frames)
    t, h, w = f.shape
    o = np.ascontiguousarray(origins, dtype=np.int32)
    dxdy = np.empty((t, 2), np.int32)
    sc = np.empty((t, 3), np.float64)
    corr = np.empty_like(f) if want_corrected else None
    side = 2 * radius + 1
    scores = np.empty((t, side, side), np.float64) if want_scores else None
    rc = lib().or_motion_frames(f, t, h, w, _f32(reference), o, len(o), patch, radius, int(subpixel),
                                threads or os.cpu_count() or 1, dxdy, sc,
                                corr.ctypes.data if corr is not None else None,
                                scores.ctypes.data if scores is not None else None)
    if rc != 0:
        raise ValueError("patch origin too close to border for search radius")
    return dict(dxdy=dxdy, sub_conf=sc, corrected=corr, scores=scores)


def summaries(corrected, segment_length: int, sigma: float = 3.0, threads: int | None = None):
    """summarize.py:95-102 over corrected frames -> (spatial f32[K,H,W], temporal f32[K,H,W])."""
    f = _f32(corrected)
    t, h, w = f.shape
    k = -(-t // segment_length)
    wts, wr = gaussian_weights(sigma)
    sp = np.empty((k, h, w), np.float32)
    tp = np.empty((k, h, w), np.float32)
    if lib().or_summaries(f, t, h, w, segment_length, wts, wr, threads or os.cpu_count() or 1, sp, tp) != 0:
        raise ValueError("temporal summary needs at least 2 frames")
    return sp, tp


def extract_trace(frames, mask) -> np.ndarray:
    """traces.py:23-34 (samples only)."""
    f = _f32(frames)
    bits = np.asarray(getattr(mask, "bits", mask), dtype=bool)
    ys, xs = np.nonzero(bits)
    if len(ys) == 0:
        raise ValueError("empty ROI mask")
    idx = np.ascontiguousarray(ys * f.shape[2] + xs, dtype=np.int32)
    out = np.empty(f.shape[0], np.float64)
    lib().or_extract_trace(f, f.shape[0], f.shape[1], f.shape[2], idx, len(idx), out)
    return out


# ---- A17 extensions (no reference counterpart: parity unpinned; the C code
# is their definition, mirrored by include/voltb200.h) ----------------------

def shading_weights(sigma: float) -> tuple[np.ndarray, int]:
    """Gaussian taps for the shading gain: scipy's _gaussian_kernel1d with
    gaussian_filter's default truncate=4 (radius = int(4 sigma + 0.5))."""
    radius = int(4.0 * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    return np.ascontiguousarray(phi / phi.sum(), dtype=np.float64), radius


def shading_gain(reference, sigma: float) -> np.ndarray:
    ref = _f32(reference)
    w, r = shading_weights(sigma)
    out = np.empty_like(ref)
    lib().or_shading_gain(ref, ref.shape[0], ref.shape[1], w, r, out)
    return out


def highpass_summary(corrected, segment_length: int, window: int, sigma: float = 3.0) -> np.ndarray:
    """Temporal summaries [K,H,W] of the whole recording with the high-pass."""
    f = _f32(corrected)
    t, h, w = f.shape
    wts, wr = gaussian_weights(sigma)
    out = np.empty((-(-t // segment_length), h, w), np.float32)
    rc = lib().or_highpass_summary(f, t, h, w, wts, wr, segment_length, window, out)
    if rc != 0:
        raise ValueError("invalid high-pass summary arguments")
    return out
