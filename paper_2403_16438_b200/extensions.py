"""A17: the north-star's shading/background correction and per-pixel temporal
high-pass filter (BASELINE.json north_star).

Neither exists in the reference (grep for shading / high-pass / vignett /
filtfilt / detrend in /root/reference/pkg/src finds nothing), so both are
OPT-IN and default off: with them off every output is the reference's.  Their
definition is this module + include/voltb200.h, restated on the CPU by
oracle/oracle.c (or_shading_gain, or_highpass_summary); parity is pinned to
that restatement only ("parity unpinned" against the reference).

* Shading correction: a flat-field gain estimated from the motion template,
  gain = G / mean(G) with G a wide float64 Gaussian of the template
  (scipy-style taps, truncate 4, "reflect").  Corrected frames are
  warped / gain (IEEE float32 division), fused into the warp kernel, so the
  summaries are taken over shading-corrected frames.
* Temporal high-pass: x - mean_N(x), a centred N-frame moving average
  (boxcar; -3 dB at ~0.443 fs / N) of the smoothed frames, reflected at the
  recording's ends.  The temporal summary becomes max - median of the
  high-passed stack; a time shard or chunk carries an N/2-frame halo on either
  side (the "filter-length halo" of the north star).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _device as D
from . import _lib

# boxcar moving average: |H(f)| = 1/sqrt(2) at f ~= 0.4429 fs / N
_BOXCAR_3DB = 0.4429


def highpass_window(cutoff_hz: float, frame_rate: float) -> int:
    """Odd moving-average length N whose high-pass (x - mean_N) has its -3 dB
    point nearest `cutoff_hz` at `frame_rate` (10 Hz at 741 fps -> 33)."""
    if cutoff_hz <= 0 or frame_rate <= 0:
        raise ValueError("cutoff and frame rate must be positive")
    n = _BOXCAR_3DB * frame_rate / cutoff_hz
    return max(3, 2 * int(math.floor(n / 2.0)) + 1)


def check_window(window: int) -> int:
    window = int(window or 0)
    if window > 1 and window % 2 == 0:
        raise ValueError("high-pass window must be odd")
    return window if window > 1 else 0


def shading_weights(sigma: float) -> tuple[np.ndarray, int]:
    """Taps of the shading Gaussian: scipy _gaussian_kernel1d(sigma, 0, radius)
    with gaussian_filter's default truncate 4 (radius = int(4 sigma + 0.5))."""
    if sigma <= 0:
        raise ValueError("shading sigma must be positive")
    radius = int(4.0 * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    return np.ascontiguousarray(phi / phi.sum(), dtype=np.float64), radius


def shading_gain_device(ref_dev: torch.Tensor, sigma: float) -> torch.Tensor:
    """Flat-field gain [H,W] float32 on the device from a device template."""
    h, w = ref_dev.shape
    wts, r = shading_weights(sigma)
    gain = torch.empty((h, w), dtype=torch.float32, device=ref_dev.device)
    _lib.call("vb_shading_gain", ref_dev.data_ptr(), h, w, wts.ctypes.data, r, gain.data_ptr(),
              D.stream_handle())
    return gain


def shading_gain(reference: np.ndarray, sigma: float) -> np.ndarray:
    """Flat-field gain of a host template (numpy in / out)."""
    ref = D.as_device_frames(np.asarray(reference, dtype=np.float32))
    return shading_gain_device(ref, sigma).cpu().numpy()
