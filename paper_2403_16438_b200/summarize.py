"""Summary stage API, drop-in for voltseg.summarize (summarize.py:1-108).

Block splitting is host bookkeeping (views); the per-block spatial mean,
Gaussian smoothing and max-minus-median run in libvoltb200 (K3/K4) and are
bit-identical to the reference's numpy/scipy results.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _device as D
from . import _lib
from .extensions import check_window
from .video import Video

DEFAULT_SEGMENT_LENGTH = 50
DEFAULT_SMOOTH_SIGMA = 3.0


@dataclass(frozen=True)
class TimeSegment:
    """summarize.py:24-34."""

    index: int
    frames: np.ndarray
    segment_length: int

    def __post_init__(self):
        if not 1 <= self.frames.shape[0] <= self.segment_length:
            raise ValueError("segment frame count out of range")


@dataclass(frozen=True)
class SummaryPair:
    """summarize.py:37-41."""

    segment_index: int
    spatial: np.ndarray
    temporal: np.ndarray


def gaussian_weights(sigma: float) -> tuple[np.ndarray, int]:
    """scipy.ndimage._filters._gaussian_kernel1d(sigma, 0, radius), radius =
    ceil(3 sigma) (summarize.py:66, :71), reversed as gaussian_filter1d does.
    Computed with numpy so the taps are bit-identical to scipy's."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    radius = math.ceil(3 * sigma)
    sigma2 = sigma * sigma
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / sigma2 * x ** 2)
    phi = phi / phi.sum()
    return np.ascontiguousarray(phi[::-1], dtype=np.float64), radius


def split_segments(video, segment_length: int = DEFAULT_SEGMENT_LENGTH) -> list[TimeSegment]:
    """summarize.py:44-52."""
    if segment_length < 2:
        raise ValueError("segment length must be >= 2")
    v = Video.wrap(video)
    t = v.frames
    return [TimeSegment(i, v.data[i * segment_length:(i + 1) * segment_length], segment_length)
            for i in range(math.ceil(t / segment_length))]


def summarize_device(frames_dev: torch.Tensor, segment_length: int, sigma: float = DEFAULT_SMOOTH_SIGMA,
                     vectors_dev: torch.Tensor | None = None, corrected_out: torch.Tensor | None = None,
                     spatial_out: torch.Tensor | None = None, temporal_out: torch.Tensor | None = None, *,
                     highpass_window: int = 0, gain: torch.Tensor | None = None, t_global0: int = 0,
                     t_total: int | None = None, interior: tuple[int, int] | None = None):
    """Device-resident summaries of a (T,H,W) recording: (spatial, temporal),
    each float32 [ceil(n/L), H, W].  With vectors_dev the motion warp is fused
    (frames are raw) and corrected_out, if given, receives the corrected video.

    Recording context (time shards / chunks): frames_dev[0] is recording frame
    t_global0 of t_total, and only the blocks of frames_dev[interior[0] :
    interior[0] + interior[1]] are summarised (corrected_out then holds those
    frames only).  A17 (opt-in, extensions.py): highpass_window = odd N takes
    the temporal summary over x - mean_N(x) (frames_dev must then include the
    N/2-frame halo around the interior); gain = shading gain [H,W]."""
    t, h, w = frames_dev.shape
    window = check_window(highpass_window)
    ioff, n = interior if interior is not None else (0, t)
    k = math.ceil(n / segment_length)
    wts, wr = gaussian_weights(sigma)
    sp = spatial_out if spatial_out is not None else torch.empty((k, h, w), dtype=torch.float32,
                                                                 device=frames_dev.device)
    tp = temporal_out if temporal_out is not None else torch.empty((k, h, w), dtype=torch.float32,
                                                                   device=frames_dev.device)
    extended = window or gain is not None or t_global0 or interior is not None or (t_total not in (None, t))
    if not extended:
        _lib.call("vb_summarize", frames_dev.data_ptr(), D.vb_dtype(frames_dev), D.ptr(vectors_dev), t, h, w,
                  segment_length, wts.ctypes.data, wr, D.ptr(corrected_out), sp.data_ptr(), tp.data_ptr(),
                  D.stream_handle())
        return sp, tp
    opts = _lib.VbSummaryOpts(int(t_global0), int(t_total if t_total is not None else t_global0 + t), int(ioff),
                              int(n), int(window), D.ptr(gain))
    _lib.call("vb_summarize_ex", frames_dev.data_ptr(), D.vb_dtype(frames_dev), D.ptr(vectors_dev), t, h, w,
              segment_length, wts.ctypes.data, wr, _lib.C.byref(opts), D.ptr(corrected_out), sp.data_ptr(),
              tp.data_ptr(), D.stream_handle())
    return sp, tp


def spatial_summary(segment: TimeSegment) -> np.ndarray:
    """summarize.py:55-57: float64 mean over the segment's frames -> float32."""
    frames = D.as_device_frames(segment.frames)
    n, h, w = frames.shape
    s = torch.empty((h, w), dtype=torch.float64, device=frames.device)
    out = torch.empty((h, w), dtype=torch.float32, device=frames.device)
    st = D.stream_handle()
    _lib.call("vb_template_sum", frames.data_ptr(), D.vb_dtype(frames), n, h, w, s.data_ptr(), 0, st)
    _lib.call("vb_template_finish", s.data_ptr(), n, h * w, out.data_ptr(), st)
    return out.cpu().numpy()


def gaussian_smooth(image: np.ndarray, sigma: float = DEFAULT_SMOOTH_SIGMA) -> np.ndarray:
    """summarize.py:60-67 (2-D image; float32 result, rounded per pass like
    the reference's float32 stacks)."""
    wts, wr = gaussian_weights(sigma)
    img = D.as_device_frames(np.asarray(image))
    if img.dim() != 2:
        raise ValueError("gaussian_smooth expects a 2-D image")
    h, w = img.shape
    out = torch.empty((1, h, w), dtype=torch.float32, device=img.device)
    _lib.call("vb_smooth_frames", img.data_ptr(), D.vb_dtype(img), 1, h, w, wts.ctypes.data, wr,
              out.data_ptr(), D.stream_handle())
    return out[0].cpu().numpy()


def _segment_pair(segment: TimeSegment, sigma: float) -> tuple[np.ndarray, np.ndarray]:
    frames = D.as_device_frames(segment.frames)
    sp, tp = summarize_device(frames, frames.shape[0], sigma)
    return sp[0].cpu().numpy(), tp[0].cpu().numpy()


def temporal_summary(segment: TimeSegment, sigma: float = DEFAULT_SMOOTH_SIGMA) -> np.ndarray:
    """summarize.py:76-92: max minus median of the smoothed segment (>= 0)."""
    if segment.frames.shape[0] < 2:
        raise ValueError("temporal summary needs at least 2 frames")
    return _segment_pair(segment, sigma)[1]


def summarize_segment(segment: TimeSegment, sigma: float = DEFAULT_SMOOTH_SIGMA) -> SummaryPair:
    """summarize.py:95-96."""
    if segment.frames.shape[0] < 2:
        raise ValueError("temporal summary needs at least 2 frames")
    sp, tp = _segment_pair(segment, sigma)
    return SummaryPair(segment.index, sp, tp)


def summarize(video, segment_length: int = DEFAULT_SEGMENT_LENGTH,
              sigma: float = DEFAULT_SMOOTH_SIGMA, *, highpass_window: int = 0) -> list[SummaryPair]:
    """summarize.py:99-102: one SummaryPair per segment (all blocks in one launch).
    highpass_window (A17, opt-in, default off): see extensions.py."""
    if segment_length < 2:
        raise ValueError("segment length must be >= 2")
    v = Video.wrap(video)
    samples = v.samples
    esz = 2 if getattr(samples, "dtype", None) == np.uint16 else 4
    blk_bytes = segment_length * v.height * v.width * esz
    free = torch.cuda.mem_get_info(D.require_cuda())[0]
    if highpass_window > 1 or v.frames * v.height * v.width * esz <= free // 3:
        frames = D.as_device_frames(samples)
        sp, tp = summarize_device(frames, segment_length, sigma, highpass_window=highpass_window)
        sp, tp = sp.cpu().numpy(), tp.cpu().numpy()
        return [SummaryPair(i, sp[i], tp[i]) for i in range(sp.shape[0])]
    # long recordings: whole blocks per device batch (blocks are independent without the high-pass)
    if v.frames % segment_length == 1:
        raise ValueError("temporal summary needs at least 2 frames")
    per = max(1, int(free // 6 // blk_bytes)) * segment_length
    pairs = []
    for a in range(0, v.frames, per):
        sp, tp = summarize_device(D.as_device_frames(samples[a:a + per]), segment_length, sigma)
        sp, tp = sp.cpu().numpy(), tp.cpu().numpy()
        pairs += [SummaryPair(len(pairs) + i, sp[i], tp[i]) for i in range(sp.shape[0])]
    return pairs


def save_summaries(pairs: list[SummaryPair], path: str | Path) -> None:
    """summarize.py:105-108 (needs tifffile, like the reference)."""
    import tifffile

    stack = np.stack([img for p in pairs for img in (p.spatial, p.temporal)])
    tifffile.imwrite(path, stack.astype(np.float32), photometric="minisblack")
