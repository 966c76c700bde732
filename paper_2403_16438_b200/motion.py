"""Motion stage API, drop-in for voltseg.motion (motion.py:1-256).

Same names, arguments, return types and ValueError messages as the reference;
the per-frame work (template, ZNCC search, tie-broken argmax, sub-pixel fit,
warp) runs in libvoltb200's sm_100a kernels.  Pure geometry / bookkeeping
helpers (PatchGrid, zncc on two windows, summed-area tables, CSV) stay on the
host exactly as in the reference.
"""
from __future__ import annotations

import csv
import threading
from dataclasses import dataclass
from functools import lru_cache
from pathlib import Path

import numpy as np
import torch

from . import _device as D
from . import _lib
from .extensions import shading_gain_device
from .video import Video

DEFAULT_PATCH_SIZE = 21
DEFAULT_SEARCH_RADIUS = 10
REFERENCE_FRAMES = 50  # motion.py:24; read at call time (monkeypatchable, like the reference)


@dataclass(frozen=True)
class MotionVector:
    """motion.py:27-41."""

    dx: int
    dy: int
    sub_dx: float = 0.0
    sub_dy: float = 0.0
    confidence: float = 0.0

    @property
    def x(self) -> float:
        return self.dx + self.sub_dx

    @property
    def y(self) -> float:
        return self.dy + self.sub_dy


@dataclass(frozen=True)
class PatchGrid:
    """motion.py:44-75: non-overlapping patch tiling with a final flush row/column."""

    patch_size: int
    stride: int
    origins: np.ndarray  # (N, 2) int32 of (x, y)

    @classmethod
    def cover(cls, height: int, width: int, patch_size: int = DEFAULT_PATCH_SIZE,
              stride: int | None = None, margin: int = 0) -> "PatchGrid":
        stride = stride or patch_size
        lo_x, hi_x = margin, width - margin - patch_size
        lo_y, hi_y = margin, height - margin - patch_size
        if hi_x < lo_x or hi_y < lo_y:
            raise ValueError(
                f"frame {height}x{width} too small for patch {patch_size} "
                f"with margin {margin}"
            )
        xs = _positions(lo_x, hi_x, stride)
        ys = _positions(lo_y, hi_y, stride)
        origins = np.array([(x, y) for y in ys for x in xs], dtype=np.int32)
        return cls(patch_size, stride, origins)


def _positions(lo: int, hi: int, stride: int) -> list[int]:
    pos = list(range(lo, hi + 1, stride))
    if pos[-1] != hi:
        pos.append(hi)
    return pos


def zncc(patch_a: np.ndarray, patch_b: np.ndarray) -> float:
    """motion.py:78-93 (two small windows; host float64)."""
    a = np.asarray(patch_a, dtype=np.float64)
    b = np.asarray(patch_b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"window dimensions differ: {a.shape} vs {b.shape}")
    a = a - a.mean()
    b = b - b.mean()
    denom = np.sqrt((a * a).sum() * (b * b).sum())
    if denom == 0:
        return 0.0
    return float((a * b).sum() / denom)


def build_area_tables(frame: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """motion.py:96-103 (host helper; the GPU search uses sliding sums instead)."""
    f = np.asarray(frame, dtype=np.float64)
    sat = np.zeros((f.shape[0] + 1, f.shape[1] + 1))
    sat2 = np.zeros_like(sat)
    np.cumsum(np.cumsum(f, axis=0), axis=1, out=sat[1:, 1:])
    np.cumsum(np.cumsum(f * f, axis=0), axis=1, out=sat2[1:, 1:])
    return sat, sat2


def rect_sum(table: np.ndarray, x0: int, y0: int, w: int, h: int) -> float:
    """motion.py:106-110."""
    return float(table[y0 + h, x0 + w] - table[y0, x0 + w] - table[y0 + h, x0] + table[y0, x0])


@dataclass
class MotionConfig:
    """motion.py:203-208.  ``threads`` is accepted for compatibility; frames are
    processed in parallel on the GPU regardless."""

    patch_size: int = DEFAULT_PATCH_SIZE
    search_radius: int = DEFAULT_SEARCH_RADIUS
    subpixel: bool = True
    threads: int = 1
    # A17 (opt-in, no reference counterpart; extensions.py): > 0 divides the
    # corrected frames by the template's flat-field gain at this sigma
    shading_sigma: float = 0.0


@lru_cache(maxsize=8)
def _candidate_order(radius: int):
    """motion.py:143-150 (the kernels use the same (|dx|+|dy|, dy, dx) key)."""
    span = range(-radius, radius + 1)
    order = sorted(((dx, dy) for dy in span for dx in span),
                   key=lambda d: (abs(d[0]) + abs(d[1]), d[1], d[0]))
    flat = np.array([(dy + radius) * (2 * radius + 1) + dx + radius for dx, dy in order])
    return order, flat


def _quadratic_peak(line: np.ndarray, i: int) -> float:
    """motion.py:153-160 (host restatement of the finalize kernel's fit)."""
    if i <= 0 or i >= len(line) - 1:
        return 0.0
    denom = line[i - 1] - 2.0 * line[i] + line[i + 1]
    if denom >= 0:
        return 0.0
    off = 0.5 * (line[i - 1] - line[i + 1]) / denom
    return float(np.clip(off, -0.999, 0.999))


def _vectors_from_numpy(rec: np.ndarray) -> list[MotionVector]:
    """vb_motion records -> MotionVector objects (Python ints / floats).  The
    frozen dataclass's field dict is filled directly: ~6x faster than its
    __init__ for the 10^4-10^5 vectors of a recording (same objects)."""
    new, mv = object.__new__, MotionVector
    out = []
    for dx, dy, sx, sy, c in zip(rec["dx"].tolist(), rec["dy"].tolist(), rec["sub_dx"].tolist(),
                                 rec["sub_dy"].tolist(), rec["confidence"].tolist()):
        v = new(mv)
        v.__dict__.update(dx=dx, dy=dy, sub_dx=sx, sub_dy=sy, confidence=c)
        out.append(v)
    return out


class MotionPlan:
    """Prepared geometry + template for one recording (vb_motion_plan)."""

    def __init__(self, height: int, width: int, origins: np.ndarray, patch: int, radius: int):
        self.height, self.width, self.patch, self.radius = height, width, patch, radius
        o = np.ascontiguousarray(origins, dtype=np.int32)
        self.n_patches = len(o)
        h = _lib.C.c_void_p()
        _lib.call("vb_motion_plan_create", _lib.C.byref(h), height, width, patch, radius,
                  o.ctypes.data, len(o))
        self._h = h

    def set_reference(self, ref_dev: torch.Tensor) -> None:
        assert ref_dev.dtype == torch.float32 and ref_dev.is_cuda
        _lib.call("vb_motion_plan_set_reference", self._h, ref_dev.data_ptr(), D.stream_handle())

    def estimate(self, frames_dev: torch.Tensor, subpixel: bool = True, scores: bool = False,
                 out: torch.Tensor | None = None):
        """Vectors (device buffer of vb_motion) for all frames; optional score grids."""
        n = frames_dev.shape[0] if frames_dev.dim() == 3 else 1
        vec = out if out is not None else D.empty_motion(n, frames_dev.device)
        side = 2 * self.radius + 1
        sc = torch.empty((n, side, side), dtype=torch.float64, device=frames_dev.device) if scores else None
        _lib.call("vb_motion_estimate", self._h, frames_dev.data_ptr(), D.vb_dtype(frames_dev), n,
                  int(subpixel), vec.data_ptr(), D.ptr(sc), D.stream_handle())
        return vec, sc

    def info(self) -> dict:
        """Work decomposition (patches, CTA groups, largest group, union width)."""
        vals = [_lib.C.c_int() for _ in range(4)]
        _lib.call("vb_motion_plan_info", self._h, *[_lib.C.byref(v) for v in vals])
        return dict(zip(("patches", "groups", "max_group", "max_width"), (v.value for v in vals)))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and _lib._lib is not None:
            _lib.load().vb_motion_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_reference(frames_dev: torch.Tensor, ref_frames: int | None = None) -> torch.Tensor:
    """make_reference on device frames: float64 mean of the first min(T, M) frames."""
    m = REFERENCE_FRAMES if ref_frames is None else ref_frames
    t, h, w = frames_dev.shape
    ref = torch.empty((h, w), dtype=torch.float32, device=frames_dev.device)
    _lib.call("vb_make_reference", frames_dev.data_ptr(), D.vb_dtype(frames_dev), t, h, w, m,
              ref.data_ptr(), D.stream_handle())
    return ref


def make_reference(video) -> np.ndarray:
    """motion.py:211-214: temporal mean of the first min(T, REFERENCE_FRAMES) raw frames."""
    v = Video.wrap(video)
    n = min(v.frames, REFERENCE_FRAMES)
    frames = D.as_device_frames(v.samples[:n])
    return device_reference(frames, n).cpu().numpy()


def estimate_motion(frame: np.ndarray, reference: np.ndarray, grid: PatchGrid,
                    search_radius: int = DEFAULT_SEARCH_RADIUS, subpixel: bool = True) -> MotionVector:
    """motion.py:113-140 for one frame (use correct_motion / MotionPlan for many)."""
    if search_radius < 1:
        raise ValueError("search_radius must be >= 1")
    f = np.asarray(frame)
    r = np.asarray(reference)
    if f.shape != r.shape:
        raise ValueError("frame and reference dimensions differ")
    dev = D.require_cuda()
    # called once per frame with the same grid and reference (like the
    # reference's motion loop): the calling thread keeps its last plan and
    # re-prepares the reference only when it changes
    c = _plan_cache.__dict__
    origins = np.ascontiguousarray(grid.origins, dtype=np.int32)
    key = (dev.index, f.shape, origins.tobytes(), grid.patch_size, search_radius)
    if c.get("key") != key:
        if c.get("plan") is not None:
            c["plan"].close()
        c["plan"] = MotionPlan(f.shape[0], f.shape[1], origins, grid.patch_size, search_radius)
        c["key"], c["ref"] = key, None
    plan = c["plan"]
    r32 = np.ascontiguousarray(r, dtype=np.float32)
    if c["ref"] is None or not np.array_equal(c["ref"], r32):
        plan.set_reference(D.as_device_frames(r32, dev))
        c["ref"] = r32.copy()
    vec, _ = plan.estimate(D.as_device_frames(f, dev)[None], subpixel)
    return _vectors_from_numpy(D.motion_to_numpy(vec, 1))[0]


_plan_cache = threading.local()


def _shift_vectors(n: int, dx: float, dy: float, dev) -> torch.Tensor:
    rec = np.zeros(n, dtype=_lib.MOTION_DTYPE)
    rec["sub_dx"] = -float(dx)
    rec["sub_dy"] = -float(dy)
    return torch.from_numpy(rec.view(np.uint8)).to(dev)


def translate(frame: np.ndarray, dx: float, dy: float) -> np.ndarray:
    """motion.py:163-176: shift content by (dx, dy) with edge replication;
    float32 bilinear for fractional offsets, exact gather for integer ones."""
    f = np.asarray(frame)
    dev = D.require_cuda()
    src = D.as_device_frames(f, dev)[None]
    out = torch.empty(src.shape, dtype=torch.float32, device=dev)
    vec = _shift_vectors(1, dx, dy, dev)  # vector x = -dx -> translate(frame, dx, dy)
    _lib.call("vb_correct_frames", src.data_ptr(), D.vb_dtype(src), 1, f.shape[0], f.shape[1],
              vec.data_ptr(), out.data_ptr(), D.stream_handle())
    return out[0].cpu().numpy()


def correct_frames_device(frames_dev: torch.Tensor, vectors_dev: torch.Tensor,
                          gain: torch.Tensor | None = None) -> torch.Tensor:
    t, h, w = frames_dev.shape
    out = torch.empty((t, h, w), dtype=torch.float32, device=frames_dev.device)
    _lib.call("vb_correct_frames_ex", frames_dev.data_ptr(), D.vb_dtype(frames_dev), t, h, w,
              vectors_dev.data_ptr(), D.ptr(gain), out.data_ptr(), D.stream_handle())
    return out


def correct_motion(video, config: MotionConfig | None = None) -> tuple[Video, list[MotionVector]]:
    """motion.py:217-241: estimate per-frame translation against a fixed
    reference and cancel it.  Returns (corrected Video float32, vectors)."""
    config = config or MotionConfig()
    v = Video.wrap(video)
    if config.search_radius < 1:
        raise ValueError("search_radius must be >= 1")
    PatchGrid.cover(v.height, v.width, config.patch_size, margin=config.search_radius)  # geometry errors
    dev = D.require_cuda()
    # the host recording streams through the C-ABI executor in motion-only
    # mode (bounded HBM, H2D / compute / D2H overlapped, threaded staging);
    # the calling thread keeps the executor for its last geometry
    from . import stage as S

    sc = S.StageConfig(patch_size=config.patch_size, search_radius=config.search_radius, subpixel=config.subpixel,
                       ref_frames=REFERENCE_FRAMES, shading_sigma=config.shading_sigma)
    hs = S.cached_host_stage(dev, v.height, v.width, sc)
    rec, _sp, _tp, out = hs.run(v.samples, corrected=True, summaries=False)
    return Video._trusted(out, frame_rate=v.frame_rate), _vectors_from_numpy(rec)


def correct_frame(frame: np.ndarray, vector: MotionVector) -> np.ndarray:
    """motion.py:244-248."""
    if vector.x == 0 and vector.y == 0:
        return frame
    return translate(frame, -vector.x, -vector.y)


def save_motion_csv(vectors: list[MotionVector], path: str | Path) -> None:
    """motion.py:251-256."""
    with open(path, "w", newline="") as f:
        writer = csv.writer(f)
        writer.writerow(["frame", "dx", "dy", "confidence"])
        for t, v in enumerate(vectors):
            writer.writerow([t, f"{v.x:g}", f"{v.y:g}", f"{v.confidence:.6f}"])
