"""Video data model mirroring voltseg.video_io.Video (video_io.py:28-58).

Same contract: (T, H, W), float32 view via ``.data``, finite, >= 0.
Extension for the B200 path: a uint16 recording is kept as ``raw`` (2 B/px
over PCIe and from HBM) and widened to float32 only if ``.data`` is read --
the widening is exact, so results are identical either way.
"""
from __future__ import annotations

import numpy as np


class Video:
    """Grayscale intensity stack with optional frame-rate metadata."""

    def __init__(self, data, frame_rate: float | None = None):
        self.frame_rate = frame_rate
        self._data = None
        self.raw = None
        arr = np.asarray(data)
        if arr.ndim != 3:
            raise ValueError(f"video data must be 3-D (T,H,W), got shape {arr.shape}")
        if 0 in arr.shape:
            raise ValueError(f"video dimensions must all be >= 1, got {arr.shape}")
        if arr.dtype == np.uint16:
            self.raw = np.ascontiguousarray(arr)  # finite and >= 0 by construction
            return
        if arr.dtype != np.float32:
            arr = arr.astype(np.float32)
        if not np.all(np.isfinite(arr)):
            raise ValueError("video intensities must be finite")
        if arr.min() < 0:
            raise ValueError("video intensities must be non-negative")
        self._data = arr

    @classmethod
    def _trusted(cls, data: np.ndarray, frame_rate: float | None = None) -> "Video":
        """A float32 (T,H,W) video this package produced (corrected frames:
        finite and non-negative by construction) -- skips the input scans."""
        v = cls.__new__(cls)
        v.frame_rate, v.raw, v._data = frame_rate, None, np.ascontiguousarray(data, dtype=np.float32)
        return v

    @classmethod
    def wrap(cls, video) -> "Video":
        """Accept this class, voltseg's Video (duck-typed) or an array."""
        if isinstance(video, Video):
            return video
        if hasattr(video, "data") and hasattr(video, "frame_rate"):
            return cls(video.data, video.frame_rate)
        return cls(video)

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            self._data = self.raw.astype(np.float32)
        return self._data

    @property
    def samples(self) -> np.ndarray:
        """The recording in its stored sample type (uint16 raw or float32)."""
        return self.raw if self.raw is not None else self._data

    @property
    def shape(self) -> tuple[int, int, int]:
        return tuple(self.samples.shape)

    @property
    def frames(self) -> int:
        return self.samples.shape[0]

    @property
    def height(self) -> int:
        return self.samples.shape[1]

    @property
    def width(self) -> int:
        return self.samples.shape[2]
