"""Recording ingest, compatible with voltseg.video_io
(video_io.py:18-175).

VSEGV1 raw stacks: 8-byte magic, little-endian u32 T, H, W, sample code, f64
frame rate, then T*H*W samples.  The reference knows sample code 0 (float32,
video_io.py:19, :135-136); this module adds code 1 = uint16 (the camera
format, half the bytes over disk/PCIe) and reads files through `np.memmap`,
so `preprocess_file` streams a recording straight from the page cache into
the C-ABI stage executor (`vb_stage_run_host` packs pageable chunks into its
pinned ring) without ever holding the whole video in host RAM -- the
long-recording case (BASELINE configs[3]: 100,000 x 512 x 512).  Multi-page
TIFF is read and written by the in-repo reader (tiff.py; the reference uses
`tifffile`, absent from this image), memory-mapped when the pages' data are
contiguous, so TIFF recordings stream into the executor the same way.
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .tiff import TiffError, read_tiff, write_tiff
from .video import Video

VSEGV_MAGIC = b"VSEGV1\0\0"
SAMPLE_F32 = 0  # video_io.py:19
SAMPLE_U16 = 1  # extension: camera counts
_HEADER = 32
_DTYPES = {SAMPLE_F32: np.dtype("<f4"), SAMPLE_U16: np.dtype("<u2")}


class VideoIOError(Exception):
    """video_io.py:24-25."""


def read_header(path: str | Path) -> tuple[int, int, int, int, float | None]:
    """(T, H, W, sample code, frame rate) of a VSEGV1 file."""
    path = Path(path)
    if not path.is_file():
        raise VideoIOError(f"cannot read video file: {path}")
    with open(path, "rb") as f:
        head = f.read(_HEADER)
    if head[:8] != VSEGV_MAGIC:
        raise VideoIOError(f"{path}: not a VSEGV1 file")
    if len(head) < _HEADER:
        raise VideoIOError(f"{path}: truncated VSEGV1 header ({len(head)} bytes)")
    t, h, w, fmt = struct.unpack_from("<IIII", head, 8)
    (rate,) = struct.unpack_from("<d", head, 24)
    if fmt not in _DTYPES:
        raise VideoIOError(f"{path}: unsupported sample-format code {fmt}")
    expected = _HEADER + t * h * w * _DTYPES[fmt].itemsize
    size = path.stat().st_size
    if size != expected:
        raise VideoIOError(f"{path}: expected {expected} bytes, found {size}")
    return t, h, w, fmt, (rate if rate > 0 else None)


def open_raw(path: str | Path) -> tuple[np.memmap, float | None]:
    """Memory-map a VSEGV1 recording: (T, H, W) uint16 or float32, no copy."""
    t, h, w, fmt, rate = read_header(path)
    arr = np.memmap(path, dtype=_DTYPES[fmt], mode="r", offset=_HEADER, shape=(t, h, w))
    return arr, rate


def load_video(path: str | Path) -> Video:
    """video_io.py:85-96: VSEGV1 (f32 or u16) or multi-page TIFF."""
    path = Path(path)
    if not path.is_file():
        raise VideoIOError(f"cannot read video file: {path}")
    with open(path, "rb") as f:
        is_raw = f.read(8) == VSEGV_MAGIC
    if is_raw:
        arr, rate = open_raw(path)
        return Video(np.array(arr), frame_rate=rate)
    return Video(np.array(_open_tiff(path)))


def _open_tiff(path: Path) -> np.ndarray:
    """video_io.py:98-126 error mapping over the in-repo TIFF reader."""
    try:
        return read_tiff(path)
    except TiffError as exc:
        msg = str(exc)
        raise VideoIOError(msg if msg.startswith(str(path)) else f"{path}: unreadable TIFF: {msg}") from exc
    except Exception as exc:  # noqa: BLE001 - mirror the reference's error mapping
        raise VideoIOError(f"{path}: unreadable TIFF: {exc}") from exc


def open_recording(path: str | Path) -> np.ndarray:
    """(T, H, W) uint16/float32 (uint8 widened) view of a VSEGV1 or TIFF file,
    memory-mapped where the layout allows: the executor streams it from the
    page cache."""
    path = Path(path)
    if not path.is_file():
        raise VideoIOError(f"cannot read video file: {path}")
    with open(path, "rb") as f:
        is_raw = f.read(8) == VSEGV_MAGIC
    if is_raw:
        return open_raw(path)[0]
    arr = _open_tiff(path)
    return arr if arr.dtype in (np.uint16, np.float32) else arr.astype(np.float32)


def save_video(video, path: str | Path, sample: str = "auto") -> None:
    """video_io.py:144-175.  `.vsegv1` writes the raw format: float32 (code 0,
    readable by the reference) or, with sample="u16" / a uint16 recording and
    sample="auto", code 1."""
    v = Video.wrap(video)
    path = Path(str(path))
    if str(path) == "":
        raise VideoIOError("empty output path")
    if path.suffix != ".vsegv1":
        # the reference writes the float32 data as a minisblack multi-page TIFF
        # (video_io.py:154-157); sample="u16" keeps the camera counts
        data = v.raw if (sample == "u16" and v.raw is not None) else v.data
        try:
            write_tiff(path, data)
        except Exception as exc:  # noqa: BLE001
            raise VideoIOError(f"cannot write {path}: {exc}") from exc
        return
    use_u16 = sample == "u16" or (sample == "auto" and v.raw is not None)
    fmt = SAMPLE_U16 if use_u16 else SAMPLE_F32
    data = v.raw if (use_u16 and v.raw is not None) else v.data
    if use_u16 and data.dtype != np.uint16:
        if not np.array_equal(data, np.round(data)) or data.max() > 65535:
            raise VideoIOError(f"cannot write {path}: samples are not 16-bit integers")
        data = data.astype(np.uint16)
    header = VSEGV_MAGIC + struct.pack("<IIIId", v.frames, v.height, v.width, fmt, v.frame_rate or 0.0)
    with open(path, "wb") as f:
        f.write(header)
        f.write(np.ascontiguousarray(data, dtype=_DTYPES[fmt]).tobytes())


def preprocess_file(path: str | Path, config=None, device: int | None = None, chunk_frames: int = 0):
    """Stream a VSEGV1 or TIFF recording from disk through the C-ABI stage executor.

    Returns (vectors record array, spatial [K,H,W], temporal [K,H,W]); the
    corrected video is formed on the fly in HBM only."""
    from . import _lib
    from .stage import HostStage

    arr = open_recording(path)
    t, h, w = arr.shape
    hs = HostStage(h, w, config, device=device, chunk_frames=chunk_frames)
    try:
        cfg = hs.cfg
        k = -(-t // cfg.segment_length)
        vec = np.empty(t, dtype=_lib.MOTION_DTYPE)
        sp = np.empty((k, h, w), np.float32)
        tp = np.empty((k, h, w), np.float32)
        dtype = _lib.VB_U16 if arr.dtype == np.uint16 else _lib.VB_F32
        hs.run_into(arr.ctypes.data, dtype, t, vec, sp, tp)
    finally:
        hs.close()
        del arr
    return vec, sp, tp
