"""Trace extraction, drop-in for voltseg.traces (traces.py:1-66) -- SURVEY.md
8(f) row 1, the first consumer of the corrected video.

`extract_trace` / `extract_all` compute the per-frame mean intensity over each
ROI mask on the GPU (vb_extract_traces: one warp per (ROI, frame), float64
accumulation); `dff` and the CSV writer are host bookkeeping like the
reference.  `extract_traces_device` works on a corrected video already in HBM
(e.g. DevicePreprocessor's output) without a host round trip, and
`extract_traces_raw_device` on the raw frames + motion vectors, fusing the
warp so the corrected video is never written.
"""
from __future__ import annotations

import csv
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _device as D
from . import _lib
from .video import Video


@dataclass
class Trace:
    """traces.py:16-20."""

    footprint_id: int
    samples: np.ndarray  # (T,) float64
    frame_rate: float | None = None


def _mask_bits(mask) -> np.ndarray:
    bits = getattr(mask, "bits", mask)
    return np.asarray(bits, dtype=bool)


def _csr(masks, h: int, w: int) -> tuple[np.ndarray, np.ndarray]:
    ptr = [0]
    idx = []
    for m in masks:
        bits = _mask_bits(m)
        if bits.shape != (h, w):
            raise ValueError(f"mask {bits.shape} does not match frames ({h}, {w})")
        ys, xs = np.nonzero(bits)
        if len(ys) == 0:
            raise ValueError("empty ROI mask")
        idx.append((ys * w + xs).astype(np.int32))
        ptr.append(ptr[-1] + len(ys))
    return np.asarray(ptr, np.int32), (np.concatenate(idx) if idx else np.zeros(0, np.int32))


def extract_traces_device(frames_dev: torch.Tensor, masks) -> torch.Tensor:
    """float64 [K, T] means of a device-resident float32 (T, H, W) video over K masks."""
    if frames_dev.dtype != torch.float32:
        frames_dev = frames_dev.to(torch.float32)
    t, h, w = frames_dev.shape
    ptr, idx = _csr(masks, h, w)
    dev = frames_dev.device
    ptr_d = torch.from_numpy(ptr).to(dev)
    idx_d = torch.from_numpy(idx).to(dev)
    out = torch.empty((len(ptr) - 1, t), dtype=torch.float64, device=dev)
    _lib.call("vb_extract_traces", frames_dev.data_ptr(), t, h, w, ptr_d.data_ptr(), idx_d.data_ptr(),
              len(ptr) - 1, out.data_ptr(), D.stream_handle())
    return out


def extract_traces_raw_device(frames_dev: torch.Tensor, vectors_dev: torch.Tensor | None, masks,
                              gain_dev: torch.Tensor | None = None) -> torch.Tensor:
    """float64 [K, T] traces straight from the RAW (T, H, W) uint16 / float32
    frames in HBM and their motion vectors (vb_motion device buffer, e.g.
    MotionPlan.estimate's output): the corrected video is never materialised
    (SURVEY 8(f) row 1).  Bit-identical to extract_traces_device on the
    corrected frames."""
    t, h, w = frames_dev.shape
    ptr, idx = _csr(masks, h, w)
    dev = frames_dev.device
    ptr_d = torch.from_numpy(ptr).to(dev)
    idx_d = torch.from_numpy(idx).to(dev)
    out = torch.empty((len(ptr) - 1, t), dtype=torch.float64, device=dev)
    _lib.call("vb_extract_traces_raw", frames_dev.data_ptr(), D.vb_dtype(frames_dev), D.ptr(vectors_dev),
              D.ptr(gain_dev), t, h, w, ptr_d.data_ptr(), idx_d.data_ptr(), len(ptr) - 1, out.data_ptr(),
              D.stream_handle())
    return out


def extract_trace(video, mask, footprint_id: int = 0) -> Trace:
    """traces.py:23-34: mean intensity over the mask pixels for every frame."""
    v = Video.wrap(video)
    bits = _mask_bits(mask)
    if bits.shape != (v.height, v.width):
        raise ValueError(f"mask {bits.shape} does not match frames ({v.height}, {v.width})")
    out = extract_traces_device(D.as_device_frames(v.data), [bits])
    return Trace(footprint_id, out[0].cpu().numpy(), v.frame_rate)


def extract_all(video, footprints) -> list[Trace]:
    """traces.py:37-40: one trace per footprint (a FootprintSet-like object
    with `.footprints[i].mask`, or a sequence of masks), order preserved."""
    fps = getattr(footprints, "footprints", footprints)
    masks = [getattr(fp, "mask", fp) for fp in fps]
    v = Video.wrap(video)
    if not masks:
        return []
    out = extract_traces_device(D.as_device_frames(v.data), masks).cpu().numpy()
    return [Trace(i, out[i], v.frame_rate) for i in range(len(masks))]


def dff(trace: Trace, baseline_percentile: float = 10.0) -> Trace:
    """traces.py:43-49."""
    baseline = np.percentile(trace.samples, baseline_percentile)
    if baseline == 0:
        raise ValueError("zero baseline, dF/F undefined")
    return Trace(trace.footprint_id, (trace.samples - baseline) / baseline, trace.frame_rate)


def save_traces_csv(traces: list[Trace], path: str | Path, sidecar_path: str | Path | None = None) -> None:
    """traces.py:52-66."""
    path = Path(path)
    with open(path, "w", newline="") as f:
        writer = csv.writer(f)
        writer.writerow(["frame"] + [str(t.footprint_id) for t in traces])
        n = len(traces[0].samples) if traces else 0
        for row in range(n):
            writer.writerow([row] + [f"{t.samples[row]:.6f}" for t in traces])
    if sidecar_path is None:
        sidecar_path = path.with_suffix(".json")
    rate = traces[0].frame_rate if traces else None
    Path(sidecar_path).write_text(json.dumps({"frame_rate": rate}))
