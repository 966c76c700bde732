"""GPU orchestration of the reference pipeline's motion + segmentation
stages: pipeline.py:190-258 `_run_motion_and_segment`
without the footprint NMF (out of scope), on the C-ABI host executor.

The reference overlaps motion correction (producer thread) with
summarize + normalize + U-Net (consumer) through a bounded queue of four
segments (pipeline.py:226-242).  Here one call streams the recording through
HBM in block-aligned chunks: H2D of chunk k+1, motion search + fused warp /
summaries of chunk k on the compute stream, U-Net tiles of chunk k-1's
blocks on a segmentation stream, D2H of the outputs -- ordered by events,
no host threads.  Stage timings mirror _StageTimer (pipeline.py:133-142).
"""
from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

import numpy as np

from . import motion as M
from . import unet as U
from .stage import HostStage, StageConfig
from .summarize import SummaryPair
from .video import Video


MIN_STAGE_SECONDS = 1e-3  # evaluate.py:16


@dataclass
class ThroughputReport:
    """evaluate.py:83-101: per-stage wall seconds, the run's total, frames/s
    and the ratio to the recording's real-time frame rate."""
    stage_seconds: dict
    total_seconds: float
    frames: int
    effective_fps: float
    target_fps: float | None = None
    realtime_ratio: float | None = None

    def to_json(self) -> str:
        keys = ("stage_seconds", "total_seconds", "frames", "effective_fps", "target_fps", "realtime_ratio")
        return json.dumps({k: getattr(self, k) for k in keys}, indent=2)


def throughput_report(frames: int, stage_seconds: dict, target_fps: float | None = None,
                      total_seconds: float | None = None) -> ThroughputReport:
    """evaluate.py:103-125.  The total defaults to the sum of the stages (pass
    it explicitly when stages overlap); totals under 1 ms clamp to 1 ms."""
    total = sum(stage_seconds.values()) if total_seconds is None else total_seconds
    total = max(total, MIN_STAGE_SECONDS)
    fps = frames / total
    return ThroughputReport(stage_seconds=dict(stage_seconds), total_seconds=total, frames=frames,
                            effective_fps=fps, target_fps=target_fps,
                            realtime_ratio=fps / target_fps if target_fps else None)


@dataclass
class SegmentationResult:
    """The fields of the reference's PipelineResult this path produces."""
    vectors: list = field(default_factory=list)              # list[MotionVector]
    pairs: list = field(default_factory=list)                # list[SummaryPair]
    probability_maps: list = field(default_factory=list)     # list[ProbabilityMap]
    corrected: Video | None = None
    seconds: dict = field(default_factory=dict)              # {"motion+segment": wall seconds}
    throughput: ThroughputReport | None = None               # pipeline.py:171-172


def run_motion_and_segment(video, weights: U.WeightBundle, *, patch_size: int = M.DEFAULT_PATCH_SIZE,
                           search_radius: int = M.DEFAULT_SEARCH_RADIUS, subpixel: bool = True,
                           segment_length: int = 50, smooth_sigma: float = 3.0, unet_stride: int = U.DEFAULT_STRIDE,
                           ref_frames: int | None = None, return_corrected: bool = False,
                           device: int | None = None, chunk_frames: int = 0) -> SegmentationResult:
    """correct_motion -> summarize_segment -> normalize_pair -> tile_and_merge
    for every segment (pipeline.py:198-224), one device pass."""
    v = Video.wrap(video)
    cfg = StageConfig(patch_size=patch_size, search_radius=search_radius, subpixel=subpixel,
                      ref_frames=ref_frames, segment_length=segment_length, sigma=smooth_sigma)
    hs = HostStage(v.height, v.width, cfg, device=device, chunk_frames=chunk_frames)
    try:
        hs.attach_unet(weights, unet_stride)
        t0 = time.perf_counter()
        rec, sp, tp, prob, corr = hs.run_segment(v.samples, corrected=return_corrected)
        dt = time.perf_counter() - t0
    finally:
        hs.close()
    res = SegmentationResult()
    res.vectors = M._vectors_from_numpy(rec)
    res.pairs = [SummaryPair(i, sp[i], tp[i]) for i in range(sp.shape[0])]
    res.probability_maps = [U.ProbabilityMap(i, prob[i]) for i in range(prob.shape[0])]
    res.corrected = Video(corr, frame_rate=v.frame_rate) if corr is not None else None
    res.seconds = {"motion+segment": dt}  # one overlapped device pass: the stages share their wall time
    res.throughput = throughput_report(v.frames, res.seconds, v.frame_rate, total_seconds=dt)
    return res
