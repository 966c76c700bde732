"""B200-native preprocessing stage of arXiv 2403.16438 (voltseg): per-frame
rigid motion correction -> per-time-block summary images.

Drop-in for voltseg.motion / voltseg.summarize / voltseg.kernels; compute runs
in libvoltb200.so (hand-written sm_100a CUDA behind a C ABI, include/voltb200.h).
"""
from . import kernels, motion, summarize, traces  # noqa: F401
from .motion import (MotionConfig, MotionVector, PatchGrid, correct_frame, correct_motion,  # noqa: F401
                     estimate_motion, make_reference, translate)
from .stage import DevicePreprocessor, HostStage, StageConfig, preprocess  # noqa: F401
from .summarize import SummaryPair, TimeSegment, split_segments  # noqa: F401
from .summarize import summarize as summarize_video  # noqa: F401
from .video import Video  # noqa: F401

__all__ = ["motion", "summarize", "kernels", "traces", "Video", "MotionConfig", "MotionVector", "PatchGrid",
           "correct_motion", "estimate_motion", "make_reference", "translate", "correct_frame",
           "split_segments", "SummaryPair", "TimeSegment", "summarize_video", "preprocess",
           "DevicePreprocessor", "HostStage", "StageConfig"]
