"""Trace extraction on C2 (runs under gpurun): traces from the raw frames +
motion vectors (warp fused, vb_extract_traces_raw) vs correcting the whole
video and then extracting (vb_correct_frames + vb_extract_traces)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_16438_b200 import motion as M, synth, traces  # noqa: E402

cfg = synth.CONFIGS["c2"].with_frames(4000)
dev = torch.device("cuda", 0)
frames, truth = synth.generate(cfg, dev, return_truth=True)
grid = M.PatchGrid.cover(cfg.height, cfg.width, 21, margin=cfg.radius)
ref = M.device_reference(frames, cfg.ref_frames)
plan = M.MotionPlan(cfg.height, cfg.width, grid.origins, 21, cfg.radius)
plan.set_reference(ref)
vec, _ = plan.estimate(frames, True)
yy, xx = np.mgrid[:cfg.height, :cfg.width]
masks = [((yy - cy) ** 2 + (xx - cx) ** 2) <= 16 for cx, cy in truth.centers]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


from paper_2403_16438_b200 import _device as D, _lib  # noqa: E402

ptr, idx = traces._csr(masks, cfg.height, cfg.width)  # ROI tables built once (host work excluded)
ptr_d, idx_d = torch.from_numpy(ptr).to(dev), torch.from_numpy(idx).to(dev)
k = len(masks)
out = torch.empty((k, cfg.frames), dtype=torch.float64, device=dev)
corr = torch.empty((cfg.frames, cfg.height, cfg.width), dtype=torch.float32, device=dev)


def fused():
    _lib.call("vb_extract_traces_raw", frames.data_ptr(), _lib.VB_U16, vec.data_ptr(), None, cfg.frames, cfg.height,
              cfg.width, ptr_d.data_ptr(), idx_d.data_ptr(), k, out.data_ptr(), D.stream_handle())


def two_step():
    _lib.call("vb_correct_frames", frames.data_ptr(), _lib.VB_U16, cfg.frames, cfg.height, cfg.width, vec.data_ptr(),
              corr.data_ptr(), D.stream_handle())
    _lib.call("vb_extract_traces", corr.data_ptr(), cfg.frames, cfg.height, cfg.width, ptr_d.data_ptr(),
              idx_d.data_ptr(), k, out.data_ptr(), D.stream_handle())


t_raw = timed(fused)
t_two = timed(two_step)
print(json.dumps({"config": f"c2: {cfg.frames}x{cfg.height}x{cfg.width} uint16, {len(masks)} ROIs of "
                            f"{int(np.mean([m.sum() for m in masks]))} px",
                  "fused_ms": t_raw, "correct_then_extract_ms": t_two,
                  "fused_frames_per_s": cfg.frames / t_raw * 1e3}))
