"""The reference's own correct_motion (oracle/_ref, unmodified) timed with its
native Cython backend and with our operator registered as a voltseg.kernels
backend (runs under gpurun; C2 frames)."""
import json
import os
import sys
import time
import types

import numpy as np

sys.path.insert(0, ".")
from oracle import ref as REF  # noqa: E402
from paper_2403_16438_b200 import kernels as K, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
motion, _s, kernels, video_io = REF.load()
cfg = synth.CONFIGS["c2"].with_frames(n)
video = video_io.Video(synth.generate_numpy(cfg).astype(np.float32), frame_rate=cfg.fps)
motion.REFERENCE_FRAMES = cfg.ref_frames
native = kernels._native
ours = types.SimpleNamespace(mean_zncc_scores=K.mean_zncc_scores)  # in place of the compiled _native
threads = os.cpu_count() or 1
out = {"config": f"c2 {n}x{cfg.height}x{cfg.width}, r={cfg.radius}: reference correct_motion(threads={threads})"}
vecs = {}
for name, thr in (("b200", 1), ("b200", threads), ("native", 1), ("native", threads)):
    kernels.BACKEND = "native"
    kernels._native = ours if name == "b200" else native
    t0 = time.perf_counter()
    _c, v = motion.correct_motion(video, motion.MotionConfig(search_radius=cfg.radius, threads=thr))
    out[f"{name}_threads{thr}_frames_per_s"] = n / (time.perf_counter() - t0)
    vecs[name] = np.array([[x.dx, x.dy] for x in v])
out["integer_shift_mismatches_vs_native"] = int((vecs["b200"] != vecs["native"]).any(axis=1).sum())
print(json.dumps(out))
