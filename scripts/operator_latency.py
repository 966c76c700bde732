"""Per-call latency of the operator-level drop-in (kernels.mean_zncc_scores,
the voltseg.kernels contract: host arrays in, float64 grid out), called once
per frame as the reference's correct_motion does (runs under gpurun)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2403_16438_b200 import kernels, motion, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.CONFIGS[name].with_frames(300)
raw = synth.generate_numpy(cfg).astype(np.float32)
ref = raw[:100].astype(np.float64).mean(0).astype(np.float32)
grid = motion.PatchGrid.cover(cfg.height, cfg.width, 21, margin=cfg.radius)
kernels.mean_zncc_scores(raw[0], ref, grid.origins, 21, cfg.radius)
t0 = time.perf_counter()
for f in raw[1:]:
    kernels.mean_zncc_scores(f, ref, grid.origins, 21, cfg.radius)
dt = (time.perf_counter() - t0) / (len(raw) - 1)
print(json.dumps({"config": f"{name} {cfg.height}x{cfg.width}, r={cfg.radius}", "ms_per_call": dt * 1e3,
                  "calls_per_s": 1 / dt}))
