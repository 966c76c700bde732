"""C4-geometry streaming check (runs under gpurun): a 512x512 uint16 recording
in pinned host memory streamed through the C-ABI executor in 2,048-frame
chunks (BASELINE.json configs[3]); prints host-to-host frames/s and checks the
outputs against the device-resident path on the same frames."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_16438_b200 import _lib, stage, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cfg = synth.CONFIGS["c4"].with_frames(n)
dev = torch.device("cuda", 0)
frames = synth.generate(cfg, dev)
host = frames.view(torch.int16).cpu().pin_memory()
sc = stage.StageConfig(search_radius=cfg.radius, segment_length=cfg.segment_length, ref_frames=cfg.ref_frames)
hs = stage.HostStage(cfg.height, cfg.width, sc, chunk_frames=2048)
k = -(-n // cfg.segment_length)
vec = np.empty(n, dtype=_lib.MOTION_DTYPE)
sp = np.empty((k, cfg.height, cfg.width), np.float32)
tp = np.empty_like(sp)
hs.run_into(host.data_ptr(), _lib.VB_U16, n, vec, sp, tp)  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
reps = 2
for _ in range(reps):
    hs.run_into(host.data_ptr(), _lib.VB_U16, n, vec, sp, tp)
torch.cuda.synchronize()
fps = n * reps / (time.perf_counter() - t0)
pre = stage.DevicePreprocessor(cfg.height, cfg.width, sc)
res = pre.run(frames)
same = (np.array_equal(res.vectors_numpy(), vec) and np.array_equal(res.spatial.cpu().numpy(), sp)
        and np.array_equal(res.temporal.cpu().numpy(), tp))
print(json.dumps({"config": f"c4 geometry: {n}x{cfg.height}x{cfg.width} uint16, r={cfg.radius}, L={cfg.segment_length}, "
                            "2048-frame chunks from pinned host memory",
                  "e2e_frames_per_s": fps, "h2d_GBps": fps * cfg.height * cfg.width * 2 / 1e9,
                  "executor_equals_device_path": bool(same)}))
