"""A full-size BASELINE.json configuration through the C-ABI host executor
(runs under gpurun): the whole uint16 recording (C4: 100,000 x 512 x 512 =
52 GB) in pinned host memory, streamed in 2,048-frame chunks; prints
host-to-host frames/s and checks the first 8,192 frames' vectors and complete
blocks against the device-resident path on the same frames.
Usage: python scripts/full_stream.py [CONFIG=c4] [FRAMES]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_16438_b200 import _lib, stage, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = synth.CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.frames
cfg = cfg.with_frames(n)
check = min(8192, n)
dev = torch.device("cuda", 0)
t_gen = time.perf_counter()
frames = synth.generate(cfg, dev)
head = frames[:check].clone()
host = torch.empty((n, cfg.height, cfg.width), dtype=torch.int16, pin_memory=True)
for f0 in range(0, n, 4096):  # device -> pinned host without a pageable copy
    host[f0:f0 + 4096].copy_(frames[f0:f0 + 4096].view(torch.int16))
del frames
torch.cuda.synchronize()
torch.cuda.empty_cache()
t_gen = time.perf_counter() - t_gen
sc = stage.StageConfig(search_radius=cfg.radius, segment_length=cfg.segment_length, ref_frames=cfg.ref_frames)
hs = stage.HostStage(cfg.height, cfg.width, sc, chunk_frames=2048)
k = -(-n // cfg.segment_length)
vec = np.empty(n, dtype=_lib.MOTION_DTYPE)
sp = np.empty((k, cfg.height, cfg.width), np.float32)
tp = np.empty_like(sp)
hs.run_into(host.data_ptr(), _lib.VB_U16, check, vec[:check], sp[:-(-check // cfg.segment_length)],
            tp[:-(-check // cfg.segment_length)])  # warm-up (ring allocation)
torch.cuda.synchronize()
t0 = time.perf_counter()
hs.run_into(host.data_ptr(), _lib.VB_U16, n, vec, sp, tp)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
pre = stage.DevicePreprocessor(cfg.height, cfg.width, sc)
res = pre.run(head)
nb = check // cfg.segment_length
same = (np.array_equal(res.vectors_numpy(), vec[:check]) and np.array_equal(res.spatial.cpu().numpy()[:nb], sp[:nb])
        and np.array_equal(res.temporal.cpu().numpy()[:nb], tp[:nb]))
print(json.dumps({"config": f"{name} full size: {n}x{cfg.height}x{cfg.width} uint16 "
                            f"({n * cfg.height * cfg.width * 2 / 1e9:.1f} GB) in pinned host memory, r={cfg.radius}, "
                            f"L={cfg.segment_length}, M={cfg.ref_frames}, 2048-frame chunks",
                  "e2e_frames_per_s": n / dt, "seconds": dt, "h2d_GBps": n * cfg.height * cfg.width * 2 / dt / 1e9,
                  "generation_seconds": t_gen,
                  f"first_{check}_frames_equal_device_path": bool(same), "blocks": k}))
