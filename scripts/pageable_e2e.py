"""Host-to-host throughput of the C-ABI executor from PAGEABLE host memory
(a plain numpy recording, as `HostStage.run` / `preprocess` callers pass it)
vs pinned memory (runs under gpurun)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_16438_b200 import _lib, stage, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.CONFIGS[name]
frames = synth.generate(cfg, torch.device("cuda", 0))
host = frames.view(torch.int16).cpu().numpy().view(np.uint16)  # pageable
pinned = torch.from_numpy(host.view(np.int16)).pin_memory()
del frames
sc = stage.StageConfig(search_radius=cfg.radius, segment_length=cfg.segment_length, ref_frames=cfg.ref_frames)
hs = stage.HostStage(cfg.height, cfg.width, sc)
n = cfg.frames
k = -(-n // cfg.segment_length)
vec = np.empty(n, dtype=_lib.MOTION_DTYPE)
sp = np.empty((k, cfg.height, cfg.width), np.float32)
tp = np.empty_like(sp)
out = {"config": name}
for label, ptr in (("pageable", host.ctypes.data), ("pinned", pinned.data_ptr())):
    hs.run_into(ptr, _lib.VB_U16, n, vec, sp, tp)  # warm-up
    t0 = time.perf_counter()
    for _ in range(3):
        hs.run_into(ptr, _lib.VB_U16, n, vec, sp, tp)
    out[label + "_frames_per_s"] = 3 * n / (time.perf_counter() - t0)
print(json.dumps(out))
