"""Where the drop-in API's time goes on C2 (stage.preprocess, corrected video
returned): host staging copy rate vs threads, pinned vs pageable input,
with / without the corrected video, Python-side result construction."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2403_16438_b200 import Video, _lib, motion, stage, synth  # noqa: E402

cfg = synth.CONFIGS["c2"]
dev = torch.device("cuda", 0)
frames = synth.generate(cfg, dev)
host_np = frames.view(torch.int16).cpu().numpy().view(np.uint16)
pinned = frames.view(torch.int16).cpu().pin_memory()
del frames
torch.cuda.empty_cache()
out = {}
L = _lib.load()
src = host_np[:1000]
dst = stage.pinned_empty((1000, 256, 512), np.uint16)
for nt in (1, 2, 4, 8, 12, 16):
    L.vb_host_copy(dst.ctypes.data, src.ctypes.data, src.nbytes, nt)
    t0 = time.perf_counter()
    for _ in range(5):
        L.vb_host_copy(dst.ctypes.data, src.ctypes.data, src.nbytes, nt)
    out[f"host_copy_GBps_{nt}thr"] = 5 * src.nbytes / (time.perf_counter() - t0) / 1e9
scfg = stage.StageConfig(search_radius=cfg.radius, segment_length=cfg.segment_length, ref_frames=cfg.ref_frames)


def timeit(name, fn, n=5):
    fn()
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    out[name] = cfg.frames * n / (time.perf_counter() - t0)


hs = stage.cached_host_stage(dev, cfg.height, cfg.width, scfg)
timeit("hoststage_pageable_nocorr", lambda: hs.run(host_np, corrected=False))
timeit("hoststage_pageable_corr", lambda: hs.run(host_np, corrected=True))
pin_np = pinned.numpy().view(np.uint16)
timeit("hoststage_pinned_corr", lambda: hs.run(pin_np, corrected=True))
timeit("hoststage_pinned_nocorr", lambda: hs.run(pin_np, corrected=False))
timeit("preprocess_pageable_corr", lambda: stage.preprocess(Video(host_np), scfg, return_corrected=True))
rec = hs.run(host_np, corrected=False)[0]
t0 = time.perf_counter()
motion._vectors_from_numpy(rec)
out["vectors_from_numpy_ms"] = 1e3 * (time.perf_counter() - t0)
t0 = time.perf_counter()
Video(host_np)
out["video_wrap_ms"] = 1e3 * (time.perf_counter() - t0)
print(json.dumps(out, indent=1))
