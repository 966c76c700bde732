"""Motion-search A/B on a BASELINE config: per-kernel device time (CUDA events
on the launching stream, vb_prof) and the vectors, saved for comparison.

  python scripts/ab_search.py CONFIG FRAMES TAG   (-> gpurun_out/ab_<TAG>_<CONFIG>.npz / .json)
Run the experiment build with switches through VB_LIBRARY=.../libvoltb200_exp.so."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2403_16438_b200 import _device as D  # noqa: E402
from paper_2403_16438_b200 import _lib, synth  # noqa: E402
from paper_2403_16438_b200.motion import MotionPlan, PatchGrid, device_reference  # noqa: E402

name, nfr, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
cfg = synth.CONFIGS[name].with_frames(nfr)
dev = torch.device("cuda", 0)
frames = synth.generate(cfg, dev)
ref = device_reference(frames, cfg.ref_frames)
g = PatchGrid.cover(cfg.height, cfg.width, 21, margin=cfg.radius)
plan = MotionPlan(cfg.height, cfg.width, g.origins, 21, cfg.radius)
plan.set_reference(ref)
L = _lib.load()
vec, sc = plan.estimate(frames, True, scores=True)
for _ in range(2):
    plan.estimate(frames, True)
torch.cuda.synchronize()
L.vb_prof_enable(1)
reps = 3
for _ in range(reps):
    plan.estimate(frames, True)
torch.cuda.synchronize()
ms = np.zeros(5)
cnt = np.zeros(5, np.int64)
L.vb_prof_collect(ms.ctypes.data, cnt.ctypes.data, 5)
L.vb_prof_enable(0)
out = {"tag": tag, "config": name, "frames": nfr, "info": plan.info(),
       "ms_per_1000": {k: float(ms[i] / reps / nfr * 1000) for i, k in enumerate(["search", "finalize", "warp", "median", "other"])}}
S = 2 * cfg.radius + 1
out["search_tflops"] = 2.0 * len(g.origins) * S * S * 441 * nfr * reps / (ms[0] / 1e3) / 1e12
p2, p1 = _lib.C.c_double(), _lib.C.c_double()
L.vb_fp32_peak_probe(_lib.C.byref(p2), _lib.C.byref(p1))
out["fp32_frac"] = out["search_tflops"] / max(p2.value, p1.value)
rec = D.motion_to_numpy(vec, nfr)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
np.savez(ROOT / "gpurun_out" / f"ab_{tag}_{name}.npz", rec=rec, scores=sc.cpu().numpy()[: min(nfr, 64)])
print(json.dumps(out))
