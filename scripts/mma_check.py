"""Tensor-core ZNCC path (uint16 frames) vs the FFMA path (the same frames as
float32) vs the float64 oracle: score grids, integer shifts, timing."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import oracle as O  # noqa: E402
from paper_2403_16438_b200 import _device as D  # noqa: E402
from paper_2403_16438_b200 import synth  # noqa: E402
from paper_2403_16438_b200.motion import MotionPlan, PatchGrid, device_reference  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
nfr = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
cfg = synth.CONFIGS[name].with_frames(nfr)
dev = torch.device("cuda", 0)
u16 = synth.generate(cfg, dev)
f32 = u16.to(torch.float32)
ref = device_reference(u16, cfg.ref_frames)
g = PatchGrid.cover(cfg.height, cfg.width, 21, margin=cfg.radius)
plan = MotionPlan(cfg.height, cfg.width, g.origins, 21, cfg.radius)
plan.set_reference(ref)
out = {"config": name, "frames": nfr}
v_u, s_u = plan.estimate(u16, True, scores=True)
v_f, s_f = plan.estimate(f32, True, scores=True)
torch.cuda.synchronize()
su, sf = s_u.cpu().numpy(), s_f.cpu().numpy()
out["max_score_diff_mma_vs_ffma"] = float(np.abs(su - sf).max())
ru, rf = D.motion_to_numpy(v_u, nfr), D.motion_to_numpy(v_f, nfr)
out["int_mismatch_mma_vs_ffma"] = int(((ru["dx"] != rf["dx"]) | (ru["dy"] != rf["dy"])).sum())
out["max_sub_diff"] = float(max(np.abs(ru["sub_dx"] - rf["sub_dx"]).max(), np.abs(ru["sub_dy"] - rf["sub_dy"]).max()))
raw = u16.view(torch.int16).cpu().numpy().view(np.uint16)
refh = ref.cpu().numpy()
errs_u, errs_f = [], []
for t in range(0, nfr, max(1, nfr // 8)):
    o = O.mean_zncc_scores(raw[t].astype(np.float32), refh, g.origins, 21, cfg.radius)
    errs_u.append(float(np.abs(su[t] - o).max()))
    errs_f.append(float(np.abs(sf[t] - o).max()))
out["max_score_err_vs_oracle_mma"] = max(errs_u)
out["max_score_err_vs_oracle_ffma"] = max(errs_f)
for label, x in (("mma_u16", u16), ("ffma_f32", f32)):
    plan.estimate(x, True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        plan.estimate(x, True)
    torch.cuda.synchronize()
    out[f"ms_per_1000_{label}"] = (time.perf_counter() - t0) / 3 / nfr * 1000 * 1000
print(json.dumps(out, indent=1))
