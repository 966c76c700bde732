"""Small tensor-core motion-search run for ncu (experiment build, VB_ZNCC_MMA=1)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2403_16438_b200 import synth  # noqa: E402
from paper_2403_16438_b200.motion import MotionPlan, PatchGrid, device_reference  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"].with_frames(1024)
dev = torch.device("cuda", 0)
frames = synth.generate(cfg, dev)
ref = device_reference(frames, cfg.ref_frames)
g = PatchGrid.cover(cfg.height, cfg.width, 21, margin=cfg.radius)
plan = MotionPlan(cfg.height, cfg.width, g.origins, 21, cfg.radius)
plan.set_reference(ref)
for _ in range(2):
    plan.estimate(frames, True)
torch.cuda.synchronize()
print("ok")
