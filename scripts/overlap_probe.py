"""Search/summaries concurrency probe: DevicePreprocessor on C2 with the
summaries of chunk k on a side stream while chunk k+1 is searched
(overlap_blocks), with and without capping the search kernel's residency."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2403_16438_b200 import synth  # noqa: E402
from paper_2403_16438_b200.stage import DevicePreprocessor, StageConfig  # noqa: E402

cfg = synth.CONFIGS["c2"].with_frames(4000)
dev = torch.device("cuda", 0)
frames = synth.generate(cfg, dev)
pre = DevicePreprocessor(cfg.height, cfg.width, StageConfig(search_radius=8, segment_length=1000, ref_frames=100))
corr = torch.empty(frames.shape, dtype=torch.float32, device=dev)
out = {}
for ob in (0, 1, 2):
    pre.overlap_blocks = ob
    for _ in range(2):
        pre.run(frames, corrected_out=corr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pre.run(frames, corrected_out=corr)
    e1.record()
    torch.cuda.synchronize()
    out[f"overlap_{ob}"] = e0.elapsed_time(e1) / 5
print(json.dumps(out))
