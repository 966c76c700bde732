"""Per-call timing of the U-Net entry points (diagnostic; runs under gpurun)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2403_16438_b200 import _lib, stage, synth, unet  # noqa: E402
from paper_2403_16438_b200 import _device as D  # noqa: E402

torch.cuda.set_device(0)
with_stage = "--stage" in sys.argv
k, h, w = 10, 256, 512
if with_stage:
    cfg = synth.CONFIGS["c2"]
    frames = synth.generate(cfg, torch.device("cuda", 0))
    pre = stage.DevicePreprocessor(cfg.height, cfg.width, stage.StageConfig(search_radius=cfg.radius,
                                   segment_length=cfg.segment_length, ref_frames=cfg.ref_frames))
    res = pre.run(frames)
    sp, tp = res.spatial.contiguous(), res.temporal.contiguous()
    del frames
else:
    sp = torch.rand((k, h, w), device='cuda') * 1000
    tp = torch.rand((k, h, w), device='cuda')
net = unet.DeviceUNet(unet.WeightBundle.random(np.random.default_rng(7)))
norm = torch.empty((k, 2, h, w), device='cuda')
prob = torch.empty((k, h, w), device='cuda')
for i in range(3):
    net.segment_device(sp, tp, out=prob)
torch.cuda.synchronize()


def t(f, n=3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print('segment', t(lambda: net.segment_device(sp, tp, out=prob)))
print('normalize', t(lambda: _lib.call("vb_normalize_pair", sp.data_ptr(), tp.data_ptr(), k, h, w, norm.data_ptr(),
                                        D.stream_handle())))
print('tile_merge', t(lambda: net.tile_merge_device(norm, out=prob)))
pat = torch.rand((1050, 2, 64, 64), device='cuda')
pr = torch.empty((1050, 64, 64), device='cuda')
print('forward 1050', t(lambda: net.forward_device(pat, out=pr)))
