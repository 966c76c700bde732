"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of libvoltb200 on C1-sized data --
the C-ABI executor (template, window statistics, TMA search, finalize,
warp + TMA smoothing, block mean, median), the device path, float32 input,
the operator entry, A17 options, fused traces, the U-Net segmentation and,
with --ipc, the frame-balanced peer-memory exchange between two processes
(CUDA IPC).  Run by scripts/sanitize.sh; exits non-zero on any failure."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2403_16438_b200 import Video, distributed, kernels, stage, synth, traces, unet  # noqa: E402
from paper_2403_16438_b200 import _device as D  # noqa: E402


def main_single(frames):
    cfg = synth.CONFIGS["c1"].with_frames(frames)
    raw = synth.generate_numpy(cfg)
    sc = stage.StageConfig(search_radius=cfg.radius, segment_length=30, ref_frames=20)
    hs = stage.HostStage(128, 128, sc, chunk_frames=30)
    vec, sp, tp, corr = hs.run(raw, corrected=True)                      # executor, u16
    hs.run(raw.astype(np.float32), corrected=False)                      # executor, f32
    hs.close()
    dp = stage.DevicePreprocessor(128, 128, sc)
    res = dp.run(D.as_device_frames(raw), corrected_out=torch.empty((frames, 128, 128), device="cuda"))
    dp.close()
    g = synth.CONFIGS["c1"]
    kernels.mean_zncc_scores(raw[0].astype(np.float32), raw[1].astype(np.float32),
                             np.array([[10, 10], [40, 50]], np.int32), 21, g.radius)   # operator
    sc2 = stage.StageConfig(search_radius=cfg.radius, segment_length=30, ref_frames=20, highpass_window=9,
                            shading_sigma=16.0)
    stage.preprocess(Video(raw), sc2)                                    # A17 options
    mask = np.zeros((128, 128), bool)
    mask[40:52, 30:45] = True
    traces.extract_traces_raw_device(D.as_device_frames(raw), res.vectors, [mask])
    net = unet.DeviceUNet(unet.WeightBundle.random(np.random.default_rng(7)))
    net.segment_device(res.spatial.contiguous(), res.temporal.contiguous())
    net.close()
    torch.cuda.synchronize()
    print("single-process workload ok", vec.shape, sp.shape)


def _ipc_worker(rank, world, port, raw):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t, h, w = raw.shape
    s = distributed.balanced_plan(t, 30, world, rank)
    runner = distributed.BalancedShardedPreprocessor(h, w, stage.StageConfig(search_radius=5, segment_length=30,
                                                                              ref_frames=20), exchange="peer")
    local = D.as_device_frames(raw[s.local_lo:s.local_hi], torch.device("cuda", 0))
    runner.run(local, s, 20)
    runner.run(local, s, 20)
    torch.cuda.synchronize()
    runner.close()
    dist.destroy_process_group()


def main_ipc(frames):
    import torch.multiprocessing as mp

    raw = synth.generate_numpy(synth.CONFIGS["c1"].with_frames(frames))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.start_processes(_ipc_worker, args=(2, port, raw), nprocs=2, join=True, start_method="spawn")
    print("ipc workload ok")


if __name__ == "__main__":
    n = int(os.environ.get("SAN_FRAMES", "60"))
    (main_ipc if "--ipc" in sys.argv else main_single)(n)
