"""Frame-balanced time shards on the CUDA path: W ranks (gloo,
all on cuda:0 -- every ordering token is host-mediated, no kernel waits on
another rank) run BalancedShardedPreprocessor with the C-ABI entry points
vb_block_piece / vb_block_finish for the blocks that straddle ranks, both
with the peer-memory exchange (the sender's kernels write into the owner's
IPC-mapped buffers) and with point-to-point sends; the gathered outputs must
equal the single-device run bit for bit (vectors, corrected frames, spatial
and temporal summaries), with and without the A17 options, on two
consecutive runs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_16438_b200 import distributed, synth
from paper_2403_16438_b200 import _device as D
from paper_2403_16438_b200.stage import DevicePreprocessor, StageConfig

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg(radius, L, m, win, shading):
    return StageConfig(search_radius=radius, segment_length=L, ref_frames=m, highpass_window=win,
                       shading_sigma=shading)


def _streamed_run(runner, raw_local, s, m, corr, piece):
    """The second run with the shard uploaded in pieces on a side stream and
    run(arrival=...) waiting per piece (bench.py's strong-scaling e2e)."""
    host = torch.from_numpy(raw_local.view(np.int16)).pin_memory()
    dev = torch.empty(host.shape, dtype=torch.int16, device="cuda")
    up = torch.cuda.Stream()
    up.wait_stream(torch.cuda.current_stream())
    evs = []
    with torch.cuda.stream(up):
        for a in range(0, host.shape[0], piece):
            b = min(host.shape[0], a + piece)
            dev[a:b].copy_(host[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(up)
            evs.append((a, b, ev))

    def arrival(a, b):
        for x, y, ev in evs:
            if x < b and y > a:
                torch.cuda.current_stream().wait_event(ev)

    return runner.run(dev.view(torch.uint16), s, m, corrected_out=corr, arrival=arrival, chunk=piece)


def _worker(rank, world, port, raw, radius, L, m, win, shading, out_dir, exchange="peer"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    exchange, _, piece = exchange.partition("+stream")
    try:
        t, h, w = raw.shape
        s = distributed.balanced_plan(t, L, world, rank, win)
        runner = distributed.BalancedShardedPreprocessor(h, w, _cfg(radius, L, m, win, shading), exchange=exchange)
        local = D.as_device_frames(raw[s.local_lo:s.local_hi], torch.device("cuda", 0))
        corr = torch.empty((s.frames, h, w), dtype=torch.float32, device="cuda")
        # two runs: the second reuses the exchange buffers (peer mode: ACK-ordered overwrite)
        first = runner.run(local, s, m, corrected_out=corr)
        first_tp = first.temporal.clone()
        if piece:  # "+stream<n>": the second run streams its shard in n-frame pieces
            res = _streamed_run(runner, np.ascontiguousarray(raw[s.local_lo:s.local_hi]), s, m, corr, int(piece))
        else:
            res = runner.run(local, s, m, corrected_out=corr)
        assert torch.equal(first_tp, res.temporal), "second run differs"
        vec = D.motion_to_numpy(res.vectors, res.n_frames)[s.frame_lo - s.local_lo:s.frame_hi - s.local_lo]
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), vec=vec, sp=res.spatial.cpu().numpy(),
                 tp=res.temporal.cpu().numpy(), corr=corr.cpu().numpy(), lo=s.block_lo, hi=s.block_hi)
        runner.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T,L,W,m,win,shading,exchange", [
    (600, 100, 4, 150, 0, 0.0, "peer"),   # C2-like: 150-frame shards, blocks straddle every boundary
    (600, 100, 4, 150, 0, 0.0, "p2p"),    # same, buffers sent point-to-point
    (300, 128, 5, 100, 0, 0.0, "peer"),   # 60-frame shards: a block spans three ranks (middle relay)
    (300, 128, 5, 100, 0, 0.0, "p2p"),
    (500, 128, 3, 100, 33, 16.0, "peer"),  # A17 high-pass halo + shading gain through the pieces
    (122, 40, 2, 100, 0, 0.0, "peer"),    # 2-frame final block
    (600, 100, 4, 150, 0, 0.0, "peer+stream37"),  # streamed shard: search per piece, whole blocks as they complete
    (300, 128, 5, 100, 0, 0.0, "p2p+stream50"),
    (400, 100, 1, 150, 0, 0.0, "peer+stream64"),  # one rank: every block whole, summarised during the upload
    (500, 128, 3, 100, 33, 16.0, "peer+stream40"),  # streamed with the A17 halo: a block waits for its halo
    (500, 128, 1, 100, 33, 0.0, "p2p+stream64"),  # pieces end on block ends: the halo must still be waited for
])
@pytest.mark.timeout(300)
def test_balanced_shards_equal_single_run(cuda, tmp_path, T, L, W, m, win, shading, exchange):
    cfg = synth.CONFIGS["c1"].with_frames(T)
    raw = synth.generate_numpy(cfg)
    pre = DevicePreprocessor(cfg.height, cfg.width, _cfg(cfg.radius, L, m, win, shading))
    frames = D.as_device_frames(raw, cuda)
    corr_full = torch.empty(frames.shape, dtype=torch.float32, device=cuda)
    full = pre.run(frames, corrected_out=corr_full)
    want_vec = full.vectors_numpy()
    want_sp, want_tp = full.spatial.cpu().numpy(), full.temporal.cpu().numpy()
    want_corr = corr_full.cpu().numpy()
    pre.close()
    del frames, corr_full
    torch.cuda.synchronize()
    mp.start_processes(_worker, args=(W, _free_port(), raw, cfg.radius, L, m, win, shading, str(tmp_path), exchange),
                       nprocs=W, start_method="spawn")
    sp, tp, corr, vec = {}, {}, [], []
    for r in range(W):
        z = np.load(tmp_path / f"r{r}.npz")
        for i, b in enumerate(range(int(z["lo"]), int(z["hi"]))):
            sp[b], tp[b] = z["sp"][i], z["tp"][i]
        corr.append(z["corr"])
        vec.append(z["vec"])
    np.testing.assert_array_equal(np.concatenate(vec), want_vec)
    np.testing.assert_array_equal(np.concatenate(corr), want_corr)
    assert sorted(sp) == list(range(want_sp.shape[0]))
    for b in sp:
        np.testing.assert_array_equal(sp[b], want_sp[b])
        np.testing.assert_array_equal(tp[b], want_tp[b])


def test_block_piece_and_finish_equal_summarize(cuda):
    """One block split into three pieces on one device == vb_summarize of it."""
    from paper_2403_16438_b200 import _lib
    from paper_2403_16438_b200.summarize import summarize_device

    cfg = synth.CONFIGS["c1"].with_frames(90)
    raw = synth.generate_numpy(cfg)
    frames = D.as_device_frames(raw, cuda)
    pre = DevicePreprocessor(cfg.height, cfg.width, StageConfig(search_radius=cfg.radius, segment_length=90,
                                                                ref_frames=50))
    res = pre.run(frames)
    ops = distributed.DeviceOps(pre)
    sm = torch.empty((90, cfg.height, cfg.width), dtype=torch.float32, device=cuda)
    acc = torch.zeros((cfg.height, cfg.width), dtype=torch.float64, device=cuda)
    for a, b in [(0, 17), (17, 61), (61, 90)]:
        ops.piece(frames[a:b], ops.vec_slice(res.vectors, a, b), 0, b - a, None, sm[a:b], acc)
    sp, tp = ops.finish(sm, 0, 0, 90, 90, acc)
    np.testing.assert_array_equal(sp.cpu().numpy(), res.spatial.cpu().numpy())
    np.testing.assert_array_equal(tp.cpu().numpy(), res.temporal.cpu().numpy())
    with pytest.raises(ValueError, match="at least 2 frames"):
        _lib.call("vb_block_finish", sm.data_ptr(), 0, 90, 0, 1, 90, 0, cfg.height, cfg.width, acc.data_ptr(),
                  sp.data_ptr(), tp.data_ptr(), D.stream_handle())
    with pytest.raises(ValueError, match="not in the smoothed buffer"):
        _lib.call("vb_block_finish", sm.data_ptr(), 10, 80, 0, 90, 90, 0, cfg.height, cfg.width, acc.data_ptr(),
                  sp.data_ptr(), tp.data_ptr(), D.stream_handle())
    pre.close()
