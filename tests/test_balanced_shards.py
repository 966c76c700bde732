"""Frame-balanced time shards with blocks straddling ranks.

CPU: the plan's invariants (every frame summarised once, every block owned
once, contributors chained in recording order) and the whole protocol --
template all-reduce, tail pieces sent forward over gloo while whole blocks
are summarised, the float64 running sum continued across ranks, head blocks
finished by the owner -- with the kernels replaced by the CPU oracle, so the
sharded outputs must equal oracle.preprocess on the whole recording bit for
bit.  GPU: tests/test_gpu_balanced.py runs the same protocol on the CUDA
entry points."""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_16438_b200 import distributed, synth


@pytest.mark.parametrize("T,L,W,win", [(10000, 1000, 8, 0), (1000, 100, 3, 0), (250, 100, 4, 0),
                                       (95, 40, 7, 0), (122, 40, 2, 0), (300, 64, 5, 33), (8, 3, 8, 0), (5, 3, 8, 0)])
def test_balanced_plan_invariants(T, L, W, win):
    hh = win // 2
    k = -(-T // L)
    owned, frames = [], []
    contrib = {b: [] for b in range(k)}
    for r in range(W):
        s = distributed.balanced_plan(T, L, W, r, win)
        frames.extend(range(s.frame_lo, s.frame_hi))
        owned.extend(range(s.block_lo, s.block_hi))
        assert s.local_lo == max(0, s.frame_lo - hh) and s.local_hi == min(T, s.frame_hi + hh)
        if s.whole_hi > s.whole_lo:
            assert s.whole_lo % L == 0 and (s.whole_hi % L == 0 or s.whole_hi == T)
            assert s.frame_lo <= s.whole_lo and s.whole_hi <= s.frame_hi
        for p in (s.head, s.tail):
            if p is None:
                continue
            contrib[p.block].append((r, p))
            assert s.local_lo <= p.c_lo <= p.c_hi <= s.local_hi  # smoothed frames are local
            assert p.c_lo <= p.m_lo <= p.m_hi <= p.c_hi
            assert p.s_lo == max(0, p.t0 - hh) and p.s_hi == min(T, p.t1 + hh)
        # summarised frames: whole blocks + own frames of the pieces == the shard
        mine = set(range(s.whole_lo, s.whole_hi))
        for p in (s.head, s.tail):
            if p is not None:
                mine |= set(range(p.m_lo, p.m_hi))
        assert mine == set(range(s.frame_lo, s.frame_hi))
    assert frames == list(range(T))
    assert owned == list(range(k))
    for b, cs in contrib.items():
        if not cs:
            continue
        cs.sort(key=lambda x: x[0])
        assert cs[0][1].role == "first" and cs[-1][1].role == "last"
        assert all(p.role == "middle" for _, p in cs[1:-1])
        for (ra, pa), (rb, pb) in zip(cs, cs[1:]):
            assert pa.next == rb and pb.prev == ra and pa.c_hi == pb.c_lo  # chained in recording order
        assert cs[0][1].c_lo == cs[0][1].s_lo and cs[-1][1].c_hi == cs[-1][1].s_hi


def test_one_frame_tail_raises_like_reference():
    with pytest.raises(ValueError, match="at least 2 frames"):
        distributed.balanced_plan(121, 40, 2, 0)


# ---------------------------------------------------------------- protocol over gloo, oracle kernels
class OracleOps:
    """CPU stand-in for distributed.DeviceOps built from oracle/ (test infrastructure)."""

    def __init__(self, oracle_mod, h, w, radius, L):
        self.O = oracle_mod
        self.origins = oracle_mod.patch_grid(h, w, 21, radius)
        self.radius, self.L = radius, L
        self.cfg = SimpleNamespace(segment_length=L)

    def template(self, frames, lo, hi, m, group):
        tsum = torch.zeros(frames.shape[1:], dtype=torch.float64)
        for f in frames[lo:hi]:
            tsum += f.double()
        distributed.allreduce_sum_(tsum, group)
        self.ref = (tsum.numpy() / m).astype(np.float32)

    def estimate(self, frames, arrival=None, chunk=0, after=None):
        vec = np.zeros((frames.shape[0], 5), np.float64)
        step = chunk if arrival is not None and chunk > 0 else frames.shape[0]
        for a in range(0, frames.shape[0], max(step, 1)):
            b = min(frames.shape[0], a + step)
            if arrival is not None:
                arrival(a, b)
            vec[a:b] = np.array([self.O.estimate_motion(f.numpy(), self.ref, self.origins, 21, self.radius)
                                 for f in frames[a:b]], dtype=np.float64).reshape(-1, 5)
            if after is not None:
                after(vec, b)
        return vec

    @staticmethod
    def vec_slice(vec, a, b):
        return vec[a:b]

    def _correct(self, frames, vec):
        return [self.O.correct_frame(f.numpy(), v[0] + v[2], v[1] + v[3]) for f, v in zip(frames, vec)]

    def frames_buffer(self, n, like):
        return torch.empty((n,) + tuple(like.shape[1:]), dtype=torch.float32)

    def sum_buffer(self, like):
        return torch.zeros(tuple(like.shape[1:]), dtype=torch.float64)

    def whole(self, frames, vec, t_global0, t_total, interior, corrected_out):
        off, n = interior
        corr = np.stack(self._correct(frames[off:off + n], vec[off:off + n]))
        if corrected_out is not None:
            corrected_out.copy_(torch.from_numpy(corr))
        sp, tp = [], []
        for b0 in range(0, n, self.L):
            blk = corr[b0:b0 + self.L]
            sp.append(self.O.spatial_summary(blk))
            tp.append(self.O.temporal_summary(blk))
        return torch.from_numpy(np.stack(sp)), torch.from_numpy(np.stack(tp))

    def piece(self, frames, vec, mean_off, mean_n, corrected_out, smoothed, partial):
        corr = self._correct(frames, vec)
        for i, c in enumerate(corr):
            smoothed[i] = torch.from_numpy(self.O.smooth_frame(c))
        for i in range(mean_off, mean_off + mean_n):
            partial += torch.from_numpy(corr[i]).double()  # sequential float64 adds, frame order
            if corrected_out is not None:
                corrected_out[i - mean_off] = torch.from_numpy(corr[i])

    def finish(self, smoothed, s_lo, t0, count, t_total, partial):
        sp = (partial.numpy() / count).astype(np.float32)
        blk = smoothed.numpy()[t0 - s_lo:t0 - s_lo + count]
        o = np.sort(blk, axis=0)
        mid = count // 2
        med = o[mid] if count % 2 else ((o[mid - 1] + o[mid]) * np.float32(0.5)).astype(np.float32)
        tp = (blk.max(axis=0) - med).astype(np.float32)
        return torch.from_numpy(sp[None]), torch.from_numpy(tp[None])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, raw, L, m, radius, out_dir, piece=0):
    from oracle import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t, h, w = raw.shape
        s = distributed.balanced_plan(t, L, world, rank)
        ops = OracleOps(O, h, w, radius, L)
        runner = distributed.BalancedShardedPreprocessor(h, w, ops=ops)
        local = torch.from_numpy(raw[s.local_lo:s.local_hi].astype(np.float32))
        corr = torch.empty((s.frames, h, w), dtype=torch.float32)
        if piece:  # streamed upload protocol: arrival(a, b) requests, in order, before use
            asked = []
            res = runner.run(local, s, m, corrected_out=corr, arrival=lambda a, b: asked.append((a, b)),
                             chunk=piece)
            n = s.local_hi - s.local_lo
            pieces = [(a, min(n, a + piece)) for a in range(0, n, piece)]
            assert asked[-1] == (0, n) and asked[-1 - len(pieces):-1] == pieces, asked
            assert len(asked) in (len(pieces) + 1, len(pieces) + 2)  # + the template rows, if any
            if len(asked) == len(pieces) + 2:
                assert 0 <= asked[0][0] < asked[0][1] <= n
        else:
            res = runner.run(local, s, m, corrected_out=corr)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), vec=res.vectors, sp=res.spatial.numpy(),
                 tp=res.temporal.numpy(), corr=corr.numpy(), lo=s.block_lo, hi=s.block_hi)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T,L,W,m,piece", [(122, 40, 2, 100, 0), (100, 30, 3, 50, 0), (90, 60, 4, 20, 0),
                                            (122, 40, 2, 100, 7), (100, 30, 1, 50, 13)])
def test_balanced_protocol_matches_oracle(tmp_path, oracle_mod, T, L, W, m, piece):
    """Sharded (gloo, W ranks, blocks straddling ranks -- incl. a block spread
    over three ranks for (90, 60, 4)) == oracle.preprocess of the whole recording;
    piece > 0: the streamed-upload protocol (run(arrival=..., chunk=piece):
    search per piece, whole blocks summarised as they complete)."""
    cfg = synth.CONFIGS["c1"].with_frames(T)
    raw = synth.generate_numpy(cfg)
    radius = cfg.radius
    mp.start_processes(_worker, args=(W, _free_port(), raw, L, m, radius, str(tmp_path), piece), nprocs=W,
                       start_method="spawn")
    want = oracle_mod.preprocess(raw.astype(np.float32), 21, radius, True, m, L, 3.0)
    sp, tp, corr, vec = {}, {}, [], []
    for r in range(W):
        z = np.load(tmp_path / f"r{r}.npz")
        for i, b in enumerate(range(int(z["lo"]), int(z["hi"]))):
            sp[b], tp[b] = z["sp"][i], z["tp"][i]
        corr.append(z["corr"])
        vec.append(z["vec"])
    vec = np.concatenate(vec)
    np.testing.assert_array_equal(vec[:, :2].astype(np.int32), want["dxdy"])
    np.testing.assert_array_equal(np.concatenate(corr), want["corrected"])
    k = -(-T // L)
    assert sorted(sp) == list(range(k))
    for b in range(k):
        np.testing.assert_array_equal(sp[b], want["spatial"][b])
        np.testing.assert_array_equal(tp[b], want["temporal"][b])
