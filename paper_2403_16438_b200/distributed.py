"""Time-sharded preprocessing over several GPUs (one process per GPU).

The stage shards by time with no halo under the reference semantics (there is
no temporal filter): per-frame motion is independent given the
template, and per-block summaries are independent given the block's frames.
Shards are whole blocks, so no block straddles two ranks.  The only exchange
is the template: the float64 per-pixel sum of the recording's first M frames
(motion.py:211-214) is contributed by whichever ranks hold those frames and
summed with one all-reduce (NCCL over NVLink on GPUs, gloo in the CPU tests),
so every rank builds a bit-identical template.  Outputs stay sharded: each
rank owns the vectors of its frames and the summaries of its blocks
(gather_outputs collects them on request).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    frame_lo: int  # global frame range [frame_lo, frame_hi)
    frame_hi: int
    block_lo: int  # global block range [block_lo, block_hi)
    block_hi: int
    n_total: int = 0  # frames in the whole recording

    @property
    def frames(self) -> int:
        return self.frame_hi - self.frame_lo


def shard_plan(n_frames: int, segment_length: int, world: int, rank: int) -> Shard:
    """Contiguous block-aligned shards; blocks split as evenly as possible."""
    if segment_length < 2:
        raise ValueError("segment length must be >= 2")
    k = math.ceil(n_frames / segment_length)
    b0, b1 = k * rank // world, k * (rank + 1) // world
    f0, f1 = min(b0 * segment_length, n_frames), min(b1 * segment_length, n_frames)
    return Shard(rank, world, f0, f1, b0, b1, n_frames)


def halo_range(shard: Shard, highpass_window: int = 0) -> tuple[int, int]:
    """Recording frames [lo, hi) a rank must hold: its shard plus, with the
    opt-in temporal high-pass (A17), the window//2-frame halo on either side
    (clipped to the recording; the filter reflects at its ends)."""
    hh = highpass_window // 2 if highpass_window and highpass_window > 1 else 0
    n = shard.n_total or shard.frame_hi
    return max(0, shard.frame_lo - hh), min(n, shard.frame_hi + hh)


def template_rows(shard: Shard, ref_frames: int, local_lo: int | None = None) -> tuple[int, int]:
    """Local frame range (frames_local[0] = recording frame local_lo, default
    the shard start) of this shard's OWN frames inside the template window
    [0, M) -- halo frames are never counted, so the all-reduced sum counts each
    template frame once."""
    base = shard.frame_lo if local_lo is None else local_lo
    lo = max(shard.frame_lo, 0)
    hi = min(shard.frame_hi, ref_frames)
    if hi <= lo:
        return 0, 0
    return lo - base, hi - base


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all-reduce when running distributed (no-op otherwise)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def gather_outputs(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    """All-gather variable-length leading-dim shards (for collecting results)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [t]
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], device=t.device, dtype=torch.int64)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    m = int(max(s.item() for s in sizes))
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[: int(s.item())] for o, s in zip(outs, sizes)]


class ShardedPreprocessor:
    """Per-rank driver: template sum -> all-reduce -> motion + summaries on the
    local shard (device-resident, the bench's `value` step)."""

    def __init__(self, height: int, width: int, config=None, group=None):
        from . import stage  # noqa: WPS433 (import cycle guard)

        self.pre = stage.DevicePreprocessor(height, width, config)
        self.group = group
        self.height, self.width = height, width

    def template(self, frames_local: torch.Tensor, shard: Shard, ref_frames: int,
                 local_lo: int | None = None) -> torch.Tensor:
        from . import _device as D
        from . import _lib

        h, w = self.height, self.width
        tsum = torch.zeros((h, w), dtype=torch.float64, device=frames_local.device)
        lo, hi = template_rows(shard, ref_frames, local_lo)
        if hi > lo:
            _lib.call("vb_template_sum", frames_local[lo:hi].data_ptr(), D.vb_dtype(frames_local), hi - lo, h, w,
                      tsum.data_ptr(), 0, D.stream_handle())
        allreduce_sum_(tsum, self.group)
        m = min(ref_frames, shard.n_total or shard.frame_hi)
        ref = torch.empty((h, w), dtype=torch.float32, device=frames_local.device)
        _lib.call("vb_template_finish", tsum.data_ptr(), m, h * w, ref.data_ptr(), D.stream_handle())
        return ref

    def run(self, frames_local: torch.Tensor, shard: Shard, ref_frames: int, corrected_out=None,
            local_lo: int | None = None):
        """frames_local = recording frames [local_lo, local_lo + len) -- the
        shard, or halo_range(shard, window) with the opt-in high-pass.  Vectors
        cover every local frame (halo ones are recomputed, not exchanged);
        summaries and corrected_out cover the shard's own blocks/frames."""
        from .stage import DeviceResult

        base = shard.frame_lo if local_lo is None else local_lo
        ref = self.template(frames_local, shard, ref_frames, base)
        self.pre.plan.set_reference(ref)
        self.pre.set_shading(ref)
        vec, sp, tp = self.pre.search_and_summarize(
            frames_local, corrected_out, t_global0=base, t_total=shard.n_total or shard.frame_hi,
            interior=(shard.frame_lo - base, shard.frames))
        return DeviceResult(vec, sp, tp, corrected_out, frames_local.shape[0])

    def close(self):
        self.pre.close()


# ------------------------------------------------------------------ frame-balanced shards
# block-aligned shards cap strong scaling at ceil(K/N)/(K/N)
# (C2 has K = 10 blocks; on 8 GPUs that is 62.5 %).  Frame-balanced shards give
# every rank T/N frames of motion search and warp/smoothing; a block that
# straddles a shard boundary is assembled at the rank holding its last frame:
# earlier contributors send their smoothed frames (the block's samples for the
# max - median selection, which does not decompose) and the block's float64
# running sum (the spatial mean, continued add by add so it stays bit-identical
# to one sequential pass) forward over NCCL point-to-point.  Whole blocks need
# no exchange.  The high-pass halo (A17) is part of the smoothed range.


def _range(n_frames: int, world: int, r: int) -> tuple[int, int]:
    return n_frames * r // world, n_frames * (r + 1) // world


def rank_of(n_frames: int, world: int, t: int) -> int:
    """The rank whose balanced shard holds recording frame t."""
    r = min(world - 1, (t * world) // max(n_frames, 1))
    while r > 0 and _range(n_frames, world, r)[0] > t:
        r -= 1
    while _range(n_frames, world, r)[1] <= t:
        r += 1
    return r


@dataclass(frozen=True)
class Piece:
    """This rank's share of a block that straddles a shard boundary."""
    block: int
    t0: int          # block frames [t0, t1)
    t1: int
    role: str        # "first" (sends), "middle" (receives, appends, sends), "last" (receives, owns)
    prev: int | None  # contributor before / after this rank
    next: int | None
    s_lo: int        # recording frames of the owner's assembled smoothed buffer [s_lo, s_hi)
    s_hi: int
    c_lo: int        # frames this rank smooths into it [c_lo, c_hi)
    c_hi: int
    m_lo: int        # this rank's own frames of the block [m_lo, m_hi): corrected + running sum
    m_hi: int


@dataclass(frozen=True)
class BalancedShard:
    rank: int
    world: int
    frame_lo: int
    frame_hi: int
    n_total: int
    segment_length: int
    local_lo: int    # frames the rank holds: the shard plus the high-pass halo
    local_hi: int
    whole_lo: int    # recording frames of the blocks lying wholly inside the shard (block aligned)
    whole_hi: int
    head: Piece | None  # straddling block holding frame_lo (role middle or last)
    tail: Piece | None  # straddling block holding frame_hi - 1 that this rank starts (role first)
    block_lo: int    # blocks whose summaries this rank outputs (those whose last frame it holds)
    block_hi: int

    @property
    def frames(self) -> int:
        return self.frame_hi - self.frame_lo


def balanced_plan(n_frames: int, segment_length: int, world: int, rank: int,
                  highpass_window: int = 0) -> BalancedShard:
    """Frame-balanced contiguous shard of rank `rank` and its straddling pieces."""
    L = segment_length
    if L < 2:
        raise ValueError("segment length must be >= 2")
    if n_frames % L == 1:  # summarize.py:79-80 on the final block
        raise ValueError("temporal summary needs at least 2 frames")
    hh = highpass_window // 2 if highpass_window and highpass_window > 1 else 0
    T = n_frames
    f0, f1 = _range(T, world, rank)
    loc_lo, loc_hi = max(0, f0 - hh), min(T, f1 + hh)

    def block(b):
        return b * L, min(T, (b + 1) * L)

    def piece(b):
        t0, t1 = block(b)
        starts, ends = t0 >= f0, t1 <= f1
        role = "first" if starts else ("last" if ends else "middle")
        prev = None if starts else rank_of(T, world, f0 - 1)
        nxt = None if ends else rank_of(T, world, f1)
        s_lo, s_hi = max(0, t0 - hh), min(T, t1 + hh)
        c_lo = s_lo if starts else f0
        c_hi = s_hi if ends else f1
        return Piece(b, t0, t1, role, prev, nxt, s_lo, s_hi, c_lo, c_hi, max(t0, f0), min(t1, f1))

    head = tail = None
    whole_lo = whole_hi = f0
    if f1 > f0:
        b_first, b_last = f0 // L, (f1 - 1) // L
        t0, t1 = block(b_first)
        if t0 < f0 or (t1 > f1):
            p = piece(b_first)
            if p.role == "first":
                tail = p
            else:
                head = p
        t0l, t1l = block(b_last)
        if b_last != b_first and t1l > f1:
            tail = piece(b_last)
        wb0 = b_first + (1 if (head is not None or tail is not None and tail.block == b_first) else 0)
        wb1 = b_last + (0 if (tail is not None and tail.block == b_last) or (head is not None and head.block == b_last)
                        else 1)
        if wb1 > wb0:
            whole_lo, whole_hi = block(wb0)[0], block(wb1 - 1)[1]
    # owned blocks: those whose last frame lies in [f0, f1)
    k = -(-T // L)
    own = [b for b in range(k) if f0 <= block(b)[1] - 1 < f1]
    b_lo, b_hi = (own[0], own[-1] + 1) if own else (0, 0)
    return BalancedShard(rank, world, f0, f1, T, L, loc_lo, loc_hi, whole_lo, whole_hi, head, tail, b_lo, b_hi)


class _P2P:
    """Forward point-to-point transfers of straddling-block buffers.  NCCL
    moves device tensors directly (one grouped launch per exchange); gloo (CPU
    tests, single-GPU multi-rank checks) stages them through host memory."""

    def __init__(self, group=None):
        self.group = group
        self.nccl = dist.get_backend(group) == "nccl"

    def start(self, sends, recvs):
        ops, post, keep = [], [], []
        for tensors, peer in sends:
            for t in tensors:
                x = t if (self.nccl or not t.is_cuda) else t.cpu()
                keep.append(x)
                ops.append(dist.P2POp(dist.isend, x, peer, self.group))
        for tensors, peer in recvs:
            for t in tensors:
                x = t if (self.nccl or not t.is_cuda) else torch.empty(t.shape, dtype=t.dtype)
                post.append((t, x))
                ops.append(dist.P2POp(dist.irecv, x, peer, self.group))
        works = dist.batch_isend_irecv(ops) if ops else []
        return works, post, keep

    @staticmethod
    def finish(handle):
        works, post, _keep = handle
        for w in works:
            w.wait()
        for t, x in post:
            if x is not t:
                t.copy_(x)


class DeviceOps:
    """The stage's CUDA entry points, as the balanced executor calls them."""

    def __init__(self, pre):
        self.pre = pre
        self.cfg = pre.cfg

    def template(self, frames, lo, hi, m, group):
        from . import _device as D
        from . import _lib

        h, w = frames.shape[1:]
        tsum = torch.zeros((h, w), dtype=torch.float64, device=frames.device)
        if hi > lo:
            _lib.call("vb_template_sum", frames[lo:hi].data_ptr(), D.vb_dtype(frames), hi - lo, h, w,
                      tsum.data_ptr(), 0, D.stream_handle())
        allreduce_sum_(tsum, group)
        ref = torch.empty((h, w), dtype=torch.float32, device=frames.device)
        _lib.call("vb_template_finish", tsum.data_ptr(), m, h * w, ref.data_ptr(), D.stream_handle())
        self.pre.plan.set_reference(ref)
        self.pre.set_shading(ref)

    def estimate(self, frames, arrival=None, chunk=0, after=None):
        """Motion vectors of every frame; with `arrival` the search runs in
        chunks of `chunk` frames, each after arrival(a, b) has made the stream
        wait for frames [a, b) (uploads still streaming in), and after(vec, b)
        is called once frames [0, b) are searched."""
        from . import _device as D

        n = frames.shape[0]
        vec = D.empty_motion(n, frames.device)
        if arrival is None or chunk <= 0:
            self.pre.plan.estimate(frames, self.cfg.subpixel, out=vec)
            return vec
        for a in range(0, n, chunk):
            b = min(n, a + chunk)
            arrival(a, b)
            self.pre.plan.estimate(frames[a:b], self.cfg.subpixel, out=self.vec_slice(vec, a, b))
            if after is not None:
                after(vec, b)
        return vec

    @staticmethod
    def vec_slice(vec, a, b):
        from . import _lib

        rec = _lib.MOTION_DTYPE.itemsize
        return vec[a * rec:b * rec]

    def frames_buffer(self, n, like):
        return torch.empty((n,) + tuple(like.shape[1:]), dtype=torch.float32, device=like.device)

    def sum_buffer(self, like):
        return torch.zeros(tuple(like.shape[1:]), dtype=torch.float64, device=like.device)

    def whole(self, frames, vec, t_global0, t_total, interior, corrected_out):
        from .summarize import summarize_device

        c = self.cfg
        return summarize_device(frames, c.segment_length, c.sigma, vectors_dev=vec, corrected_out=corrected_out,
                                highpass_window=self.pre.window, gain=self.pre.gain, t_global0=t_global0,
                                t_total=t_total, interior=interior)

    def piece(self, frames, vec, mean_off, mean_n, corrected_out, smoothed, partial):
        from . import _device as D
        from . import _lib

        n, h, w = frames.shape
        pre = self.pre
        _lib.call("vb_block_piece", frames.data_ptr(), D.vb_dtype(frames), D.ptr(vec), n, h, w,
                  pre.weights.ctypes.data, pre.wradius, D.ptr(pre.gain), mean_off, mean_n, D.ptr(corrected_out),
                  D.ptr(smoothed), D.ptr(partial), D.stream_handle())

    def finish(self, smoothed, s_lo, t0, count, t_total, partial):
        from . import _device as D
        from . import _lib

        n, h, w = smoothed.shape
        sp = torch.empty((1, h, w), dtype=torch.float32, device=smoothed.device)
        tp = torch.empty_like(sp)
        _lib.call("vb_block_finish", smoothed.data_ptr(), s_lo, n, t0, count, t_total, self.pre.window, h, w,
                  partial.data_ptr(), sp.data_ptr(), tp.data_ptr(), D.stream_handle())
        return sp, tp


@dataclass
class ShardResult:
    vectors: object          # vectors of every local frame (shard + halo)
    spatial: torch.Tensor    # [block_hi - block_lo, H, W]: the blocks this rank owns
    temporal: torch.Tensor
    corrected: torch.Tensor | None  # the shard's own frames
    n_frames: int

    def vectors_numpy(self):
        from . import _device as D

        return D.motion_to_numpy(self.vectors, self.n_frames)


class _CudaArray:
    """Zero-copy torch view of a raw device allocation (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _wrap(ptr: int, shape: tuple, dtype) -> torch.Tensor:
    typestr = {torch.float32: "<f4", torch.float64: "<f8"}[dtype]
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device="cuda")


class _Tokens:
    """Ordering messages between neighbour ranks for the peer-memory exchange:
    READY (the block data has been written into the owner's memory) and ACK
    (the owner has consumed its buffers; the sender may overwrite them next
    run).  NCCL tokens are stream-ordered; gloo tokens (CPU tests, ranks
    sharing one GPU) follow a stream synchronisation."""

    def __init__(self, group=None):
        self.group = group
        self.nccl = dist.get_backend(group) == "nccl"
        self._keep = []

    def send(self, peer: int) -> None:
        """Never waited on inside a run: an ACK is only received by the peer's
        next run, after the next collective (waiting here would deadlock it)."""
        if self.nccl:
            t = torch.ones(1, device="cuda")
        else:
            torch.cuda.current_stream().synchronize()
            t = torch.ones(1)
        self._keep = [(x, w) for x, w in self._keep if not w.is_completed()]
        self._keep.append((t, dist.isend(t, peer, self.group)))

    def recv(self, peer: int) -> None:
        t = torch.empty(1, device="cuda") if self.nccl else torch.empty(1)
        dist.irecv(t, peer, self.group).wait()

    def drain(self) -> None:
        for _t, w in self._keep:
            w.wait()
        self._keep.clear()


class _PeerBlocks:
    """IPC buffers of the straddling-block exchange: each rank
    that finishes or relays a block allocates its receive buffers with
    vb_ipc_alloc; the sender maps its next owner's buffers (vb_ipc_open) and
    its warp+smooth kernel and running sum write the block there directly
    (over NVLink on a multi-GPU node), tile by tile, instead of a separate
    send of the finished buffers."""

    def __init__(self, shard: BalancedShard, height: int, width: int, group=None):
        from . import _lib

        self.lib = _lib
        hw = height * width
        self.own = None    # (buf ptr, sum ptr) of this rank's head piece
        self.peer = None   # (buf ptr, sum ptr) mapped from the next owner
        self._alloc = []
        mine = {}
        if shard.head is not None:
            p = shard.head
            nbuf = (p.c_hi - p.s_lo) * hw * 4
            bptr, bh = self._ipc_alloc(nbuf)
            sptr, sh = self._ipc_alloc(hw * 8)
            self.own = (bptr, sptr)
            mine = {"buf": bh, "sum": sh}
        handles = [None] * shard.world
        dist.all_gather_object(handles, mine, group)
        nxt = shard.tail.next if shard.tail is not None else (
            shard.head.next if shard.head is not None and shard.head.role == "middle" else None)
        if nxt is not None:
            self.peer = (self._ipc_open(handles[nxt]["buf"]), self._ipc_open(handles[nxt]["sum"]))

    def _ipc_alloc(self, nbytes: int):
        import ctypes as C
        ptr = C.c_void_p()
        handle = (C.c_ubyte * 64)()
        self.lib.call("vb_ipc_alloc", nbytes, C.byref(ptr), handle)
        self._alloc.append(("free", ptr.value))
        return ptr.value, bytes(handle)

    def _ipc_open(self, handle: bytes) -> int:
        import ctypes as C
        ptr = C.c_void_p()
        buf = (C.c_ubyte * 64).from_buffer_copy(handle)
        self.lib.call("vb_ipc_open", buf, C.byref(ptr))
        self._alloc.append(("close", ptr.value))
        return ptr.value

    def close(self) -> None:
        lib = self.lib.load()
        for kind, ptr in reversed(self._alloc):
            (lib.vb_ipc_close if kind == "close" else lib.vb_ipc_free)(ptr)
        self._alloc.clear()


class BalancedShardedPreprocessor:
    """Per-rank driver over frame-balanced shards (balanced_plan):
    template all-reduce -> motion search of every local frame -> the tail
    piece is smoothed and sent forward while the whole blocks are summarised
    -> the head piece is received, completed and (if this rank holds the
    block's last frame) finished.  `ops` defaults to the CUDA entry points;
    the CPU tests pass an oracle-backed stand-in to check the protocol."""

    def __init__(self, height: int, width: int, config=None, group=None, ops=None, exchange: str = "peer"):
        """exchange: "peer" -- the sender's kernels write the straddling block
        straight into the owner's IPC-mapped buffers (device ops only); "p2p" --
        the finished buffers are sent with NCCL / gloo point-to-point."""
        if ops is None:
            from . import stage

            ops = DeviceOps(stage.DevicePreprocessor(height, width, config))
        if exchange not in ("peer", "p2p"):
            raise ValueError("exchange must be 'peer' or 'p2p'")
        self.ops = ops
        self.group = group
        self.height, self.width = height, width
        self.exchange = exchange if isinstance(ops, DeviceOps) else "p2p"
        self._peer = None
        self._peer_key = None
        self._tokens = None
        self._runs = 0
        self._tail_next = None
        self._whole = None

    def run(self, frames_local, shard: BalancedShard, ref_frames: int, corrected_out=None,
            arrival=None, chunk: int = 0) -> ShardResult:
        """frames_local = recording frames [shard.local_lo, shard.local_hi);
        corrected_out (optional) = [shard.frames, H, W] for the shard's own frames.
        arrival (optional, streamed uploads): arrival(a, b) makes the current
        stream wait until local frames [a, b) are resident; the template waits
        for its rows, the motion search runs in chunks of `chunk` frames as they
        land, and the summaries start once every frame is in."""
        ops, s = self.ops, shard
        base, T, f0 = s.local_lo, s.n_total, s.frame_lo
        n_local = s.local_hi - s.local_lo
        if frames_local.shape[0] != n_local:
            raise ValueError("frames_local must hold the shard and its halo")
        lo, hi = template_rows(Shard(s.rank, s.world, s.frame_lo, s.frame_hi, 0, 0, T), ref_frames, base)
        if arrival is not None and hi > lo:
            arrival(lo, hi)
        ops.template(frames_local, lo, hi, min(ref_frames, T), self.group)

        def corr(a, b):
            return None if corrected_out is None else corrected_out[a - f0:b - f0]

        self._whole = None
        if arrival is not None and chunk > 0:
            # whole blocks are summarised as soon as their frames are searched,
            # while later pieces are still uploading
            wl, wh, L = s.whole_lo - base, s.whole_hi - base, ops.cfg.segment_length
            # the temporal high-pass (A17) reads window // 2 frames past a block's end
            halo = max(0, int(getattr(getattr(ops, "pre", None), "window", 0) or 0)) // 2
            parts, done = [], [wl]

            def after(vec, b):
                while done[0] < wh and (min(done[0] + L, wh) + halo <= b or b == n_local):
                    e = min(done[0] + L, wh)
                    parts.append(ops.whole(frames_local, vec, base, T, (done[0], e - done[0]),
                                           corr(done[0] + base, e + base)))
                    done[0] = e

            vec = ops.estimate(frames_local, arrival, chunk, after)
            arrival(0, n_local)
            if parts:
                self._whole = (torch.cat([p[0] for p in parts]), torch.cat([p[1] for p in parts]))
        else:
            if arrival is not None:
                arrival(0, n_local)
            vec = ops.estimate(frames_local)

        def run_piece(p: Piece, smoothed, acc):
            ops.piece(frames_local[p.c_lo - base:p.c_hi - base], ops.vec_slice(vec, p.c_lo - base, p.c_hi - base),
                      p.m_lo - p.c_lo, p.m_hi - p.m_lo, corr(p.m_lo, p.m_hi), smoothed, acc)

        if s.world > 1 and self.exchange == "peer":
            return self._run_peer(frames_local, s, vec, corr, run_piece, corrected_out)
        p2p = _P2P(self.group) if s.world > 1 else None
        sends, recvs = [], []
        if s.tail is not None:  # this rank starts a block that a later rank finishes
            tb = ops.frames_buffer(s.tail.c_hi - s.tail.c_lo, frames_local)
            ts = ops.sum_buffer(frames_local)
            run_piece(s.tail, tb, ts)
            sends.append(([tb, ts], s.tail.next))
        head_buf = head_sum = None
        if s.head is not None:
            p = s.head
            head_buf = ops.frames_buffer(p.c_hi - p.s_lo, frames_local)
            head_sum = ops.sum_buffer(frames_local)
            recvs.append(([head_buf[:p.c_lo - p.s_lo], head_sum], p.prev))
        handle = p2p.start(sends, recvs) if (sends or recvs) else None
        sp_parts, tp_parts = [], []
        whole = self._whole  # already summarised while the upload streamed (run(arrival=...))
        if whole is None and s.whole_hi > s.whole_lo:
            whole = ops.whole(frames_local, vec, base, T, (s.whole_lo - base, s.whole_hi - s.whole_lo),
                              corr(s.whole_lo, s.whole_hi))
        if handle is not None:
            p2p.finish(handle)
        if s.head is not None:
            p = s.head
            # continue the received running sum with this rank's frames, append its smoothed frames
            run_piece(p, head_buf[p.c_lo - p.s_lo:], head_sum)
            if p.role == "middle":
                p2p.finish(p2p.start([([head_buf, head_sum], p.next)], []))
            else:
                sp_h, tp_h = ops.finish(head_buf, p.s_lo, p.t0, p.t1 - p.t0, T, head_sum)
                sp_parts.append(sp_h)
                tp_parts.append(tp_h)
        if whole is not None:
            sp_parts.append(whole[0])
            tp_parts.append(whole[1])
        if sp_parts:
            sp, tp = torch.cat(sp_parts), torch.cat(tp_parts)
        else:
            sp = torch.empty((0, self.height, self.width), dtype=torch.float32, device=frames_local.device)
            tp = sp.clone()
        assert sp.shape[0] == s.block_hi - s.block_lo
        return ShardResult(vec, sp, tp, corrected_out, frames_local.shape[0])

    def _run_peer(self, frames_local, s: BalancedShard, vec, corr, run_piece, corrected_out) -> ShardResult:
        """The straddling-block exchange through peer memory (see _PeerBlocks)."""
        ops, base, T = self.ops, s.local_lo, s.n_total
        h, w = self.height, self.width
        key = (s.rank, s.world, s.frame_lo, s.frame_hi, s.local_lo, s.local_hi, s.n_total)
        if self._peer_key != key:  # collective: every rank (re)maps together
            if self._peer is not None:
                self._peer.close()
            self._peer = _PeerBlocks(s, h, w, self.group)
            self._peer_key = key
            self._tokens = _Tokens(self.group)
            self._runs = 0
        pb, tk = self._peer, self._tokens
        first = self._runs == 0
        self._tail_next = s.tail.next if s.tail is not None else (
            s.head.next if s.head is not None and s.head.role == "middle" else None)
        if s.tail is not None:  # write this rank's piece into the next owner's buffers
            p = s.tail
            if not first:
                tk.recv(p.next)  # ACK: the owner is done with last run's data
            from . import _device as D
            from . import _lib
            _lib.call("vb_memset_async", pb.peer[1], 0, h * w * 8, D.stream_handle())  # the sum starts at 0
            run_piece(p, pb.peer[0], pb.peer[1])  # raw peer addresses: the kernels write the owner's memory
            tk.send(p.next)  # READY
        whole = self._whole  # already summarised while the upload streamed (run(arrival=...))
        if whole is None and s.whole_hi > s.whole_lo:
            whole = ops.whole(frames_local, vec, base, T, (s.whole_lo - base, s.whole_hi - s.whole_lo),
                              corr(s.whole_lo, s.whole_hi))
        sp_parts, tp_parts = [], []
        if s.head is not None:
            p = s.head
            n_buf = p.c_hi - p.s_lo
            head_buf = _wrap(pb.own[0], (n_buf, h, w), torch.float32)
            head_sum = _wrap(pb.own[1], (h, w), torch.float64)
            tk.recv(p.prev)  # READY: the earlier contributors' frames and running sum are in place
            if p.role == "middle":  # relay: prefix and sum to the next owner, own piece written there directly
                if not first:
                    tk.recv(p.next)
                nb, ns = pb.peer
                from . import _device as D
                from . import _lib
                npre = p.c_lo - p.s_lo
                _lib.call("vb_copy_async", nb, head_buf.data_ptr(), npre * h * w * 4, D.stream_handle())
                _lib.call("vb_copy_async", ns, head_sum.data_ptr(), h * w * 8, D.stream_handle())
                run_piece(p, nb + npre * h * w * 4, ns)
                tk.send(p.next)
            else:
                run_piece(p, head_buf[p.c_lo - p.s_lo:], head_sum)
                sp_h, tp_h = ops.finish(head_buf, p.s_lo, p.t0, p.t1 - p.t0, T, head_sum)
                sp_parts.append(sp_h)
                tp_parts.append(tp_h)
            tk.send(p.prev)  # ACK for the next run (stream-ordered after the reads above)
        if whole is not None:
            sp_parts.append(whole[0])
            tp_parts.append(whole[1])
        if sp_parts:
            sp, tp = torch.cat(sp_parts), torch.cat(tp_parts)
        else:
            sp = torch.empty((0, h, w), dtype=torch.float32, device=frames_local.device)
            tp = sp.clone()
        self._runs += 1
        assert sp.shape[0] == s.block_hi - s.block_lo
        return ShardResult(vec, sp, tp, corrected_out, frames_local.shape[0])

    def close(self):
        """Collective with the neighbours: outstanding ACKs are matched first."""
        if self._peer is not None:
            torch.cuda.synchronize()
            s_tail = self._peer_key is not None and self._runs > 0
            if s_tail and self._tail_next is not None:
                self._tokens.recv(self._tail_next)  # the last run's ACK
            self._tokens.drain()
            self._peer.close()
            self._peer = None
        close = getattr(getattr(self.ops, "pre", None), "close", None)
        if close is not None:
            close()
