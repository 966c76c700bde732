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
