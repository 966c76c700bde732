"""N>1 path on CPU: two gloo ranks run the sharding plan and the template
all-reduce of distributed.py and must reproduce the single-process template
bit-exactly (integer camera samples); gather_outputs reassembles shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_16438_b200 import distributed, synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, raw, L, m, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = raw.shape[0]
        shard = distributed.shard_plan(t, L, world, rank)
        local = raw[shard.frame_lo:shard.frame_hi]
        lo, hi = distributed.template_rows(shard, m)
        # float64 per-pixel partial sum of this rank's template frames (what
        # vb_template_sum computes on the device), in frame order
        part = np.zeros(raw.shape[1:], np.float64)
        for f in local[lo:hi]:
            part += f.astype(np.float64)
        tsum = torch.from_numpy(part)
        distributed.allreduce_sum_(tsum)
        ref = (tsum.numpy() / min(m, t)).astype(np.float32)
        np.save(os.path.join(out_dir, f"ref{rank}.npy"), ref)
        # each rank owns its blocks' outputs; gather them back in rank order
        blocks = torch.arange(shard.block_lo, shard.block_hi, dtype=torch.int64)
        got = torch.cat(distributed.gather_outputs(blocks))
        np.save(os.path.join(out_dir, f"blocks{rank}.npy"), got.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("t,L,m", [(150, 50, 100), (120, 40, 30), (90, 30, 100)])
def test_template_allreduce_matches_single_process(tmp_path, oracle_mod, t, L, m):
    raw = synth.generate_numpy(synth.CONFIGS["c1"].with_frames(t))
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), raw, L, m, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    want = oracle_mod.make_reference(raw.astype(np.float32), m)
    k = -(-t // L)
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"ref{r}.npy"), want)
        np.testing.assert_array_equal(np.load(tmp_path / f"blocks{r}.npy"), np.arange(k))
