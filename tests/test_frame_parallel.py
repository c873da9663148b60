# SPDX-License-Identifier: Apache-2.0
"""Host logic of the frame-parallel multi-GPU mode, run with world_size 2 on
the gloo backend (CPU): disjoint round-robin shards covering the stream, and
the max-over-ranks / sum-over-ranks reductions the benchmark uses."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1712_03084_b200.frame_parallel import max_over_ranks, shard_frames, sum_over_ranks


def test_shards_cover_disjoint():
    for n, w in [(300, 1), (300, 2), (300, 8), (7, 4), (4096, 8), (3, 8)]:
        shards = [shard_frames(n, r, w) for r in range(w)]
        flat = sorted(f for s in shards for f in s)
        assert flat == list(range(n))
        assert max(len(s) for s in shards) - min(len(s) for s in shards) <= 1
    with pytest.raises(ValueError):
        shard_frames(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    frames = shard_frames(300, rank, world)
    # per-rank "elapsed ms" stands in for the CUDA-event time of the shard
    ms = 10.0 + 5.0 * rank
    out[rank] = (max_over_ranks(ms), sum_over_ranks(len(frames)), frames[:3])
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == 15.0  # max over ranks
    assert out[0][1] == out[1][1] == 300   # every frame processed exactly once
    assert out[0][2] == [0, 2, 4] and out[1][2] == [1, 3, 5]
