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


def test_stream_order_visits_every_pose():
    from paper_1712_03084_b200.frame_parallel import rank_frames, stream_frame
    assert sorted(stream_frame(g, 300) for g in range(300)) == list(range(300))
    assert sorted(stream_frame(g, 60) for g in range(60)) == list(range(60))
    for world in (1, 2, 4, 8):
        steps = 300 // world if 300 % world == 0 else 300 // world + 1
        got = [f for r in range(world) for f in rank_frames(r, world, steps, 300)]
        assert set(got) == set(range(300))
    # the first 20 global steps already span the stream (not the flat first poses)
    assert max(stream_frame(g, 300) for g in range(20)) - min(stream_frame(g, 300) for g in range(20)) > 250


def test_bench_launcher_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks
    (torch.distributed.run, gloo here); the ranks' frame plans are disjoint
    and together cover the stream once."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--plan", "--gpus", "2", "--steps", "150"],
                         capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and len(d["frames_by_rank"]) == 2
    a, b = d["frames_by_rank"]
    assert not set(a) & set(b) and sorted(a + b) == list(range(300))


def test_bench_launcher_c4_shards_the_4096_stream():
    """C4: `bench.py --workload c4 --gpus 2` gives each rank its
    whole shard of the 4096-frame kick stream (steps = shard size, --steps
    ignored); the shards are disjoint and cover make_kick_sequence(4096)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--plan", "--workload", "c4", "--gpus", "2",
                          "--steps", "10"], capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    a, b = d["frames_by_rank"]
    assert len(a) == len(b) == 2048
    assert not set(a) & set(b) and sorted(a + b) == list(range(4096))
