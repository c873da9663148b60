# SPDX-License-Identifier: Apache-2.0
"""Frame-parallel sharding of a capture stream over ranks.

`recon::reconstruct_frame` is a pure function of one frame's views
(the CLI's GoF loop, volcap.cpp:304-320, carries no state), so a
stream shards over GPUs with no data-path collective: rank r takes frames
r, r+N, r+2N, ...  The only cross-rank traffic is the timing reduction
(max over ranks) and optional result gathering on the host.
"""
from __future__ import annotations


def shard_frames(n_frames: int, rank: int, world: int) -> list[int]:
    """Round-robin frame indices of `rank` (disjoint, covering 0..n_frames-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_frames, world))


def max_over_ranks(value: float, device=None) -> float:
    """MAX all-reduce of one scalar (the benchmark's timing rule); identity when
    torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
