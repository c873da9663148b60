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


STREAM_STRIDE = 97  # coprime with 300: consecutive global steps walk the whole kick stream


def stream_frame(global_step: int, n_frames: int, stride: int = STREAM_STRIDE) -> int:
    """Frame of the capture stream processed at `global_step` (0, 1, 2, ... over
    all ranks): frame = stride * global_step mod n_frames.  With the stride
    coprime to n_frames, any n_frames consecutive global steps visit every
    frame once, so a short run samples every pose instead of the first few."""
    return (stride * global_step) % n_frames


def rank_frames(rank: int, world: int, steps: int, n_frames: int, stride: int = STREAM_STRIDE) -> list[int]:
    """Frames of `rank` for `steps` steps: global steps rank, rank+world, ...
    (the stream's frames interleaved over ranks, as shard_frames, then
    permuted by the stride)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return [stream_frame(i * world + rank, n_frames, stride) for i in range(steps)]


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
