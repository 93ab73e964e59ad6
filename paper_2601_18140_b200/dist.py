"""Multi-GPU plumbing for lane sharding: one process per
GPU, every rank owns a contiguous range of *global* lanes, no data-path
collective.  Stimulus and hashes are functions of global lane ids, so results
do not depend on the GPU count.  torch.distributed carries only the timing
reduction (max over ranks) and the optional gather of per-lane results.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional, Tuple


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    lane0: int      # first global lane of this rank
    n_lanes: int    # lanes of this rank


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1-process defaults)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_weak(rank: int, world: int, lanes_per_rank: int) -> Shard:
    """Weak scaling: every rank simulates `lanes_per_rank` lanes of its own."""
    return Shard(rank, world, rank * lanes_per_rank, lanes_per_rank)


def shard_strong(rank: int, world: int, total_lanes: int) -> Shard:
    """Strong scaling: `total_lanes` split into contiguous, near-equal ranges
    ([d*L/D, (d+1)*L/D))."""
    b = rank * total_lanes // world
    e = (rank + 1) * total_lanes // world
    return Shard(rank, world, b, e - b)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device timing) over all ranks."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_lanes(local, dist=None, device=None):
    """Concatenate per-rank [n_cycles, n_lanes_rank] u64 results along lanes on
    every rank (all_gather of equal-size shards; verification only)."""
    import numpy as np
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    t = torch.from_numpy(np.ascontiguousarray(local).view(np.int64)).to(device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return np.concatenate([p.cpu().numpy().view(np.uint64) for p in parts], axis=1)
