"""Multi-GPU host plumbing (torch.distributed): one process per GPU.

The update path has no data exchange in replica mode: every rank owns an
independent map and frame stream on its own device; collectives only carry the barrier and the
max-over-ranks reduction of device timings. `shard_bounds` is the scan-order-preserving batch
split the exact point-batch sharding of one frame uses: rank g takes the
contiguous batch [g*N/G, (g+1)*N/G), so the global point index stays the ray id used for k*.
"""
from __future__ import annotations

import os
from typing import Tuple


def rank_env() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, scan-order-preserving batch of n points for `rank` of `world`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return (n * rank) // world, (n * (rank + 1)) // world


def _device_for(dist):
    import torch
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(value: float, dist=None) -> float:
    """Max of a per-rank scalar (the timing reduction of bench.py); identity without dist."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def weak_scaling_value(points_per_rank_per_step: int, steps: int, world: int, max_seconds: float) -> float:
    """Whole-job points/s: every rank integrates its own frames; time = slowest rank."""
    return world * points_per_rank_per_step * steps / max_seconds
