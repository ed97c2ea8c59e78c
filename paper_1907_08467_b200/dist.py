"""Multi-GPU plumbing: env sharding and the one collective.

Environments are independent, so the path shards trivially: rank r of G owns the contiguous
global env ids [r*E, (r+1)*E) (env_index_base = r*E); every env's trajectory is keyed by its
global id, so results do not depend on G.  The only cross-GPU exchange is an all_reduce(SUM)
of the int64[4] counters {frames, episodes finished, episode-return sum, faults} per reporting
window, plus MAX of the per-rank elapsed time for the benchmark (PAPER.md P:112 gives no
mechanism for multi-GPU; BASELINE.json cfg5).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(envs_per_rank: int, rank: int) -> tuple[int, int]:
    """(env_index_base, count) of a rank under weak scaling."""
    return rank * envs_per_rank, envs_per_rank


def shard_total(total_envs: int, rank: int, world: int) -> tuple[int, int]:
    """(env_index_base, count) when a fixed total is split as evenly as possible."""
    base, rem = divmod(total_envs, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def reduce_counters(counters: torch.Tensor, group=None) -> torch.Tensor:
    """all_reduce(SUM) of the int64[4] counters; returns a new tensor (input untouched)."""
    out = counters.clone()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def max_over_ranks(value: float, device=None, group=None) -> float:
    """MAX of a per-rank scalar (device time of the timed region)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
