"""Env-index sharding across GPUs (one process per GPU).

Envs are independent and each env's trajectory depends only on its own seed
(reference tests/test_engine.py:215-223, partition independence), so GPU g
of N plays global env indices [g*B, (g+1)*B) with seeds spawn(seed, index):
the union of the shards is bit-identical to one run of N*B envs.  The hot
path has no collective; ``reduce_stats`` is the single all-reduce of the
rollout statistics at the end.
"""

from __future__ import annotations

import os

STATS = ("env_steps", "p1_wins", "p2_wins", "draws", "truncated", "envs")


def world():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(rank, world_size, batch_per_rank):
    """Global env indices owned by ``rank`` (weak scaling: fixed per-rank batch)."""
    first = rank * batch_per_rank
    return first, first + batch_per_rank


def split_even(total, world_size, rank):
    """Strong-scaling split of ``total`` envs: contiguous, sizes differ by <= 1."""
    base, extra = divmod(total, world_size)
    first = rank * base + min(rank, extra)
    return first, first + base + (1 if rank < extra else 0)


def reduce_stats(stats, group=None):
    """Sum a stats tensor over ranks in place (NCCL on GPU, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def max_over_ranks(value, group=None):
    """Max of a scalar tensor over ranks (timing: the slowest rank defines the run)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(value, op=dist.ReduceOp.MAX, group=group)
    return value
