"""Batch-index sharding of independent KKT systems across GPUs.

Independent systems have no exchange step, so the multi-GPU path is pure
partitioning: rank g of G owns a contiguous range of global batch indices,
and system i is always generated from seed0 + i, so results do not depend on
G. The only collectives are outside the data path (barriers and a max-reduce
of the timed region).
"""
from __future__ import annotations


def shard_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [first, last) slice of `batch` systems for `rank` of `world`
    (the same split b2p_solve_batched_multi uses: ceil(batch / world) per rank)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    per = (batch + world - 1) // world
    first = min(batch, rank * per)
    return first, min(batch, first + per)


def weak_shard(per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank owns `per_rank` systems of its own."""
    return rank * per_rank, (rank + 1) * per_rank


def seeds(seed0: int, first: int, last: int) -> list[int]:
    """Seeds of the systems in [first, last) (bench-pcg rule seed0 + i)."""
    return [seed0 + i for i in range(first, last)]


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Timed-region length as the max over ranks (torch.distributed all_reduce MAX)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
