"""Multi-GPU plumbing (one process per GPU, torch.distributed).

Every (b,h) slice is an independent problem, so the data
path needs no collective.  The one exchange is the gradient of the shared
Cauchy scale eps (one scalar per layer, reading D20): each rank
contributes one f64, the ranks all-gather them and every rank sums them in
rank order -- the same bits on every rank, run to run (no reduction-order
ambiguity of an all-reduce).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def partition(total: int, world: int, rank: int) -> range:
    """Contiguous, balanced split of `total` (b,h) slices: rank r gets range(lo, hi)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return range(lo, hi)


def weak_slices(bh_per_rank: int, rank: int) -> range:
    """Global slice ids of rank `rank` when every rank runs its own batch (weak scaling)."""
    return range(rank * bh_per_rank, (rank + 1) * bh_per_rank)


def combine_d_eps(d_eps: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather one f64 per rank and sum in rank order (deterministic). In place; returns d_eps."""
    if not dist.is_available() or not dist.is_initialized():
        return d_eps
    world = dist.get_world_size(group)
    if world == 1:
        return d_eps
    parts = [torch.empty_like(d_eps) for _ in range(world)]
    dist.all_gather(parts, d_eps.contiguous(), group=group)
    total = parts[0].clone()
    for p in parts[1:]:
        total += p
    d_eps.copy_(total)
    return d_eps
