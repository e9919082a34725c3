"""Multi-GPU plumbing for the evaluation.

Replays are independent, so ranks shard the work with no data-path
collective: rank r of W replays trace seeds ``r*S .. r*S+S-1`` (weak scaling).
The one exchange is the global argmax over every rank's seeds: an all-reduce
(SUM) of the per-(candidate, QPS) met counts — int64, exact, so the result is
independent of rank count and reduction order — then the argmax kernel
(``Context.argmax_device``) on each rank.  Goodput sums are gathered and added
in rank order so they are deterministic too.  Works with NCCL (CUDA tensors)
and gloo (CPU tensors, used by the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def rank_seeds(rank: int, seeds_per_rank: int, base: int = 0) -> list[int]:
    """Seed block of one rank (weak scaling: every rank owns S distinct seeds)."""
    return [base + rank * seeds_per_rank + j for j in range(seeds_per_rank)]


def allreduce_met(met: torch.Tensor, group=None) -> torch.Tensor:
    """Σ over ranks of int64 met counts, in place (exact)."""
    if met.dtype != torch.int64:
        raise TypeError("met counts must be int64")
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(met, op=dist.ReduceOp.SUM, group=group)
    return met


def sum_goodput_rank_order(good: torch.Tensor, group=None) -> torch.Tensor:
    """Σ over ranks of FP64 goodput, added in ascending rank order."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return good.clone()
    parts = [torch.empty_like(good) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, good.contiguous(), group=group)
    out = parts[0].clone()
    for p in parts[1:]:
        out += p
    return out


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a host scalar over ranks (timing: the slowest rank defines the step)."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
