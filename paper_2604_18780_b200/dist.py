"""Batch-sharded multi-GPU semi-CRF: the path's only collective.

Sequences are independent, so each rank owns a slice of the batch and runs the
whole posterior on its GPU. The shared-parameter gradients grad_T (C, C) and
grad_B (K, C) are the only values that cross GPUs: every rank all-gathers the
per-rank fp64 partials and sums them in fixed rank order, so the result is
bit-identical on every rank and for any launch order (the reference reduces
segment-major then batch-major in a fixed order, streaming.py:389-395).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of the batch owned by `rank`."""
    base, rem = divmod(batch, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def reduce_shared_grads(grad_T: torch.Tensor, grad_B: torch.Tensor, group=None):
    """Fixed-rank-order sum of grad_T / grad_B over the process group.

    all_gather of the flat fp64 partials (C*C + K*C values: 197 KB at c4), then a
    sequential sum in rank order on every rank. Returns new (grad_T, grad_B).
    """
    if not dist.is_available() or not dist.is_initialized():
        return grad_T, grad_B
    world = dist.get_world_size(group)
    if world == 1:
        return grad_T, grad_B
    flat = torch.cat([grad_T.reshape(-1), grad_B.reshape(-1)]).to(torch.float64).contiguous()
    parts = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(parts, flat, group=group)
    tot = parts[0].clone()
    for p in parts[1:]:
        tot += p
    nT = grad_T.numel()
    return tot[:nT].view_as(grad_T), tot[nT:].view_as(grad_B)
