"""Batch-sharded multi-GPU semi-CRF: the path's only collective.

Sequences are independent, so each rank owns a contiguous slice of the
batch and runs the whole posterior for it on its GPU; logZ, grad_S, grad_P and the marginals
of a sequence never leave its rank. The shared-parameter gradients grad_T (C, C) and grad_B
(K, C) are the only values that cross GPUs. Every rank all-gathers the PER-SEQUENCE fp64
partials (scrf_backward_partials: upstream-unscaled, accumulated in an order that depends only
on the sequence, never on the batch size) in global batch order and runs the library's own
fixed-order batch reduction (scrf_reduce_partials, the same kernel and order the single-GPU
posterior finishes with), so grad_T / grad_B are bit-identical on every rank AND for 1, 2, 4
or 8 GPUs (the reference reduces segment-major then batch-major in a fixed order,
streaming.py:389-395).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of the batch owned by `rank`."""
    base, rem = divmod(batch, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_batch_rows(local: torch.Tensor, batch: int, group=None) -> torch.Tensor:
    """All-gather per-sequence rows (B_local, ...) of every rank into (batch, ...) in global
    batch order (shards are contiguous and ordered by rank; uneven shards are padded)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    spans = [shard_bounds(batch, r, world) for r in range(world)]
    width = max(h - lo for lo, h in spans)
    pad = local.new_zeros((width,) + tuple(local.shape[1:]))
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    return torch.cat([p[: h - lo] for p, (lo, h) in zip(parts, spans)], dim=0)


def fixed_order_sum(parts: torch.Tensor, upstream: torch.Tensor | None = None) -> torch.Tensor:
    """sum_b upstream[b] * parts[b] in batch order, one rounding per multiply and add.

    CUDA tensors: the library's scrf_reduce_partials (the reduction the single-GPU posterior
    ends with). CPU tensors (the gloo host-logic tests): the same operation order in numpy.
    """
    B = parts.shape[0]
    flat = parts.reshape(B, -1).to(torch.float64).contiguous()
    if flat.is_cuda:
        from . import _lib

        lib = _lib.load()
        out = torch.empty(flat.shape[1], dtype=torch.float64, device=flat.device)
        up = None if upstream is None else upstream.to(device=flat.device, dtype=torch.float64).contiguous()
        _lib.check(lib.scrf_reduce_partials(B, flat.shape[1], _lib.ptr(flat), _lib.ptr(up), _lib.ptr(out),
                                            _lib.stream_handle()), "scrf_reduce_partials")
        return out.view(parts.shape[1:])
    p = flat.numpy()
    u = np.ones(B) if upstream is None else upstream.to(torch.float64).numpy()
    tot = np.zeros(p.shape[1])
    for b in range(B):
        tot = tot + u[b] * p[b]  # numpy: separate multiply and add, as the kernel's __dmul_rn / __dadd_rn
    return torch.from_numpy(tot).view(parts.shape[1:])


def reduce_shared_grads_exact(gT_part: torch.Tensor, gB_part: torch.Tensor, batch: int,
                              upstream: torch.Tensor | None = None, group=None):
    """Global grad_T / grad_B from this rank's per-sequence partials (B_local, C, C) and
    (B_local, K, C): all-gather in batch order, fixed-order reduction with the global upstream."""
    allT = gather_batch_rows(gT_part, batch, group)
    allB = gather_batch_rows(gB_part, batch, group)
    return fixed_order_sum(allT, upstream), fixed_order_sum(allB, upstream)


def sharded_posterior(cum, params, delta=None, upstream=None, *, group=None, memory: str = "auto"):
    """posterior() of this rank's shard of the batch (one process per GPU, torch.distributed).

    Returns ((lo, hi), logZ, GradientSet, MarginalSet): per-sequence arrays for sequences
    lo..hi-1 only; grad_T / grad_B for the WHOLE batch, identical on every rank and to the
    single-GPU result bit for bit."""
    from dataclasses import replace

    from . import streaming as S
    from .diagnostics import GradientSet, MarginalSet

    B = cum.batch_size
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = shard_bounds(B, rank, world)
    sl = slice(lo, hi)
    local = replace(cum, S=cum.S[sl], lengths=np.asarray(cum.lengths)[sl],
                    proj_start=None if cum.proj_start is None else cum.proj_start[sl],
                    proj_end=None if cum.proj_end is None else cum.proj_end[sl])
    prob = S.DeviceProblem.from_host(local, params)
    up = None if upstream is None else torch.as_tensor(np.asarray(upstream, dtype=np.float64), device=prob.S.device)
    # per-position gradients carry this shard's upstream; the partials are upstream-unscaled
    fwd, bw = S.device_posterior(prob, delta, None if up is None else up[sl],
                                 memory=S.choose_memory_mode(prob, delta, memory))
    gT, gB = S.device_grad_partials(prob, fwd, bw)
    rT, rB = reduce_shared_grads_exact(gT, gB, B, up, group)
    S._raise_if_dead(fwd)
    host = lambda t: None if t is None else t.cpu().numpy()  # noqa: E731
    grads = GradientSet(grad_S=host(bw.grad_S), grad_T=host(rT), grad_B=host(rB), grad_P_start=host(bw.grad_P_start),
                        grad_P_end=host(bw.grad_P_end))
    marg = MarginalSet(host(bw.position_marginals), host(bw.boundary_posterior), host(bw.expected_segment_count),
                       np.asarray(local.lengths))
    return (lo, hi), host(fwd.logZ), grads, marg


def reduce_shared_grads(grad_T: torch.Tensor, grad_B: torch.Tensor, group=None):
    """Rank-order sum of already batch-reduced grad_T / grad_B (weak-scaling jobs where each rank
    owns a separate batch). Bit-identical on every rank; for one batch split across ranks use
    reduce_shared_grads_exact, which also matches the single-GPU result bit for bit."""
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
