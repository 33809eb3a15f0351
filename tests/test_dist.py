"""Multi-process (gloo, world_size 2, CPU) checks of the batch-sharded path's host logic:
shard bounds and the fixed-rank-order reduction of the shared gradients."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_18780_b200.dist import reduce_shared_grads, shard_bounds


def test_shard_bounds_cover_the_batch():
    for B in (1, 7, 8, 64):
        for W in (1, 2, 3, 8):
            spans = [shard_bounds(B, r, W) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    gT = torch.from_numpy(rng.standard_normal((5, 5)))
    gB = torch.from_numpy(rng.standard_normal((7, 5)))
    rT, rB = reduce_shared_grads(gT, gB)
    out[rank] = (rT.numpy().copy(), rB.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_fixed_order_reduction_world2():
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    parts = []
    for r in range(world):
        rng = np.random.default_rng(100 + r)
        parts.append((rng.standard_normal((5, 5)), rng.standard_normal((7, 5))))
    wantT = parts[0][0] + parts[1][0]
    wantB = parts[0][1] + parts[1][1]
    for r in range(world):
        # bit-identical on every rank and equal to the rank-ordered sum
        assert np.array_equal(res[r][0], wantT)
        assert np.array_equal(res[r][1], wantB)


def test_single_process_is_identity():
    gT, gB = torch.ones(2, 2), torch.zeros(3, 2)
    rT, rB = reduce_shared_grads(gT, gB)
    assert rT is gT and rB is gB


def _worker_exact(rank, world, port, out):
    """Uneven shards of a batch of 5 sequences: gathered per-sequence partials reduced in batch
    order equal the single-process fixed-order reduction bit for bit, on every rank."""
    from paper_2604_18780_b200.dist import reduce_shared_grads_exact

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    allT, allB = rng.standard_normal((5, 4, 4)), rng.standard_normal((5, 9, 4))
    up = torch.from_numpy(rng.uniform(-1.0, 2.0, 5))
    lo, hi = shard_bounds(5, rank, world)
    rT, rB = reduce_shared_grads_exact(torch.from_numpy(allT[lo:hi]), torch.from_numpy(allB[lo:hi]), 5, up)
    out[rank] = (rT.numpy().copy(), rB.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_reduction_bit_identical_to_single_process(world):
    from paper_2604_18780_b200.dist import fixed_order_sum

    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker_exact, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    rng = np.random.default_rng(7)
    allT, allB = rng.standard_normal((5, 4, 4)), rng.standard_normal((5, 9, 4))
    up = torch.from_numpy(rng.uniform(-1.0, 2.0, 5))
    wantT = fixed_order_sum(torch.from_numpy(allT), up).numpy()
    wantB = fixed_order_sum(torch.from_numpy(allB), up).numpy()
    seqT = np.zeros((4, 4))
    for b in range(5):
        seqT = seqT + up.numpy()[b] * allT[b]
    assert np.array_equal(wantT, seqT)
    for r in range(world):
        assert np.array_equal(res[r][0], wantT)
        assert np.array_equal(res[r][1], wantB)
