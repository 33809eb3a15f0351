"""Sublinear-memory mode (north-star subsystem 3): real checkpoint rows,
`recompute_alpha` on the device, and the checkpoint-replay backward.

Reference: CheckpointSet (streaming.py:49-67), recompute_alpha (:232-261), the per-segment
replay inside streaming_backward (:332-336); tests mirror TestRecomputeAlpha
(pkg/tests/test_streaming.py:167-226) against the fp64 golden fixtures of the real reference.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import golden_io  # noqa: E402
import parity  # noqa: E402
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.potentials import CenteringMode  # noqa: E402


@pytest.fixture(params=["fp32", "fp64"])
def precision(request):
    S.set_precision(request.param)
    yield request.param
    S.set_precision("fp32")


def _host(fwd, bw):
    out = {k: getattr(bw, k).cpu().numpy() for k in ("grad_S", "grad_T", "grad_B", "position_marginals",
                                                      "boundary_posterior", "expected_segment_count")}
    out["logZ"] = fwd.logZ.cpu().numpy()
    out["N"] = fwd.N.cpu().numpy()
    return out


SHAPES = [
    # seed, T, K, C, B, ragged, projections, delta
    (0, 300, 8, 4, 3, True, True, None),
    (1, 700, 20, 6, 2, True, False, 37),     # delta < K + 32: windows of several checkpoint periods
    (2, 1200, 64, 5, 4, True, True, None),   # several windows, ragged lengths across them
    (3, 2000, 100, 24, 2, False, False, 150),
    (4, 600, 3, 3, 5, True, False, 1),       # delta = 1: every position is a checkpoint
]


@pytest.mark.parametrize("shape", SHAPES)
def test_sublinear_posterior_matches_full_mode(shape, precision):
    seed, T, K, C, B, ragged, proj, delta = shape
    _, params, cum = scrf.equivalence_instance(seed, T=T, K=K, C=C, B=B, mode=CenteringMode.MEAN, ragged=ragged,
                                               projections=proj)
    prob = scrf.DeviceProblem.from_host(cum, params)
    full = _host(*S.device_posterior(prob, delta, memory="full"))
    sub = _host(*S.device_posterior(prob, delta, memory="sublinear"))
    # identical sweeps (the replays reproduce the stored messages); the posterior passes differ
    # only in where the cut normalisers sit
    assert np.array_equal(full["logZ"], sub["logZ"])
    assert np.array_equal(full["N"], sub["N"])
    tol = 1e-5 if precision == "fp32" else 1e-11
    for k, v in full.items():
        assert parity.scaled_err(sub[k], v) <= tol, (k, parity.scaled_err(sub[k], v))


@pytest.mark.parametrize("name", ["small", "c1rp", "c2", "c3s", "c4s", "c5s", "shmax"])
def test_sublinear_matches_reference_goldens(name, precision):
    if name == "small":
        cases = [(i, p, c, d, u, e) for i, p, c, d, u, e in golden_io.small_cases()]
    else:
        case = golden_io.equiv_case(name)
        if case is None:
            pytest.skip("fixture missing")
        params, cum, delta, exp = case
        cases = [(name, params, cum, delta, None, exp)]
    for cid, params, cum, delta, upstream, exp in cases:
        logZ, grads, marg = scrf.posterior(cum, params, delta, upstream, memory="sublinear")
        parity.compare_posterior(logZ, grads, marg, exp, precision, nb=exp["grad_S"].shape[0])


def test_streaming_backward_replays_from_checkpoints(precision):
    """streaming_forward keeps checkpoint rows only; streaming_backward replays alpha from them."""
    case = golden_io.equiv_case("c4s")
    params, cum, delta, exp = case
    logZ, ck = scrf.streaming_forward(cum, params, delta)
    assert ck._fwd.sparse
    np.testing.assert_allclose(ck.N, exp["N"], rtol=parity.TOL[precision]["logZ"], atol=1e-9)
    grads, marg = scrf.streaming_backward(cum, params, logZ, ck)
    parity.compare_posterior(logZ, grads, marg, exp, precision)


def _mode_bytes(B, T, K, C):
    dev = torch.device("cuda", 0)
    prob = scrf.DeviceProblem(torch.zeros((B, T + 1, C), dtype=torch.float64, device=dev),
                              torch.full((B,), T, dtype=torch.int64, device=dev),
                              torch.zeros((C, C), dtype=torch.float64, device=dev),
                              torch.zeros((K, C), dtype=torch.float64, device=dev))
    lib = scrf._lib.load()
    p = prob.c_struct()
    delta = S.choose_checkpoint_interval(T, K)
    sizes = {}
    for name in ("scrf_checkpoint_bytes", "scrf_backward_work_bytes", "scrf_sparse_checkpoint_bytes",
                 "scrf_sparse_backward_work_bytes"):
        n = S.ctypes_size()
        scrf._lib.check(getattr(lib, name)(p, delta, 0, n), name)
        sizes[name] = n.value
    full = sizes["scrf_checkpoint_bytes"] + sizes["scrf_backward_work_bytes"]
    sparse = sizes["scrf_sparse_checkpoint_bytes"] + sizes["scrf_sparse_backward_work_bytes"]
    return sizes, full, sparse


def test_checkpoint_rows_are_sublinear():
    """c4 (B=8, T=1e5, K=1000, C=24): the sparse checkpoint rows are a small fraction of the
    full-memory message store, and the sparse working set grows like sqrt(T) (O(sqrt(T K) C):
    checkpoint rows, one replay window and its pass buffers) while the full one grows like T."""
    from paper_2604_18780_b200.instances import CONFIGS

    c = CONFIGS["c4"]
    B, T, K, C = c["B"], c["T"], c["K"], c["C"]
    sizes, full, sparse = _mode_bytes(B, T, K, C)
    _, full4, sparse4 = _mode_bytes(B, 4 * T, K, C)
    print(sizes, full / sparse, full4 / full, sparse4 / sparse)
    assert sizes["scrf_sparse_checkpoint_bytes"] < 0.1 * sizes["scrf_checkpoint_bytes"]
    # (the replay window rows are double-buffered so the posterior passes of one replay launch
    # overlap the next launch; at c4 the sparse working set is ~0.4 of the full one and the
    # growth checks below carry the sublinear claim)
    assert sparse < 0.45 * full
    assert full4 / full > 3.5
    assert sparse4 / sparse < 2.5


class TestRecomputeAlpha:
    """pkg/tests/test_streaming.py:167-226 on the device path, against the forward's own
    messages and the reference's replay blocks."""

    def test_every_segment_matches_forward_messages(self, precision):
        _, params, cum = scrf.equivalence_instance(9, T=23, K=4, C=3, B=2, ragged=True)
        delta = 5
        logZ, ck = scrf.streaming_forward(cum, params, delta)
        # forward alpha (fp64 oracle of the same instance) in each checkpoint's frame
        import os
        import sys

        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
        import streaming_oracle as oracle

        T = cum.max_length
        _, ock, _ = oracle.forward(cum, params, delta)
        tol = 2e-5 if precision == "fp32" else 1e-9
        for i in range(ck.n_checkpoints):
            t0, t1 = i * delta, min((i + 1) * delta, T)
            block = scrf.recompute_alpha(ck.omega[:, i], ck.N[:, i], cum, params, t0, t1)
            want = oracle.replay(ock.omega[:, i], cum, params, t0, t1)
            assert block.shape == want.shape == (2, t1 - t0 + 1, 3)
            live = want > -1e8
            np.testing.assert_array_equal(block > -1e8, live)
            np.testing.assert_allclose(block[live], want[live], atol=tol, rtol=0)

    def test_zero_length_segment_is_pure_restore(self):
        _, params, cum = scrf.equivalence_instance(4, T=12, K=3, C=2, B=1)
        _, ck = scrf.streaming_forward(cum, params, 4)
        block = scrf.recompute_alpha(ck.omega[:, 1], ck.N[:, 1], cum, params, 4, 4)
        assert block.shape == (1, 1, 2)
        np.testing.assert_array_equal(block[0, 0], ck.omega[0, 1, 4 % 3, :])

    @pytest.mark.parametrize("name", ["c3f", "c4f", "c5f"])
    def test_full_length_replay_block_matches_reference(self, name, precision):
        """The reference's own recompute_alpha block at a full BASELINE length (fixture from
        make_golden_full.py: the middle checkpoint window, sampled rows) and its omega."""
        z = golden_io.load(name)
        if z is None:
            pytest.skip(f"golden_{name}.npz not generated")
        _, params, cum = scrf.equivalence_instance(int(z["seed"]), T=int(z["T"]), K=int(z["K"]), C=int(z["C"]),
                                                   B=int(z["B"]), mode=CenteringMode(str(z["mode"])))
        assert golden_io.digest(cum.S) == str(z["S_digest"])
        kb = int(z["keep_b"])
        logZ, ck = scrf.streaming_forward(cum, params)
        assert parity.rel_err(logZ, z["logZ"]) <= parity.TOL[precision]["logZ"]
        np.testing.assert_allclose(ck.N, z["N"], rtol=parity.TOL[precision]["logZ"])
        om = ck.omega[:kb][:, z["omega_idx"]]
        want = z["omega"]
        live = want > -1e8
        np.testing.assert_array_equal(om > -1e8, live)
        tol = 2e-5 if precision == "fp32" else 1e-9
        # omega values are alpha relative to N_i: O(1e3) magnitudes at these lengths
        assert np.abs(om[live] - want[live]).max() <= tol * max(1.0, np.abs(want[live]).max())
        i = int(z["replay_i"])
        t0 = i * ck.delta
        t1 = min((i + 1) * ck.delta, int(z["T"]))
        block = scrf.recompute_alpha(ck.omega[:, i], ck.N[:, i], cum, params, t0, t1)[:kb][:, z["replay_rows"]]
        want = z["replay"]
        live = want > -1e8
        assert np.abs(block[live] - want[live]).max() <= tol * max(1.0, np.abs(want[live]).max())
