"""Pin the CPU oracle (oracle/streaming_oracle.py) before trusting it.

The oracle is checked against (a) every golden fixture produced by running the
real reference (tests/golden/make_golden.py) and (b) the reference tests'
known-answer values for this path (test_streaming.py:85-88, 229-236, 352-355,
411-414; test_reference.py:65-68, 322-336; test_validation.py:30-43). CPU only.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import streaming_oracle as O  # noqa: E402

import golden_io  # noqa: E402
from paper_2604_18780_b200.potentials import (  # noqa: E402
    CenteredEmissions, CenteringMode, SemiCRFParams, build_cumulative,
)


def cum_from_centered(centered, lengths=None):
    centered = np.asarray(centered, dtype=np.float64)
    if centered.ndim == 2:
        centered = centered[None]
    B, T, C = centered.shape
    L = np.full(B, T, dtype=np.int64) if lengths is None else np.asarray(lengths, np.int64)
    return build_cumulative(CenteredEmissions(centered, L, CenteringMode.NONE, np.zeros((B, C))))


def zero_params(K, C):
    return SemiCRFParams(np.zeros((C, C)), np.zeros((K, C)))


def check_against(expected, logZ, N, grads, segs, scores, tol=1e-12):
    np.testing.assert_allclose(logZ, expected["logZ"], rtol=tol, atol=0)
    np.testing.assert_allclose(N, expected["N"], rtol=tol, atol=tol)
    nb = expected["grad_S"].shape[0]
    for key in ("grad_S", "position_marginals", "boundary_posterior", "grad_P_start", "grad_P_end"):
        if key in expected:
            np.testing.assert_allclose(grads[key][:nb], expected[key], atol=tol, err_msg=key)
    for key in ("grad_T", "grad_B", "expected_segment_count"):
        np.testing.assert_allclose(grads[key], expected[key], atol=tol * max(1.0, np.abs(expected[key]).max()), err_msg=key)
    assert [tuple(p) for p in segs] == expected["vit_segments"]
    assert np.array_equal(scores, expected["vit_scores"])  # bit-exact


def test_oracle_matches_reference_small_fixtures():
    n = 0
    for i, params, cum, delta, up, exp in golden_io.small_cases():
        logZ, ck, _ = O.forward(cum, params, delta)
        grads = O.backward(cum, params, logZ, ck, up)
        segs, scores = O.viterbi(cum, params)
        check_against(exp, logZ, ck.N, grads, segs, scores)
        n += 1
    assert n >= 40


@pytest.mark.parametrize("name", ["c1", "c1rp", "shmax", "c3s"])
def test_oracle_matches_reference_equiv_fixtures(name):
    case = golden_io.equiv_case(name)
    if case is None:
        pytest.skip(f"fixture {name} not generated")
    params, cum, delta, exp = case
    logZ, ck, _ = O.forward(cum, params, delta)
    grads = O.backward(cum, params, logZ, ck)
    segs, scores = O.viterbi(cum, params)
    check_against(exp, logZ, ck.N, grads, segs, scores)


class TestKnownAnswers:
    def test_one_position_two_labels_ln4(self):
        logZ, _, _ = O.forward(cum_from_centered(np.zeros((1, 2))), zero_params(1, 2))
        assert logZ[0] == pytest.approx(math.log(4.0), abs=1e-12)

    def test_T4_K2_C2_ln88(self):
        logZ, _, _ = O.forward(cum_from_centered(np.zeros((4, 2))), zero_params(2, 2))
        assert logZ[0] == pytest.approx(math.log(88.0), abs=1e-12)

    def test_two_positions_one_label_ln2(self):
        logZ, _, _ = O.forward(cum_from_centered(np.zeros((2, 1))), zero_params(2, 1))
        assert logZ[0] == pytest.approx(math.log(2.0), abs=1e-12)

    def test_single_path_gradients(self):
        cum, params = cum_from_centered(np.zeros((1, 1))), zero_params(1, 1)
        logZ, g = O.posterior(cum, params)
        assert g["grad_B"][0, 0] == pytest.approx(1.0, abs=1e-12)
        assert g["grad_T"][0, 0] == pytest.approx(1.0, abs=1e-12)
        assert g["position_marginals"][0, 0, 0] == pytest.approx(1.0, abs=1e-12)

    def test_zero_score_duration_gradients(self):
        # test_validation.py:30-43: T=2, K=2, C=2 all zero -> grad_B[1] = 1/6, grad_B[0] = 2/3
        cum, params = cum_from_centered(np.zeros((2, 2))), zero_params(2, 2)
        _, g = O.posterior(cum, params)
        np.testing.assert_allclose(g["grad_B"][1], 1.0 / 6.0, atol=1e-12)
        np.testing.assert_allclose(g["grad_B"][0], 2.0 / 3.0, atol=1e-12)

    def test_viterbi_tie_break_longest_first(self):
        segs, _ = O.viterbi(cum_from_centered(np.zeros((5, 2))), zero_params(2, 2))
        assert segs[0] == ((0, 1, 0), (1, 3, 0), (3, 5, 0))

    def test_forced_boundary_path(self):
        # test_reference.py:322-336
        em = np.zeros((5, 2))
        em[:3, 1], em[:3, 0], em[3:, 0], em[3:, 1] = 5.0, -5.0, 5.0, -5.0
        params = SemiCRFParams(np.array([[0.0, -2.0], [-2.0, 0.0]]), np.zeros((4, 2)))
        segs, scores = O.viterbi(cum_from_centered(em), params)
        assert segs[0] == ((0, 3, 1), (3, 5, 0))
        assert scores[0] == pytest.approx(23.0, abs=1e-12)

    def test_checkpoint_interval_table(self):
        for T, K, want in [(100, 25, 50), (1, 1, 1), (1000, 8, 89), (100_000, 8, 894), (1_000_000, 200, 14_142), (4, 25, 4)]:
            assert O.checkpoint_interval(T, K) == want

    def test_dead_sequence_diagnosed(self):
        params = SemiCRFParams(np.zeros((2, 2)), np.full((2, 2), -2.0e9))
        with pytest.raises(ValueError, match=r"t=1"):
            O.forward(cum_from_centered(np.zeros((6, 2))), params)
