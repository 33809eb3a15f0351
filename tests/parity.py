"""Tolerances and comparison helpers shared by the GPU parity tests.

Bars, against the fp64 reference / oracle:
  fp32 kernels: logZ <= 1e-5 relative; gradients and marginals <= MARG_TOL in the
                reference's own metric max|d| / max(1, max|ref|) (validation.py:215-232)
  fp64 kernels: logZ <= 1e-9 relative; gradients / marginals <= 1e-8 (test_streaming.py:98, 246)
  Viterbi:      segments and scores bit-identical.
"""

from __future__ import annotations

import numpy as np

TOL = {
    "fp32": dict(logZ=1e-5, grad=1e-5),
    "fp64": dict(logZ=1e-9, grad=1e-8),
}


def scaled_err(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if want.size == 0:
        return 0.0
    return float(np.abs(got - want).max() / max(1.0, float(np.abs(want).max())))


def rel_err(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))))


GRAD_KEYS = ("grad_S", "grad_T", "grad_B", "grad_P_start", "grad_P_end")
MARG_KEYS = ("position_marginals", "boundary_posterior", "expected_segment_count")


def compare_posterior(logZ, grads, marg, expected, precision: str, nb: int | None = None) -> dict:
    """Returns {name: error}; asserts every error is within the precision's bar."""
    tol = TOL[precision]
    errs = {"logZ": rel_err(logZ, expected["logZ"])}
    nb = nb if nb is not None else expected["grad_S"].shape[0]
    for k in GRAD_KEYS:
        if k not in expected or expected[k] is None:
            continue
        got = getattr(grads, k)
        assert got is not None, f"{k} missing"
        if k in ("grad_T", "grad_B"):
            errs[k] = scaled_err(got, expected[k])
        else:
            errs[k] = scaled_err(got[:nb], expected[k])
    for k in MARG_KEYS:
        got = getattr(marg, k)
        want = expected[k]
        errs[k] = scaled_err(got if k == "expected_segment_count" else got[:nb], want)
    bad = {k: v for k, v in errs.items() if v > (tol["logZ"] if k == "logZ" else tol["grad"])}
    assert not bad, f"parity failure ({precision}): {bad} (all: {errs})"
    return errs
