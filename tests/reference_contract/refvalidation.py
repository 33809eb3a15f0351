"""`streamcrf.validation` for the contract suite (TEST INFRASTRUCTURE ONLY).

The acceptance criteria call three harness functions of the reference's validation module
(pkg/src/streamcrf/validation.py); they are restated here over this package's device API
(the "streaming" backend) and oracle/dense_oracle.py (the "dense" backend):

  backend_equivalence       validation.py:235-337  (k1/k2 routes omitted: no fast paths)
  finite_diff_gradcheck     validation.py:79-165
  training_convergence_demo validation.py:344-491  (the synthetic batch and the reference's
                            own dense-backend curve come from tests/golden/golden_train.npz,
                            produced by the real reference; the streaming curve is computed
                            here through the device posterior)
"""

from __future__ import annotations

import os
from dataclasses import replace

import numpy as np

import dense_oracle as D
from paper_2604_18780_b200.instances import equivalence_instance  # noqa: F401  (re-exported)
from paper_2604_18780_b200.potentials import (
    CenteringMode, EmissionBatch, Segmentation, SemiCRFParams, build_scores,
)
from paper_2604_18780_b200.streaming import decode, forward_logZ, posterior, streaming_viterbi

COSINE_MIN = 0.9999
NORM_MAX_ERR_MAX = 5e-5
_MODES = (CenteringMode.NONE, CenteringMode.MEAN, CenteringMode.SHARED_MAX)
DEFAULT_TRAIN_CONFIG = {"B": 4, "T": 160, "C": 12, "K": 12, "lr": 0.05, "seed": 20240817, "train_emissions": True}
GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "golden")


def _tol(x: float) -> float:
    from refconf import F

    return F(x)


def _cos(a, b) -> float:
    a, b = np.ravel(a), np.ravel(b)
    na, nb = float(np.linalg.norm(a)), float(np.linalg.norm(b))
    if na == 0.0 and nb == 0.0:
        return 1.0
    return 0.0 if na == 0.0 or nb == 0.0 else float(a @ b / (na * nb))


def _nme(analytic, numeric) -> float:
    return float(np.abs(analytic - numeric).max(initial=0.0)) / max(1.0, float(np.abs(numeric).max(initial=0.0)))


def _rel(a, b) -> float:
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def backend_equivalence(trials, max_T=6, max_K=3, max_C=3, seed=0, *, max_B=2) -> dict:
    """Streaming (device) vs dense vs enumeration on random small instances: log Z, gradients,
    Viterbi paths (dims drawn exactly as validation.py:268-276)."""
    failures, rows = [], []
    worst_z = worst_g = 0.0
    enumerated = 0
    for trial in range(trials):
        d = np.random.default_rng([seed, trial])
        T, K, C, B = (int(d.integers(1, m + 1)) for m in (max_T, max_K, max_C, max_B))
        mode = _MODES[int(d.integers(0, 3))]
        ragged = B > 1 and bool(d.integers(0, 2))
        proj = bool(d.integers(0, 4) == 0)
        _, params, cum = equivalence_instance(seed, T=T, K=K, C=C, B=B, mode=mode, ragged=ragged, projections=proj)
        row = dict(trial=trial, T=T, K=K, C=C, B=B, ok=True, enumerated=False)

        def fail(stage, msg):
            row["ok"] = False
            failures.append(dict(row, stage=stage, detail=msg))

        dense = D.dense_forward(cum, params)
        z = forward_logZ(cum, params)
        r = _rel(z, dense.logZ)
        worst_z = max(worst_z, r)
        if r > _tol(1e-9):
            fail("logZ", f"rel {r:.2e}")
        if T <= 12 and K <= 4 and C <= 4:
            row["enumerated"] = True
            enumerated += 1
            for b in range(B):
                e = D.enumerate_logZ(cum, params, b)
                r = abs(e - float(dense.logZ[b])) / max(1.0, abs(e))
                worst_z = max(worst_z, r)
                if r > _tol(1e-9):
                    fail("enumeration", f"b={b} rel {r:.2e}")
        _, gd = D.dense_backward_marginals(cum, params, dense)
        _, gs, _ = posterior(cum, params)
        g = 0.0
        for k in ("grad_S", "grad_T", "grad_B", "grad_P_start", "grad_P_end"):
            a_, b_ = getattr(gd, k), getattr(gs, k)
            if a_ is None and b_ is None:
                continue
            g = max(g, _nme(b_, a_))
        worst_g = max(worst_g, g)
        if g > _tol(1e-8):
            fail("gradients", f"{g:.2e}")
        paths, _ = streaming_viterbi(cum, params)
        paths2, _ = decode(cum, params)
        for b in range(B):
            seg, _ = D.dense_viterbi(cum, params, b)
            if seg.segments != paths[b].segments or seg.segments != paths2[b].segments:
                fail("viterbi", f"b={b}")
        rows.append(row)
    return {"trials": trials, "seed": seed, "rows": rows, "failures": failures, "all_pass": not failures,
            "enumerated": enumerated, "max_rel_logZ": worst_z, "max_grad_diff": worst_g}


def finite_diff_gradcheck(cum, params, eps, *, include_grads=False) -> dict:
    """Central differences of sum_b log Z over every element (forward passes only) against the
    device backward (validation.py:79-165)."""
    _, grads, _ = posterior(cum, params)

    def f(c2, p2):
        return float(forward_logZ(c2, p2).sum())

    def sweep(base, rebuild):
        num = np.zeros_like(base)
        flat, src = num.reshape(-1), base.reshape(-1)
        for i in range(src.size):
            x = src.copy()
            x[i] = src[i] + eps
            hi = f(*rebuild(x.reshape(base.shape)))
            x[i] = src[i] - eps
            lo = f(*rebuild(x.reshape(base.shape)))
            flat[i] = (hi - lo) / (2.0 * eps)
        return num

    pairs = {
        "cum_scores": (grads.grad_S[:, 1:], sweep(cum.S[:, 1:], lambda blk: (
            replace(cum, S=np.concatenate([cum.S[:, :1], blk], axis=1)), params))),
        "transition": (grads.grad_T, sweep(params.transition, lambda t2: (cum, replace(params, transition=t2)))),
        "duration_bias": (grads.grad_B, sweep(params.duration_bias,
                                              lambda b2: (cum, replace(params, duration_bias=b2)))),
    }
    tensors, ok = {}, True
    for name, (an, nu) in pairs.items():
        row = {"elements": int(nu.size), "cosine": _cos(an, nu), "norm_max_err": _nme(an, nu)}
        ok = ok and row["cosine"] >= COSINE_MIN and row["norm_max_err"] < NORM_MAX_ERR_MAX
        tensors[name] = row
    return {"eps": float(eps), "tensors": tensors, "passed": ok}


def _gold_stats(cum, params, golds):
    """Gold log-scores (summed over the virtual source) and their gradients in (e, T, B)."""
    B, T, C = cum.S.shape[0], cum.S.shape[1] - 1, cum.S.shape[2]
    K = params.max_duration
    scores = np.zeros(B)
    ge, gT, gB = np.zeros((B, T, C)), np.zeros((C, C)), np.zeros((K, C))
    for b, g in enumerate(golds):
        body, prev = 0.0, None
        for s, e, c in g.segments:
            body += (cum.S[b, e, c] - cum.S[b, s, c]) + params.duration_bias[e - s - 1, c]
            if prev is not None:
                body += params.transition[prev, c]
            prev = c
        first = g.segments[0][2]
        src = params.transition[:, first] + body
        m = src.max()
        scores[b] = m + np.log(np.exp(src - m).sum())
        p_src = np.exp(src - scores[b])
        prev = None
        for s, e, c in g.segments:
            ge[b, s:e, c] += 1.0
            gB[e - s - 1, c] += 1.0
            if prev is None:
                gT[:, c] += p_src
            else:
                gT[prev, c] += 1.0
            prev = c
    return scores, ge, gT, gB


def training_convergence_demo(config=None, epochs=100, backends=("dense", "streaming")) -> dict:
    """Plain gradient descent from identical state, one run per backend (validation.py:438-491).
    dense: the real reference's recorded curve; streaming: the device posterior."""
    z = dict(np.load(os.path.join(GOLDEN, "golden_train.npz")))
    B, T, C, K = (int(z[k]) for k in ("B", "T", "C", "K"))
    lr = float(z["lr"])
    golds = [Segmentation(tuple(tuple(int(v) for v in row) for row in z[f"gold_{b}"])) for b in range(B)]
    L = np.full(B, T, dtype=np.int64)
    out = {}
    for backend in backends:
        if backend == "dense":
            curve = [float(v) for v in z["dense_curve"][: epochs + 1]]
        else:
            e = z["emissions"].copy()
            tm, bm = np.zeros((C, C)), np.zeros((K, C))

            def evaluate():
                cum = build_scores(EmissionBatch(e, L), SemiCRFParams(tm, bm), CenteringMode.NONE)
                logZ, grads, _ = posterior(cum, SemiCRFParams(tm, bm))
                ge_model = grads.grad_S[:, :0:-1, :].cumsum(axis=1)[:, ::-1, :]  # suffix sums (validation.py:410)
                gs, ge, gT, gB = _gold_stats(cum, SemiCRFParams(tm, bm), golds)
                return float(np.mean(logZ - gs)), (ge_model - ge) / B, (grads.grad_T - gT) / B, (grads.grad_B - gB) / B

            nll, g_e, g_T, g_B = evaluate()
            curve = [nll]
            for _ in range(epochs):
                e = e - lr * g_e
                tm = tm - lr * g_T
                bm = bm - lr * g_B
                nll, g_e, g_T, g_B = evaluate()
                curve.append(nll)
        streak, div = 0, None
        for i in range(1, len(curve)):
            streak = streak + 1 if curve[i] > curve[i - 1] else 0
            if streak >= 5 and div is None:
                div = i - 1
        out[backend] = {"curve": curve, "final": curve[-1], "diverged": div is not None, "diverged_at": div}
    rep = {"epochs": epochs, "backends": out, "final_rel_diff": None, "curve_cosine": None}
    if len(backends) >= 2:
        a, b = out[backends[0]], out[backends[1]]
        rep["final_rel_diff"] = abs(b["final"] - a["final"]) / max(abs(a["final"]), 1e-12)
        rep["curve_cosine"] = _cos(np.array(a["curve"]), np.array(b["curve"]))
    return rep
