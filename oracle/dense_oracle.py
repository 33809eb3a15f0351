"""Dense semi-CRF DP and path enumeration -- CPU test oracle (TEST INFRASTRUCTURE ONLY).

Restates the reference's dense backend (pkg/src/streamcrf/reference.py) so the reference's own
contract tests (tests/reference_contract/) can run where /root/reference does not exist (the
GPU box): full (B, T+1, C) alpha / beta tables, the joint segment marginals
mu[b, e, k-1, c, c'] and Viterbi with backpointers. Only tests import this module; the
product path never does.

  dense_forward            reference.py:174-202
  dense_backward_marginals reference.py:205-283
  dense_viterbi            reference.py:330-368 (ties: longest k, then smallest c', _numerics.py:78-89)
  enumerate_logZ           reference.py:126-139 (every source label x tiling x labelling)
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

NEG_INF = -1.0e9
_GUARD = NEG_INF + 1.0


def lse(a: np.ndarray, axis) -> np.ndarray:
    """Guarded log-sum-exp: slices whose max is at or below the guard give the sentinel."""
    a = np.asarray(a, dtype=np.float64)
    m = np.max(a, axis=axis, keepdims=True)
    ok = m > _GUARD
    base = np.where(ok, m, 0.0)
    with np.errstate(under="ignore", divide="ignore"):
        out = base + np.log(np.maximum(np.sum(np.exp(a - base), axis=axis, keepdims=True), 1e-300))
    return np.squeeze(np.where(ok, out, NEG_INF), axis=axis)


@dataclass
class DenseMessages:
    alpha: np.ndarray  # (B, T+1, C): prefixes whose last segment ends at t with label c
    beta: np.ndarray | None  # (B, T+1, C): suffixes from boundary t given previous label c'
    logZ: np.ndarray  # (B,)


def _edges_ending(cum, params, t: int, kmax: int) -> np.ndarray:
    """h[b, k-1, c] of the segments [t-k, t), k = 1..kmax."""
    ks = np.arange(1, kmax + 1)
    h = (cum.S[:, t][:, None, :] - cum.S[:, t - ks]) + params.duration_bias[:kmax][None]
    if cum.proj_start is not None:
        h = h + cum.proj_start[:, t - ks]
    if cum.proj_end is not None:
        h = h + cum.proj_end[:, t - 1][:, None, :]
    return h


def dense_forward(cum, params, ledger=None) -> DenseMessages:
    B, T1, C = cum.S.shape
    T, K = T1 - 1, params.max_duration
    L = np.asarray(cum.lengths)
    alpha = np.full((B, T + 1, C), NEG_INF)
    alpha[:, 0] = 0.0
    for t in range(1, T + 1):
        kmax = min(K, t)
        h = _edges_ending(cum, params, t, kmax)  # (B, k, c)
        prev = alpha[:, t - np.arange(1, kmax + 1)]  # (B, k, c')
        cand = (prev[:, :, :, None] + params.transition[None, None]) + h[:, :, None, :]  # (B, k, c', c)
        new = lse(cand.reshape(B, kmax * C, C), axis=1)
        live = t <= L
        alpha[live, t] = new[live]
    logZ = lse(alpha[np.arange(B), L], axis=1)
    return DenseMessages(alpha, None, logZ)


def dense_backward_marginals(cum, params, msgs: DenseMessages, ledger=None):
    """(mu (B, T+1, K, C, C'), GradientSet) with mu indexed by segment end."""
    from paper_2604_18780_b200.diagnostics import GradientSet

    S = cum.S
    B, T1, C = S.shape
    T, K = T1 - 1, params.max_duration
    L = np.asarray(cum.lengths)
    beta = np.full((B, T + 1, C), NEG_INF)
    beta[np.arange(B), L] = 0.0
    mu = np.zeros((B, T + 1, K, C, C))
    for b in range(B):
        for t in range(int(L[b]) - 1, -1, -1):
            kmax = min(K, int(L[b]) - t)
            ks = np.arange(1, kmax + 1)
            h = (S[b, t + ks] - S[b, t][None]) + params.duration_bias[:kmax]
            if cum.proj_start is not None:
                h = h + cum.proj_start[b, t][None]
            if cum.proj_end is not None:
                h = h + cum.proj_end[b, t + ks - 1]
            hb = h + beta[b, t + ks]  # (k, c)
            q = hb[:, None, :] + params.transition[None]  # (k, c', c)
            beta[b, t] = lse(q.transpose(1, 0, 2).reshape(C, kmax * C), axis=1)
            lm = hb[:, :, None] + params.transition.T[None] + msgs.alpha[b, t][None, None, :] - msgs.logZ[b]
            mu[b, t + ks, ks - 1] = np.exp(np.minimum(lm, 0.0))
    np.clip(mu, 0.0, 1.0, out=mu)
    msgs.beta = beta
    seg = mu.sum(axis=4)  # (B, T+1, K, C) by end
    gS = seg.sum(axis=2).copy()
    gPs = np.zeros((B, T, C)) if cum.proj_start is not None else None
    gPe = np.zeros((B, T, C)) if cum.proj_end is not None else None
    for k in range(1, min(K, T) + 1):
        ends = seg[:, k:, k - 1]
        gS[:, : T + 1 - k] -= ends
        if gPs is not None:
            gPs[:, : T + 1 - k] += ends
        if gPe is not None:
            gPe[:, k - 1 : T] += ends
    grads = GradientSet(grad_S=gS, grad_T=mu.sum(axis=(0, 1, 2)).T, grad_B=seg.sum(axis=(0, 1)),
                        grad_P_start=gPs, grad_P_end=gPe)
    return mu, grads


def dense_viterbi(cum, params, b: int = 0, ledger=None):
    from paper_2604_18780_b200.potentials import Segmentation

    L = int(cum.lengths[b])
    C, K = params.num_labels, params.max_duration
    best = np.full((L + 1, C), NEG_INF)
    best[0] = 0.0
    back = np.zeros((L + 1, C, 2), dtype=np.int64)
    for t in range(1, L + 1):
        kmax = min(K, t)
        h = _edges_ending(cum, params, t, kmax)[b]  # (k, c)
        prev = best[t - np.arange(1, kmax + 1)]  # (k, c')
        cand = (prev[:, :, None] + params.transition[None]) + h[:, None, :]  # (k, c', c)
        for c in range(C):
            flat = cand[::-1, :, c].reshape(-1)  # longest k first, then smallest c'
            j = int(np.argmax(flat))
            ki, cp = kmax - 1 - j // C, j % C
            best[t, c] = cand[ki, cp, c]
            back[t, c] = (ki + 1, cp)
    c = int(np.argmax(best[L]))
    score = float(best[L, c])
    segs, t = [], L
    while t > 0:
        k, cp = (int(v) for v in back[t, c])
        segs.append((t - k, t, c))
        t, c = t - k, cp
    return Segmentation(tuple(reversed(segs))), score


def _tilings(n: int, K: int):
    if n == 0:
        yield ()
        return
    for k in range(1, min(K, n) + 1):
        for rest in _tilings(n - k, K):
            yield (k,) + rest


def enumerate_logZ(cum, params, b: int = 0) -> float:
    """log sum over (virtual source, tiling, labelling) of the path score."""
    L = int(cum.lengths[b])
    C = params.num_labels
    S = cum.S[b]
    scores = []
    for durs in _tilings(L, params.max_duration):
        bounds = np.concatenate([[0], np.cumsum(durs)]).astype(int)
        for labels in itertools.product(range(C), repeat=len(durs)):
            body = 0.0
            for i, c in enumerate(labels):
                s, e = bounds[i], bounds[i + 1]
                body += (S[e, c] - S[s, c]) + params.duration_bias[e - s - 1, c]
                if cum.proj_start is not None:
                    body += cum.proj_start[b, s, c] + cum.proj_end[b, e - 1, c]
                if i:
                    body += params.transition[labels[i - 1], c]
            for src in range(C):
                scores.append(params.transition[src, labels[0]] + body)
    return float(lse(np.array(scores), axis=0))
