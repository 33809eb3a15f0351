"""CPU ORACLE for the streaming semi-CRF hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
leg may import it. The product path (`paper_2604_18780_b200.streaming`) never
imports anything under `oracle/` and fails loudly without its CUDA library.

It restates, in float64 numpy and in the reference's literal (unfactored)
K*C^2 form, the algorithm of `pkg/src/streamcrf/streaming.py`:

* `forward`   — streaming_forward, streaming.py:155-229 (K-slot ring, shift and
                snapshot every delta positions, dead-sequence diagnosis)
* `replay`    — recompute_alpha, streaming.py:232-261
* `backward`  — streaming_backward, streaming.py:264-408 (2K-slot beta ring,
                clipped joint marginals, per-(b, segment) workspace reduced
                segment-major then batch-major)
* `viterbi`   — streaming_viterbi, streaming.py:411-470 (reversed-duration
                argmax: ties -> longest k, then smallest source, then
                smallest final label)
* `finalize_marginals` — diagnostics.py:54-79

with the numerics of `_numerics.py:41-101` (sentinel NEG_INF = -1e9, guarded
log-sum-exp, +-1e6 clamp of finite intermediates). Viterbi keeps the
reference's exact fp64 operation order, so its paths and scores are
bit-identical to the reference's.

Pinning: `tests/golden/make_golden.py` runs the real reference
(`/root/reference/pkg/src/streamcrf`) on seeded instances and commits the
outputs as `tests/golden/*.npz`; `tests/test_oracle.py` checks this oracle
against every fixture and against the reference's own known-answer values
(ln 4, ln 88, ln 2, the T=5 tie-break path, grad_B = 2/3, 1/6, ...).
"""

from __future__ import annotations

from dataclasses import dataclass
from math import sqrt

import numpy as np

NEG_INF = -1.0e9
CLAMP = 1.0e6
_GUARD = NEG_INF + 1.0


# -- numerics (_numerics.py:41-75) -------------------------------------------


def clamp_log(v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    keep = v <= _GUARD
    if not (~keep & (np.abs(v) > CLAMP)).any():
        return v
    return np.where(keep, v, np.clip(v, -CLAMP, CLAMP))


def lse(a: np.ndarray, axis) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    m = np.max(a, axis=axis, keepdims=True)
    live = m > _GUARD
    m0 = np.where(live, m, 0.0)
    with np.errstate(under="ignore"):
        s = np.sum(np.exp(a - m0), axis=axis, keepdims=True)
    out = np.where(live, m0 + np.log(np.maximum(s, 1e-300)), NEG_INF)
    return np.squeeze(out, axis=axis)


def checkpoint_interval(T: int, K: int) -> int:
    """round(sqrt(T*K)) clamped to [1, T] (streaming.py:101-109)."""
    if T < 1:
        raise ValueError(f"sequence length must be positive, got {T}")
    return max(1, min(T, int(round(sqrt(T * K)))))


# -- segment scores (streaming.py:112-125) -----------------------------------


def _h_ending(cum, params, t: int, ks: np.ndarray) -> np.ndarray:
    """(B, len(ks), C): content + duration (+ projections) of segments [t-k, t)."""
    h = cum.S[:, t, None, :] - cum.S[:, t - ks, :] + params.duration_bias[None, ks - 1, :]
    if cum.proj_start is not None:
        h = h + cum.proj_start[:, t - ks, :]
    if cum.proj_end is not None:
        h = h + cum.proj_end[:, None, t - 1, :]
    return h


def _alpha_step(ring: np.ndarray, t: int, cum, params) -> np.ndarray:
    """alpha[t] = LSE over (k, c') of ring[t-k, c'] + T[c', c] + h[k, c] (streaming.py:128-152)."""
    K = params.max_duration
    ks = np.arange(1, min(K, t) + 1)
    h = clamp_log(_h_ending(cum, params, t, ks))  # (B, kmax, C)
    prev = ring[(t - ks) % K]  # (kmax, B, C')
    cand = prev[:, :, :, None] + params.transition[None, None] + h.transpose(1, 0, 2)[:, :, None, :]
    B, C = h.shape[0], h.shape[2]
    flat = cand.transpose(1, 0, 2, 3).reshape(B, len(ks) * C, C)
    return clamp_log(lse(flat, axis=1))


@dataclass(frozen=True)
class Checkpoints:
    omega: np.ndarray  # (B, n_ckpt, K, C): ring after the shift at i*delta
    N: np.ndarray  # (B, n_ckpt): accumulated normaliser
    delta: int


def forward(cum, params, delta: int | None = None):
    """(logZ (B,), Checkpoints, first_dead (B,)) — streaming.py:155-229.

    Raises ValueError exactly like the reference when a sequence has no finite
    path mass.
    """
    B, T, C = cum.S.shape[0], cum.S.shape[1] - 1, cum.S.shape[2]
    K = params.max_duration
    delta = checkpoint_interval(T, K) if delta is None else int(delta)
    if delta < 1:
        raise ValueError(f"checkpoint interval must be >= 1, got {delta}")
    n_ckpt = -(-T // delta)
    L = np.asarray(cum.lengths)
    ring = np.full((K, B, C), NEG_INF)
    ring[0] = 0.0
    acc = np.zeros(B)
    omega = np.empty((B, n_ckpt, K, C))
    N = np.empty((B, n_ckpt))
    omega[:, 0] = ring.transpose(1, 0, 2)
    N[:, 0] = 0.0
    first_dead = np.full(B, -1, dtype=np.int64)
    for t in range(1, T + 1):
        new = _alpha_step(ring, t, cum, params)
        live = t <= L
        dead = live & (new.max(axis=1) <= _GUARD) & (first_dead < 0)
        first_dead[dead] = t
        ring[t % K] = np.where(live[:, None], new, ring[t % K])
        if t % delta == 0:
            sh = new.max(axis=1)
            sh = np.where(live & (sh > _GUARD), sh, 0.0)
            ring = np.where(ring > _GUARD, ring - sh[None, :, None], ring)
            acc = acc + sh
            i = t // delta
            if i < n_ckpt:
                omega[:, i] = ring.transpose(1, 0, 2)
                N[:, i] = acc
    raw = lse(ring[L % K, np.arange(B)], axis=1)
    if np.any(raw <= _GUARD):
        b = int(np.argmax(raw <= _GUARD))
        td = int(first_dead[b]) if first_dead[b] >= 0 else int(L[b])
        raise ValueError(
            f"sequence {b}: log-partition diverged to -inf; every duration/source "
            f"candidate fell below the guard first at t={td}"
        )
    return raw + acc, Checkpoints(omega, N, delta), first_dead


def replay(omega_i: np.ndarray, cum, params, t0: int, t1: int) -> np.ndarray:
    """Alpha block (B, t1-t0+1, C) replayed from one snapshot (streaming.py:232-261)."""
    if not 0 <= t0 <= t1 <= cum.S.shape[1] - 1:
        raise ValueError(f"bad replay window [{t0}, {t1}] for T={cum.S.shape[1] - 1}")
    K = params.max_duration
    ring = np.ascontiguousarray(omega_i.transpose(1, 0, 2))
    out = np.empty((omega_i.shape[0], t1 - t0 + 1, omega_i.shape[2]))
    out[:, 0] = ring[t0 % K]
    L = np.asarray(cum.lengths)
    for t in range(t0 + 1, t1 + 1):
        new = _alpha_step(ring, t, cum, params)
        ring[t % K] = np.where((t <= L)[:, None], new, ring[t % K])
        out[:, t - t0] = ring[t % K]
    return out


def finalize_marginals(coverage_diff, boundary, total_mass, lengths):
    """(position (B,T,C), boundary (B,T), count (B,)) — diagnostics.py:54-79."""
    T = coverage_diff.shape[1] - 1
    pos = np.cumsum(coverage_diff, axis=1)[:, :T, :]
    valid = np.arange(T)[None, :] < np.asarray(lengths)[:, None]
    pos = np.where(valid[:, :, None], np.clip(pos, 0.0, 1.0), 0.0)
    bnd = np.where(valid, np.clip(boundary, 0.0, 1.0), 0.0)
    return pos, bnd, np.asarray(total_mass, dtype=np.float64)


@dataclass
class _BwdState:
    beta: np.ndarray
    work: np.ndarray
    gS: np.ndarray
    gPs: np.ndarray | None
    gPe: np.ndarray | None
    cov: np.ndarray
    bnd: np.ndarray
    mass: np.ndarray
    scale: np.ndarray
    L: np.ndarray
    R: int
    proj: bool


def _beta_step(st: _BwdState, cum, params, t: int, i: int, alpha_t: np.ndarray, shift: np.ndarray) -> None:
    """One backward position: beta[t], joint marginals of segments starting at t (streaming.py:337-387)."""
    B, T, C = cum.S.shape[0], cum.S.shape[1] - 1, cum.S.shape[2]
    K = params.max_duration
    trans = params.transition
    ks = np.arange(1, min(K, T - t) + 1)
    h = cum.S[:, t + ks, :] - cum.S[:, t, None, :] + params.duration_bias[None, : len(ks), :]
    if st.proj:
        h = h + cum.proj_start[:, None, t, :] + cum.proj_end[:, t + ks - 1, :]
    h = clamp_log(h)
    hb = h + st.beta[(t + ks) % st.R].transpose(1, 0, 2)  # (B, kmax, C)
    ok = (t + ks)[None, :] <= st.L[:, None]
    hb = np.where(ok[:, :, None], hb, NEG_INF)
    q = hb[:, :, None, :] + trans[None, None]  # (B, kmax, C', C)
    nb = lse(q.transpose(0, 2, 1, 3).reshape(B, C, len(ks) * C), axis=2)
    lm = hb[:, :, :, None] + trans.T[None, None] + alpha_t[:, None, None, :]
    lm = lm + shift[:, None, None, None]
    np.clip(lm, -80.0, 80.0, out=lm)
    mu = np.where(ok[:, :, None, None], np.exp(lm), 0.0)
    mug = mu * st.scale[:, None, None, None]
    st.work[:, i, : len(ks)] += mug
    post = mu.sum(axis=3)
    grad = mug.sum(axis=3)
    st.gS[:, t, :] -= grad.sum(axis=1)
    st.gS[:, t + ks, :] += grad
    if st.proj:
        st.gPs[:, t, :] += grad.sum(axis=1)
        st.gPe[:, t + ks - 1, :] += grad
    st.cov[:, t, :] += post.sum(axis=1)
    st.cov[:, t + ks, :] -= post
    s0 = post.sum(axis=(1, 2))
    st.bnd[:, t] += s0
    st.mass += s0
    w = t < st.L
    st.beta[t % st.R] = np.where(w[:, None], clamp_log(nb), st.beta[t % st.R])


def steady_position_seconds(cum, params, n_steps: int = 8) -> float:
    """CPU seconds per position of fwd + replay + bwd in steady state (t >= K, t + K <= T).

    Times the oracle's own per-position bodies (`_alpha_step`, `_beta_step`) on a
    primed state; per-position cost is value-independent once t >= K (numpy
    does the same work), which is how BASELINE.md §4 extrapolates c4/c5.
    """
    import time

    B, T, C = cum.S.shape[0], cum.S.shape[1] - 1, cum.S.shape[2]
    K = params.max_duration
    ring = np.zeros((K, B, C))
    t_lo = K
    if K + n_steps + 1 > T:
        raise ValueError("instance too short for a steady-state sample")
    t0 = time.perf_counter()
    for t in range(t_lo + 1, t_lo + 1 + n_steps):
        ring[t % K] = _alpha_step(ring, t, cum, params)
    t_fwd = (time.perf_counter() - t0) / n_steps
    R = 2 * K
    st = _BwdState(np.zeros((R, B, C)), np.zeros((B, 1, K, C, C)), np.zeros((B, T + 1, C)), None, None,
                   np.zeros((B, T + 1, C)), np.zeros((B, T)), np.zeros(B), np.ones(B),
                   np.asarray(cum.lengths), R, cum.proj_start is not None)
    if st.proj:
        st.gPs, st.gPe = np.zeros((B, T, C)), np.zeros((B, T, C))
    alpha_t = np.zeros((B, C))
    shift = np.zeros(B)
    t0 = time.perf_counter()
    for t in range(n_steps, 0, -1):  # t + K <= T: every duration is live
        _beta_step(st, cum, params, t, 0, alpha_t, shift)
    t_bwd = (time.perf_counter() - t0) / n_steps
    return 2.0 * t_fwd + t_bwd  # forward + replay + backward per position (B sequences)


def backward(cum, params, logZ, ckpts: Checkpoints, upstream=None) -> dict:
    """Gradients + marginals by checkpointed replay (streaming.py:264-408).

    Returns a dict with grad_S, grad_T, grad_B, grad_P_start, grad_P_end,
    position_marginals, boundary_posterior, expected_segment_count.
    """
    B, T, C = cum.S.shape[0], cum.S.shape[1] - 1, cum.S.shape[2]
    K = params.max_duration
    delta = ckpts.delta
    n_ckpt = ckpts.omega.shape[1]
    if n_ckpt != -(-T // delta):
        raise RuntimeError(f"checkpoint set holds {n_ckpt} segments; T={T} with delta={delta}")
    L = np.asarray(cum.lengths)
    scale = np.ones(B) if upstream is None else np.asarray(upstream, dtype=np.float64)
    if scale.shape != (B,):
        raise ValueError(f"upstream must be shaped ({B},), got {scale.shape}")
    trans = params.transition
    logZ = np.asarray(logZ, dtype=np.float64)

    R = 2 * K
    beta = np.full((R, B, C), NEG_INF)
    beta[L % R, np.arange(B)] = 0.0
    work = np.zeros((B, n_ckpt, K, C, C))  # [k, label, source]
    gS = np.zeros((B, T + 1, C))
    proj = cum.proj_start is not None  # reference quirk: both-or-neither (streaming.py:325)
    gPs = np.zeros((B, T, C)) if proj else None
    gPe = np.zeros((B, T, C)) if proj else None
    cov = np.zeros((B, T + 1, C))
    bnd = np.zeros((B, T))
    mass = np.zeros(B)

    st = _BwdState(beta, work, gS, gPs, gPe, cov, bnd, mass, scale, L, R, proj)
    for i in range(n_ckpt - 1, -1, -1):
        t0, t1 = i * delta, min((i + 1) * delta, T)
        alpha = replay(ckpts.omega[:, i], cum, params, t0, t1)
        shift = ckpts.N[:, i] - logZ
        for t in range(t1 - 1, t0 - 1, -1):
            _beta_step(st, cum, params, t, i, alpha[:, t - t0], shift)

    gT = np.zeros((C, C))
    gB = np.zeros((K, C))
    for i in range(n_ckpt):
        for b in range(B):
            gT += work[b, i].sum(axis=0).T
            gB += work[b, i].sum(axis=2)
    pos, bp, cnt = finalize_marginals(cov, bnd, mass, L)
    return dict(
        grad_S=gS, grad_T=gT, grad_B=gB, grad_P_start=gPs, grad_P_end=gPe,
        position_marginals=pos, boundary_posterior=bp, expected_segment_count=cnt,
    )


def viterbi(cum, params):
    """(list of segment tuples per sequence, scores (B,)) — streaming.py:411-470.

    Same fp64 operation order as the reference: cand = (prev + T) + h with
    h = ((S[t] - S[t-k]) + B) (+ Ps) (+ Pe); the first maximum of the
    reversed-duration flattening wins.
    """
    B, T, C = cum.S.shape[0], cum.S.shape[1] - 1, cum.S.shape[2]
    K = params.max_duration
    ring = np.full((K, B, C), NEG_INF)
    ring[0] = 0.0
    back_k = np.zeros((T + 1, B, C), dtype=np.int64)
    back_c = np.zeros((T + 1, B, C), dtype=np.int64)
    L = np.asarray(cum.lengths)
    for t in range(1, T + 1):
        kmax = min(K, t)
        ks = np.arange(1, kmax + 1)
        h = _h_ending(cum, params, t, ks)
        prev = ring[(t - ks) % K]
        cand = prev.transpose(1, 0, 2)[:, :, :, None] + params.transition[None, None] + h[:, :, None, :]
        rev = cand[:, ::-1].reshape(B, kmax * C, C)
        arg = np.argmax(rev, axis=1)
        best = np.take_along_axis(rev, arg[:, None, :], axis=1)[:, 0, :]
        kr, src = np.divmod(arg, C)
        ring[t % K] = np.where((t <= L)[:, None], best, ring[t % K])
        back_k[t] = kmax - kr
        back_c[t] = src
    paths, scores = [], np.empty(B)
    for b in range(B):
        t = int(L[b])
        fin = ring[t % K, b]
        c = int(np.argmax(fin))
        scores[b] = fin[c]
        segs = []
        while t > 0:
            k = int(back_k[t, b, c])
            segs.append((t - k, t, c))
            c = int(back_c[t, b, c])
            t -= k
        paths.append(tuple(reversed(segs)))
    return paths, scores


def posterior(cum, params, delta=None, upstream=None):
    logZ, ck, _ = forward(cum, params, delta)
    return logZ, backward(cum, params, logZ, ck, upstream)
