"""Full-length golden vectors from the REAL reference (build container only).

SURVEY §7.1 asks for a full-T config-4 fixture so that fp32 parity is pinned at
the benchmarked sequence length, not only at truncated T. The reference is
pure numpy on one core, so these runs take ~1-2 h each; they are started in the
background:

    nohup python tests/golden/make_golden_full.py c4f > /tmp/c4f.log 2>&1 &

Per-position arrays (grad_S, marginals, boundary) are stored on a fixed row
sample (`rows`: first 512, last 512 and every 64th boundary) to keep the
fixtures small; scalars, grad_T/grad_B, N, Viterbi segments and scores are
stored in full; Omega and one `recompute_alpha` block on a subset of
checkpoints/rows (`omega_idx`, `replay_i`, `replay_rows`).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from make_golden import flat_segments, s_digest  # noqa: E402
from streamcrf import potentials as P  # noqa: E402  (the reference)
from streamcrf.streaming import (  # noqa: E402
    recompute_alpha, streaming_backward, streaming_forward, streaming_viterbi,
)
from streamcrf.validation import equivalence_instance  # noqa: E402


def sample_rows(n: int) -> np.ndarray:
    rows = set(range(min(512, n))) | set(range(max(0, n - 512), n)) | set(range(0, n, 64))
    return np.array(sorted(rows), np.int64)


def make_full(name, seed, T, K, C, B, mode, ragged=False, projections=False, keep_b=1):
    t0 = time.time()
    _, params, cum = equivalence_instance(
        seed, T=T, K=K, C=C, B=B, mode=mode, ragged=ragged, projections=projections
    )
    logZ, ck = streaming_forward(cum, params)
    print(f"{name}: forward {time.time() - t0:.0f}s logZ={logZ}", flush=True)
    n_ck = ck.N.shape[1]
    ri = n_ck // 2
    t_lo = ri * ck.delta
    t_hi = min((ri + 1) * ck.delta, T)
    # a COPY of the snapshot: with B = 1 the reference's recompute_alpha restores its ring as a
    # view of omega_i (np.ascontiguousarray of a size-1-axis transpose is a view) and would
    # overwrite the checkpoint set that streaming_backward replays from next
    block = recompute_alpha(ck.omega[:, ri].copy(), ck.N[:, ri], cum, params, t_lo, t_hi)
    print(f"{name}: replay {time.time() - t0:.0f}s", flush=True)
    omega_idx = np.unique(np.array([0, 1, ri, n_ck - 1], np.int64))
    kb = slice(0, keep_b)
    # snapshot omega BEFORE the backward: with B = 1 the reference's streaming_backward replays
    # each window through recompute_alpha, whose ring is a view of ckpts.omega[:, i] (see above),
    # and so overwrites every checkpoint it replays
    omega_snap = ck.omega[kb][:, omega_idx].copy()
    grads, marg = streaming_backward(cum, params, logZ, ck)
    print(f"{name}: backward {time.time() - t0:.0f}s", flush=True)
    segs, scores = streaming_viterbi(cum, params)
    print(f"{name}: viterbi {time.time() - t0:.0f}s", flush=True)
    rows_s = sample_rows(T + 1)          # grad_S rows (boundaries 0..T)
    rows_p = rows_s[rows_s < T]          # per-position rows 0..T-1
    replay_rows = sample_rows(block.shape[1])
    st, en, lb, of = flat_segments(segs)
    out = dict(
        seed=np.int64(seed), T=np.int64(T), K=np.int64(K), C=np.int64(C), B=np.int64(B),
        mode=np.array(mode.value), ragged=np.bool_(ragged), projections=np.bool_(projections),
        keep_b=np.int64(keep_b), delta_arg=np.int64(-1), S_digest=np.array(s_digest(cum.S)),
        logZ=logZ, N=ck.N, delta=np.int64(ck.delta),
        omega_idx=omega_idx, omega=omega_snap,
        replay_i=np.int64(ri), replay_rows=replay_rows, replay=block[kb][:, replay_rows],
        rows_s=rows_s, rows_p=rows_p,
        grad_S=grads.grad_S[kb][:, rows_s], grad_T=grads.grad_T, grad_B=grads.grad_B,
        position_marginals=marg.position_marginals[kb][:, rows_p],
        boundary_posterior=marg.boundary_posterior[kb][:, rows_p],
        expected_segment_count=marg.expected_segment_count,
        # size-independent checksums over the FULL arrays
        grad_S_rowsum_absmax=np.abs(grads.grad_S.sum(axis=(1, 2))).max(keepdims=True),
        pm_total=marg.position_marginals.sum(axis=(1, 2)),
        bp_total=marg.boundary_posterior.sum(axis=1),
        vit_scores=scores, vit_start=st, vit_end=en, vit_label=lb, vit_offsets=of,
    )
    path = os.path.join(HERE, f"golden_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB) in {time.time() - t0:.0f}s", flush=True)


M = P.CenteringMode
JOBS = {
    # BASELINE config 4 at full length, one sequence: ~1.5 h.
    "c4f": lambda: make_full("c4f", 0, 100_000, 1000, 24, 1, M.MEAN),
    # config 5 shape at full length, one sequence: ~2 h.
    "c5f": lambda: make_full("c5f", 0, 20_000, 256, 128, 1, M.MEAN),
    # config 3 exactly (B=32, full T): ~15 min; rows kept for 4 sequences.
    "c3f": lambda: make_full("c3f", 0, 4000, 64, 39, 32, M.MEAN, keep_b=4),
}

def patch_omega(name):
    """Re-take omega of an existing fixture from a fresh forward (fixtures written before the
    snapshot fix above hold the post-backward, overwritten checkpoints when B = 1)."""
    path = os.path.join(HERE, f"golden_{name}.npz")
    z = dict(np.load(path))
    t0 = time.time()
    _, params, cum = equivalence_instance(int(z["seed"]), T=int(z["T"]), K=int(z["K"]), C=int(z["C"]),
                                          B=int(z["B"]), mode=P.CenteringMode(str(z["mode"])))
    assert s_digest(cum.S) == str(z["S_digest"])
    logZ, ck = streaming_forward(cum, params)
    assert np.array_equal(logZ, z["logZ"]) and np.array_equal(ck.N, z["N"])
    z["omega"] = ck.omega[: int(z["keep_b"])][:, z["omega_idx"]].copy()
    np.savez_compressed(path, **z)
    print(f"patched omega of {path} in {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--patch-omega":
        for n in args[1:]:
            patch_omega(n)
    else:
        for n in args or list(JOBS):
            JOBS[n]()
