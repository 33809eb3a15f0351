"""Generate golden vectors by running the REAL reference (`/root/reference/pkg/src/streamcrf`).

Run in the build container only (the GPU box has no /root/reference):

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py small c1   # a subset

Each fixture is an .npz holding the reference's outputs for one instance set:
logZ, checkpoint normalisers, gradients, marginals, Viterbi segments and
scores. Inputs are either stored (small random instances, incl. scalar
boundary folding and every centering mode) or regenerated from
`paper_2604_18780_b200.instances.equivalence_instance`, which is
bit-identical to the reference's generator — an input checksum is stored to
prove it at test time.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from streamcrf import potentials as P  # noqa: E402  (the reference)
from streamcrf.streaming import streaming_backward, streaming_forward, streaming_viterbi  # noqa: E402
from streamcrf.validation import equivalence_instance  # noqa: E402


def s_digest(S: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(S).tobytes()).hexdigest()


def flat_segments(segs):
    starts, ends, labels, offs = [], [], [], [0]
    for seg in segs:
        for s, e, c in seg.segments:
            starts.append(s)
            ends.append(e)
            labels.append(c)
        offs.append(len(starts))
    return (np.array(starts, np.int64), np.array(ends, np.int64),
            np.array(labels, np.int64), np.array(offs, np.int64))


def run_reference(cum, params, delta=None, upstream=None, keep_b=None):
    logZ, ck = streaming_forward(cum, params, delta)
    grads, marg = streaming_backward(cum, params, logZ, ck, upstream)
    segs, scores = streaming_viterbi(cum, params)
    sl = slice(None) if keep_b is None else slice(0, keep_b)
    out = dict(
        logZ=logZ, N=ck.N, delta=np.int64(ck.delta),
        grad_S=grads.grad_S[sl], grad_T=grads.grad_T, grad_B=grads.grad_B,
        position_marginals=marg.position_marginals[sl],
        boundary_posterior=marg.boundary_posterior[sl],
        expected_segment_count=marg.expected_segment_count,
        vit_scores=scores,
    )
    if grads.grad_P_start is not None:
        out["grad_P_start"] = grads.grad_P_start[sl]
        out["grad_P_end"] = grads.grad_P_end[sl]
    st, en, lb, of = flat_segments(segs)
    out.update(vit_start=st, vit_end=en, vit_label=lb, vit_offsets=of)
    return out


def save(name, **arrays):
    path = os.path.join(HERE, f"golden_{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)")


def make_small(n_cases: int = 48):
    """Small random instances covering modes, ragged, projections, scalar pi, deltas."""
    modes = [P.CenteringMode.NONE, P.CenteringMode.MEAN, P.CenteringMode.SHARED_MAX]
    arrays = {}
    for i in range(n_cases):
        rng = np.random.default_rng([20240817, i])
        T = int(rng.integers(1, 41))
        K = int(rng.integers(1, 9))
        C = int(rng.integers(1, 6))
        B = int(rng.integers(1, 4))
        mode = modes[i % 3]
        ragged = B > 1 and i % 2 == 0
        proj = i % 4 == 1
        scal = i % 5 == 2
        em = rng.uniform(-2.0, 2.0, (B, T, C))
        if ragged and T > 1:
            L = rng.integers(1, T + 1, size=B)
            L[rng.integers(0, B)] = T
        else:
            L = np.full(B, T, dtype=np.int64)
        params = P.SemiCRFParams(
            rng.uniform(-1.0, 1.0, (C, C)), rng.uniform(-0.5, 0.5, (K, C)),
            rng.uniform(-1.0, 1.0, C) if scal else None,
            rng.uniform(-1.0, 1.0, C) if scal else None,
        )
        ps = rng.uniform(-0.5, 0.5, (B, T, C)) if proj else None
        pe = rng.uniform(-0.5, 0.5, (B, T, C)) if proj else None
        cum = P.build_scores(P.EmissionBatch(em, L), params, mode, ps, pe)
        delta = (1 if i % 2 else min(3, T)) if i % 3 == 0 else None
        upstream = rng.uniform(-1.0, 2.0, B) if i % 7 == 3 else None
        ref = run_reference(cum, params, delta, upstream)
        pre = f"c{i:03d}_"
        arrays[pre + "emissions"] = em
        arrays[pre + "lengths"] = np.asarray(L, np.int64)
        arrays[pre + "transition"] = params.transition
        arrays[pre + "duration_bias"] = params.duration_bias
        arrays[pre + "mode"] = np.array(mode.value)
        if scal:
            arrays[pre + "pi_start"] = params.pi_start
            arrays[pre + "pi_end"] = params.pi_end
        if proj:
            arrays[pre + "proj_start"] = ps
            arrays[pre + "proj_end"] = pe
        if upstream is not None:
            arrays[pre + "upstream"] = upstream
        arrays[pre + "delta_arg"] = np.int64(-1 if delta is None else delta)
        arrays[pre + "S_digest"] = np.array(s_digest(cum.S))
        for k, v in ref.items():
            arrays[pre + k] = v
    arrays["n_cases"] = np.int64(n_cases)
    save("small", **arrays)


def make_equiv(name, seed, T, K, C, B, mode, ragged=False, projections=False, keep_b=None, delta=None):
    t0 = time.time()
    _, params, cum = equivalence_instance(
        seed, T=T, K=K, C=C, B=B, mode=mode, ragged=ragged, projections=projections
    )
    ref = run_reference(cum, params, delta=delta, keep_b=keep_b)
    meta = dict(seed=np.int64(seed), T=np.int64(T), K=np.int64(K), C=np.int64(C), B=np.int64(B),
                mode=np.array(mode.value), ragged=np.bool_(ragged), projections=np.bool_(projections),
                keep_b=np.int64(-1 if keep_b is None else keep_b),
                delta_arg=np.int64(-1 if delta is None else delta),
                S_digest=np.array(s_digest(cum.S)))
    save(name, **meta, **ref)
    print(f"  {name}: {time.time() - t0:.1f}s")


def make_masked():
    """Min-duration mask (duration_bias[0] = -2e9, at or below the NEG_INF guard) with K = 2:
    position 1 is dead, later even positions are not. The reference's streaming path returns a
    different log Z here than its own dense DP and K=2 fast path because clamp_log fires on
    sentinel arithmetic (streaming.py:150-152, _numerics.py:41-56: RunStats counts the events);
    the fixture holds the dense DP outputs (reference.py:174-283, no clamping) and, for the
    record, the streaming path's log Z and clamp-event count."""
    from streamcrf._numerics import RunStats
    from streamcrf.diagnostics import position_marginals
    from streamcrf.reference import dense_backward_marginals, dense_forward

    _, params, cum = equivalence_instance(5, T=40, K=2, C=3, B=2, mode=P.CenteringMode.MEAN)
    db = params.duration_bias.copy()
    db[0, :] = -2.0e9
    params = P.SemiCRFParams(params.transition, db)
    object.__setattr__(cum, "lengths", np.array([40, 22]))
    msgs = dense_forward(cum, params)
    mu, grads = dense_backward_marginals(cum, params, msgs)
    marg = position_marginals(mu, cum.lengths)
    st = RunStats()
    z_stream, _ = streaming_forward(cum, params, stats=st)
    save("masked", logZ=msgs.logZ, grad_S=grads.grad_S, grad_T=grads.grad_T, grad_B=grads.grad_B,
         position_marginals=marg.position_marginals, boundary_posterior=marg.boundary_posterior,
         expected_segment_count=marg.expected_segment_count, S_digest=np.array(s_digest(cum.S)),
         streaming_logZ=z_stream, streaming_clamp_events=np.int64(st.clamp_events))


def make_train():
    """Acceptance criterion 04 (test_acceptance.py:128-137): the reference's 100-epoch
    gradient-descent training demo (validation.py:344-491) with the dense backend, plus its
    synthetic batch (datagen.generate_imbalanced) so the device path can replay the same run."""
    from streamcrf.datagen import generate_imbalanced
    from streamcrf.validation import DEFAULT_TRAIN_CONFIG, training_convergence_demo

    cfg = dict(DEFAULT_TRAIN_CONFIG)
    B, T, C, K = cfg["B"], cfg["T"], cfg["C"], cfg["K"]
    seqs, golds = [], []
    for b in range(B):
        batch_b, gold_b = generate_imbalanced(T, C, (1.0 / C,) * C, 1.0, seed=[cfg["seed"], b], max_duration=K)
        seqs.append(batch_b.emissions[0])
        golds.append(np.array(gold_b.segments, np.int64))
    t0 = time.time()
    rep = training_convergence_demo(epochs=100, backends=("dense",))
    print(f"  train: {time.time() - t0:.1f}s final {rep['backends']['dense']['final']}")
    arrays = dict(B=np.int64(B), T=np.int64(T), C=np.int64(C), K=np.int64(K), lr=np.float64(cfg["lr"]),
                  emissions=np.stack(seqs), dense_curve=np.array(rep["backends"]["dense"]["curve"]))
    for b, g in enumerate(golds):
        arrays[f"gold_{b}"] = g
    save("train", **arrays)


def make_io():
    """The reference's serialisers (potentials.py:467-552) on a ragged instance with
    projections: emissions CSV / JSON, params JSON, segmentation JSON (for byte-level checks of
    this package's writers and readers)."""
    import json as _json

    batch, params, cum = equivalence_instance(3, T=13, K=4, C=3, B=3, ragged=True, projections=True)
    P.save_emissions_csv(batch, os.path.join(HERE, "io_emissions.csv"))
    P.save_emissions_json(batch, os.path.join(HERE, "io_emissions.json"))
    params = P.SemiCRFParams(params.transition, params.duration_bias, np.arange(3) * 0.25, -np.arange(3) * 0.5)
    P.save_params_json(params, os.path.join(HERE, "io_params.json"))
    segs = [P.Segmentation(((0, 2, 1), (2, 3, 0))), P.Segmentation(((0, 1, 2),))]
    with open(os.path.join(HERE, "io_segments.json"), "w") as fh:
        _json.dump(P.segmentations_to_json(segs), fh)
    print("wrote io_* fixtures")


M = P.CenteringMode
JOBS = {
    "masked": make_masked,
    "io": make_io,
    "train": make_train,
    "small": lambda: make_small(),
    # c1 exactly as BASELINE.json config 1 (MEAN centering), plus ragged+projections.
    "c1": lambda: make_equiv("c1", 0, 256, 8, 4, 4, M.MEAN),
    "c1rp": lambda: make_equiv("c1rp", 0, 256, 8, 4, 4, M.MEAN, ragged=True, projections=True),
    # c2 exactly as config 2; per-sequence arrays kept for the first 8 sequences.
    "c2": lambda: make_equiv("c2", 0, 512, 16, 9, 64, M.MEAN, keep_b=8),
    # c3/c4/c5 shapes (same K, C) at reduced T so the fp64 reference finishes.
    "c3s": lambda: make_equiv("c3s", 0, 300, 64, 39, 2, M.MEAN, ragged=True),
    "c4s": lambda: make_equiv("c4s", 0, 1100, 1000, 24, 1, M.MEAN, delta=100),
    "c5s": lambda: make_equiv("c5s", 0, 300, 256, 128, 1, M.MEAN),
    "shmax": lambda: make_equiv("shmax", 1, 400, 32, 6, 3, M.SHARED_MAX, ragged=True, projections=True),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(JOBS)
    for n in names:
        JOBS[n]()
