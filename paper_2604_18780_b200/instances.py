"""Seeded synthetic semi-CRF instances (the reference's measurement inputs).

`equivalence_instance` restates `validation.equivalence_instance`
(`pkg/src/streamcrf/validation.py:180-212`): the RNG key
`[seed, T, K, C, B, ragged, projections, mode_index]` and the draw order
(emissions U[-2,2] -> ragged lengths -> transition U[-1,1] -> duration bias
U[-0.5,0.5] -> projections U[-0.5,0.5]) are kept, so the same arguments give
bit-identical arrays to the reference's. BASELINE.json's configs are defined
on these instances.
"""

from __future__ import annotations

import numpy as np

from .potentials import CenteringMode, EmissionBatch, SemiCRFParams, build_scores

_MODES = (CenteringMode.NONE, CenteringMode.MEAN, CenteringMode.SHARED_MAX)

# BASELINE.json "configs" (B, T, K, C); c1 is the reference's CPU-runnable case.
CONFIGS = {
    "c1": dict(B=4, T=256, K=8, C=4),
    "c2": dict(B=64, T=512, K=16, C=9),
    "c3": dict(B=32, T=4000, K=64, C=39),
    "c4": dict(B=8, T=100_000, K=1000, C=24),
    "c5": dict(B=16, T=20_000, K=256, C=128),
}


def equivalence_instance(
    seed: int,
    *,
    T: int,
    K: int,
    C: int,
    B: int = 1,
    mode: CenteringMode = CenteringMode.NONE,
    ragged: bool = False,
    projections: bool = False,
):
    """Returns (EmissionBatch, SemiCRFParams, CumulativeScores)."""
    rng = np.random.default_rng([seed, T, K, C, B, int(ragged), int(projections), _MODES.index(mode)])
    emissions = rng.uniform(-2.0, 2.0, (B, T, C))
    lengths = np.full(B, T, dtype=np.int64)
    if ragged and B > 1:
        lengths = rng.integers(1, T + 1, size=B)
        lengths[0] = T
    batch = EmissionBatch(emissions, lengths)
    params = SemiCRFParams(rng.uniform(-1.0, 1.0, (C, C)), rng.uniform(-0.5, 0.5, (K, C)))
    ps = pe = None
    if projections:
        ps = rng.uniform(-0.5, 0.5, (B, T, C))
        pe = rng.uniform(-0.5, 0.5, (B, T, C))
    cum = build_scores(batch, params, mode, proj_start=ps, proj_end=pe)
    return batch, params, cum
