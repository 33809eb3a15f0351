"""Load the committed golden fixtures and rebuild their inputs.

Fixtures come from `tests/golden/make_golden.py` (the real reference run in the
build container). Inputs are rebuilt with this package's input stage, whose
prefix sums must hash to the digest the reference recorded.
"""

from __future__ import annotations

import hashlib
import os

import numpy as np

from paper_2604_18780_b200.instances import equivalence_instance
from paper_2604_18780_b200.potentials import CenteringMode, EmissionBatch, SemiCRFParams, build_scores

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(S):
    return hashlib.sha256(np.ascontiguousarray(S).tobytes()).hexdigest()


def load(name):
    path = os.path.join(GOLDEN, f"golden_{name}.npz")
    if not os.path.exists(path):
        return None
    return dict(np.load(path, allow_pickle=False))


def _outputs(z, pre=""):
    out = {k[len(pre):]: v for k, v in z.items() if k.startswith(pre)}
    offs = out["vit_offsets"]
    segs = []
    for b in range(len(offs) - 1):
        sl = slice(offs[b], offs[b + 1])
        segs.append(tuple(zip(out["vit_start"][sl].tolist(), out["vit_end"][sl].tolist(),
                              out["vit_label"][sl].tolist())))
    out["vit_segments"] = segs
    return out


def small_cases():
    """Yields (case_id, params, cum, delta, upstream, expected) for golden_small."""
    z = load("small")
    if z is None:
        return
    for i in range(int(z["n_cases"])):
        pre = f"c{i:03d}_"
        g = lambda k: z.get(pre + k)  # noqa: E731
        params = SemiCRFParams(g("transition"), g("duration_bias"), g("pi_start"), g("pi_end"))
        cum = build_scores(EmissionBatch(g("emissions"), g("lengths")), params,
                           CenteringMode(str(g("mode"))), g("proj_start"), g("proj_end"))
        assert digest(cum.S) == str(g("S_digest")), f"input stage drifted for case {i}"
        d = int(g("delta_arg"))
        yield i, params, cum, (None if d < 0 else d), g("upstream"), _outputs(z, pre)


def equiv_case(name):
    """(params, cum, delta, expected) for an equivalence-instance fixture, or None."""
    z = load(name)
    if z is None:
        return None
    _, params, cum = equivalence_instance(
        int(z["seed"]), T=int(z["T"]), K=int(z["K"]), C=int(z["C"]), B=int(z["B"]),
        mode=CenteringMode(str(z["mode"])), ragged=bool(z["ragged"]), projections=bool(z["projections"]),
    )
    assert digest(cum.S) == str(z["S_digest"]), f"input stage drifted for {name}"
    d = int(z["delta_arg"])
    return params, cum, (None if d < 0 else d), _outputs(z)
