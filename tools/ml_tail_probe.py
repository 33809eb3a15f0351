"""Random shapes that put more than 16 labels on a tail CTA (many sequences, large C), so the sweep
runs the multi-label exp-space tails (tail_loop_blocked_ml): fp32 posterior against the fp64
instantiation of the same kernels (itself pinned to the reference), at the north-star bar 1e-5
in the reference's metric, both sweep directions, ragged lengths, projections on some shapes."""
import os
import random
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import parity  # noqa: E402
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402

rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
worst = 0.0
fails = 0
for i in range(n):
    C = rng.choice([40, 48, 64, 96, 128])
    K = rng.choice([64, 100, 160, 256, 300])
    B = rng.choice([12, 16])
    T = rng.choice([K + 40, 400, 700])
    proj = rng.random() < 0.4
    _, params, cum = scrf.equivalence_instance(i, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN, ragged=True,
                                               projections=proj)
    out = {}
    for prec in ("fp32", "fp64"):
        S.set_precision(prec)
        logZ, grads, marg = scrf.posterior(cum, params)
        out[prec] = dict(logZ=logZ, grad_S=grads.grad_S, grad_T=grads.grad_T, grad_B=grads.grad_B,
                         pos=marg.position_marginals, bnd=marg.boundary_posterior)
    S.set_precision("fp32")
    errs = {"logZ": parity.rel_err(out["fp32"]["logZ"], out["fp64"]["logZ"])}
    for k in ("grad_S", "grad_T", "grad_B", "pos", "bnd"):
        errs[k] = parity.scaled_err(out["fp32"][k], out["fp64"][k])
    w = max(errs.values())
    worst = max(worst, w)
    ok = w <= 1e-5
    fails += 0 if ok else 1
    print(f"C={C} K={K} B={B} T={T} proj={proj} {'ok' if ok else 'FAIL'} worst {w:.1e}", flush=True)
print(f"{n - fails}/{n} within 1e-5, worst {worst:.1e}")
