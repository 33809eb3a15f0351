"""Full vs sublinear posterior on the golden small cases: per-case errors and where they sit."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import golden_io  # noqa: E402
import parity  # noqa: E402
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
S.set_precision(prec)
for i, params, cum, delta, up, exp in golden_io.small_cases():
    res = {}
    for mode in ("full", "sublinear"):
        logZ, grads, marg = scrf.posterior(cum, params, delta, up, memory=mode)
        res[mode] = dict(logZ=logZ, grad_S=grads.grad_S, pm=marg.position_marginals, bp=marg.boundary_posterior,
                         gT=grads.grad_T, gB=grads.grad_B)
    errs = {k: parity.scaled_err(res["sublinear"][k], res["full"][k]) for k in res["full"]}
    worst = max(errs.values())
    B, T1, C = cum.S.shape
    d = delta if delta is not None else S.choose_checkpoint_interval(T1 - 1, params.max_duration)
    if worst > 1e-5:
        dd = np.abs(res["sublinear"]["pm"] - res["full"]["pm"]).max(-1)
        loc = np.unravel_index(np.argmax(dd), dd.shape)
        print(f"case {i}: B={B} T={T1-1} K={params.max_duration} C={C} delta={d} L={list(cum.lengths)} "
              f"proj={cum.proj_start is not None} worst={worst:.2e} errs={ {k: f'{v:.1e}' for k, v in errs.items()} } "
              f"pm-err at {loc}; row errs {np.round(dd[loc[0]] * 1e4, 1).tolist()}")
print("done")
