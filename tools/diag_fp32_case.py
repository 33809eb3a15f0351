import os, sys
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import streaming_oracle as O
import paper_2604_18780_b200 as scrf
from paper_2604_18780_b200 import streaming as S
import random
rng = random.Random(23)
for i in range(40):
    C = rng.choice([1, 2, 3, 5, 8, 12]); K = rng.choice([1, 2, 3, 5, 8, 16, 17, 20, 40]); B = rng.choice([1, 2, 3])
    T = rng.choice([K + 3, 60, 150, 300]); proj = rng.random() < 0.5
    if (C, K, B, T, proj) != (3, 16, 1, 300, True):
        continue
    _, params, cum = scrf.equivalence_instance(i, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN, ragged=True, projections=proj)
    zl, exp = O.posterior(cum, params)
    S.set_precision("fp32")
    logZ, grads, marg = scrf.posterior(cum, params)
    L = int(cum.lengths[0])
    for name, got, want in (("pos", marg.position_marginals, exp["position_marginals"]), ("gS", grads.grad_S, exp["grad_S"]),
                            ("bnd", marg.boundary_posterior, exp["boundary_posterior"])):
        d = np.abs(got - want)
        idx = np.unravel_index(np.argmax(d), d.shape)
        print(name, "max", d.max(), "at", idx, "L", L, "T", T, "value", want[idx])
    d = np.abs(marg.position_marginals - exp["position_marginals"])[0].max(-1)
    print("pos err by position (every 25):", np.round(d[::25] * 1e6, 2).tolist())
