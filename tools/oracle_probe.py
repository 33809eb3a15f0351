"""GPU posterior vs the CPU oracle (oracle/streaming_oracle.py, the reference restated) on random
small shapes with ragged lengths and projections, both precisions, at the tests' tolerances.

    python tools/oracle_probe.py [n_shapes] [seed]
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import parity  # noqa: E402
import streaming_oracle as O  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
worst = {}
for i in range(n):
    C = rng.choice([1, 2, 3, 5, 8, 12])
    K = rng.choice([1, 2, 3, 5, 8, 16, 17, 20, 40])
    B = rng.choice([1, 2, 3])
    T = rng.choice([K + 3, 60, 150, 300])
    proj = rng.random() < 0.5
    _, params, cum = scrf.equivalence_instance(i, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN, ragged=True,
                                               projections=proj)
    zl, exp = O.posterior(cum, params)
    exp = dict(exp)
    exp["logZ"] = zl
    for prec in ("fp32", "fp64"):
        S.set_precision(prec)
        try:
            logZ, grads, marg = scrf.posterior(cum, params)
            errs = parity.compare_posterior(logZ, grads, marg, exp, prec)
            w = max(errs.values())
            worst[prec] = max(worst.get(prec, 0.0), w)
            print(f"C={C} K={K} B={B} T={T} proj={proj} {prec} ok worst {w:.1e}", flush=True)
        except AssertionError as e:
            print(f"C={C} K={K} B={B} T={T} proj={proj} {prec} FAIL {str(e)[:300]}", flush=True)
        finally:
            S.set_precision("fp32")
print("worst per precision:", {k: f"{v:.1e}" for k, v in worst.items()})
