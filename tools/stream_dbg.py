"""Streamed-input debugging: posterior() at a few shapes, wall time and gate status."""
import os
import sys
import time

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402

for (B, T, K, C) in [(2, 100000, 64, 24), (2, 100000, 1000, 24), (8, 100000, 64, 24), (8, 100000, 1000, 24)]:
    _, params, cum = scrf.equivalence_instance(0, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN)
    for rep in range(2):
        t0 = time.perf_counter()
        try:
            scrf.posterior(cum, params, memory="full")
            st = "ok"
        except RuntimeError as e:
            st = str(e)
        print(B, T, K, C, rep, f"{time.perf_counter() - t0:.3f}s", st, flush=True)
