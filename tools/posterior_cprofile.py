"""Host-side profile of one numpy posterior() call at config 4 (cProfile, after warm-up)."""
import cProfile
import os
import pstats
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

c = CONFIGS["c4"]
_, params, cum = scrf.equivalence_instance(0, T=c["T"], K=c["K"], C=c["C"], B=c["B"], mode=scrf.CenteringMode.MEAN)
for _ in range(3):
    scrf.posterior(cum, params)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
scrf.posterior(cum, params)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
