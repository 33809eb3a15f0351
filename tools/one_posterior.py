"""One (warm) posterior call at a config, for ncu launch lists: python tools/one_posterior.py c4 [full|sublinear]"""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"])
mode = sys.argv[2] if len(sys.argv) > 2 else "full"
_, params, cum = scrf.equivalence_instance(0, T=cfg["T"], K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
S.device_posterior(prob, memory=mode)
torch.cuda.synchronize()
S.device_posterior(prob, memory=mode)
torch.cuda.synchronize()
