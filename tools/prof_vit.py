"""One Viterbi decode of a config at reduced T (for ncu captures): python tools/prof_vit.py c4 4000"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
T = int(sys.argv[2])
_, params, cum = scrf.equivalence_instance(0, T=T, K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
S.device_viterbi(prob)
torch.cuda.synchronize()
print("done")
