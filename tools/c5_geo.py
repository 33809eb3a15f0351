"""c5 fwd+bwd device time under geometry overrides (env passed in): python tools/c5_geo.py"""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
_, params, cum = scrf.equivalence_instance(0, T=c["T"], K=c["K"], C=c["C"], B=c["B"], mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
for _ in range(2):
    r = S.device_posterior(prob, memory="full")
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    r = S.device_posterior(prob, memory="full")
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print({k: v for k, v in os.environ.items() if k.startswith("SCRF_")}, f"{ms:.2f} ms {c['B'] * c['T'] / ms / 1e3:.2f} M pos/s",
      float(r[0].logZ[0]))
