"""Sublinear-memory posterior device time at a config, SCRF_SPARSE_OVL on / off, and equality."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
_, params, cum = scrf.equivalence_instance(0, T=c["T"], K=c["K"], C=c["C"], B=c["B"], mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
res = {}
for mode in ("1", "0", "1", "0"):
    os.environ["SCRF_SPARSE_OVL"] = mode
    for _ in range(2):
        r = S.device_posterior(prob, memory="sublinear")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        r = S.device_posterior(prob, memory="sublinear")
    b.record()
    torch.cuda.synchronize()
    res[mode] = r
    print("SCRF_SPARSE_OVL", mode, f"{a.elapsed_time(b) / 3:.2f} ms", flush=True)
f1, b1 = res["1"]
f0, b0 = res["0"]
for k in ("grad_S", "grad_T", "grad_B", "position_marginals", "boundary_posterior"):
    print(k, "bit-identical" if torch.equal(getattr(b1, k), getattr(b0, k)) else "DIFFERENT")
