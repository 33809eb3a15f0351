"""Device time and peak memory of the full and sublinear posterior at a BASELINE config."""
import json
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"])
B, T, K, C = cfg["B"], cfg["T"], cfg["K"], cfg["C"]
_, params, cum = scrf.equivalence_instance(0, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
torch.cuda.synchronize()
out = {"config": cfg}
for mode in ("full", "sublinear"):
    for _ in range(2):
        S.device_posterior(prob, memory=mode)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 3
    for _ in range(n):
        r = S.device_posterior(prob, memory=mode)
        del r
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    out[mode] = {"ms": ms, "positions_per_s": B * T / ms * 1e3,
                 "peak_bytes_above_inputs": torch.cuda.max_memory_allocated() - base,
                 "launches": scrf._lib.launches()}
print(json.dumps(out))
