"""Phase timing of the forward sweep (clock64 of CTA 0 / thread 0) for a config.

    python tools/trace_fwd.py c4 [T]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import _lib  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
_, params, cum = scrf.equivalence_instance(0, T=T, K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
prob = scrf.DeviceProblem.from_host(cum, params)
S.device_forward(prob)
buf = torch.zeros((256, 8), dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.scrf_debug_trace(buf.data_ptr())
S.device_forward(prob)
lib.scrf_debug_trace(None)
torch.cuda.synchronize()
tr = buf.cpu().numpy()[50:250].astype(np.float64)
names = ["adv+arm+merge_parts", "k1 term+add+send", "C (bulk)", "wait", "amax", "gamma", "g/ring/book"]
d = np.diff(tr[:, :8], axis=1)
step = np.diff(tr[:, 0])
print("cycles per phase (median over positions 50..250):")
for i, n in enumerate(names):
    print(f"  {n:22s} {np.median(d[:, i]):8.0f}")
print(f"  {'sync+loop (rest)':22s} {np.median(step[:-0 or None] - (tr[1:, 0] - tr[:-1, 0] - 0) + 0) if False else np.median(tr[1:, 0] - tr[:-1, 7]):8.0f}")
print(f"  {'step total':22s} {np.median(step):8.0f}")
