"""Phase stamps of the sweep (cluster 0): chain lane 0 and near thread 0, positions 64..319.

    python tools/trace_sweep.py c4 [T] [dirs: fwd|post]
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
buf = torch.zeros((256, 16), dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.scrf_debug_trace(buf.data_ptr())
S.device_forward(prob)
lib.scrf_debug_trace(None)
torch.cuda.synchronize()
tr = buf.cpu().numpy().astype(np.float64)
ch, nr = tr[:, 0:8], tr[:, 8:16]
print("chain (median cycles): step", np.median(np.diff(ch[:, 0])))
names = ["B+lse3", "max+gemv", "publish+arrive"]
for i, n in enumerate(names):
    print(f"  {n:14s} {np.median(ch[:, i + 1] - ch[:, i]):8.0f}")
print("near (median cycles): step", np.median(np.diff(nr[:, 0])))
names = ["sync A", "prep", "ring_lse", "tail+part"]
for i, n in enumerate(names):
    print(f"  {n:14s} {np.median(nr[:, i + 1] - nr[:, i]):8.0f}")
print("near start - chain start (median):", np.median(nr[:, 0] - ch[:, 0]))
