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
buf = torch.zeros((512, 16), dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.scrf_debug_trace(buf.data_ptr())
S.device_forward(prob)
lib.scrf_debug_trace(None)
torch.cuda.synchronize()
trall = buf.cpu().numpy().astype(np.float64)
tr = trall[:256]
tl = trall[256:]
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

if tl[:, 0].any():
    print("tail warp0 (median cycles): step/group", np.median(np.diff(tl[:, 0])))
    for i, n in enumerate(["src wait", "fma", "reduce+send"]):
        print(f"  {n:14s} {np.median(tl[:, i + 1] - tl[:, i]):8.0f}")
    # near group 0 handles even p; near tr[5..6] = tail wait
    ev = nr[::2]
    print("near tail wait (median):", np.median(ev[:, 6] - ev[:, 5]), " ring write time - tail src arrival")
    # align: tail target u (row u-64) src arrival tl[:,2]; near sends source q at iteration q+4 (tr[7] of row q+4-64)
    ks = 11
    # near row index for iteration p = row p-64; source q sent at iteration q+4; tail target u uses source u-ks
    lat = []
    for r in range(0, 256):
        u = r + 64; q = u - ks; pr = q + 4 - 64
        if 0 <= pr < 256 and nr[pr, 7] > 0 and tl[r, 2] > 0:
            lat.append(tl[r, 2] - nr[pr, 7])
    if lat: print("source send -> tail wakeup (median cycles):", np.median(lat))
    lat = []
    for r in range(0, 256):
        if nr[r, 6] > 0 and tl[r, 3] > 0:
            lat.append(nr[r, 6] - tl[r, 3])
    if lat: print("tail lse done (warp0) -> near wakeup (median):", np.median(lat))
