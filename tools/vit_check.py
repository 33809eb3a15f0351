"""Viterbi: compare the current kernel against SCRF_VIT_OLD=1 (bit-identical) and time both.

    python tools/vit_check.py c4 20000 [old]
"""
import os
import pickle
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 3 and sys.argv[3] == "child":
    import torch

    import paper_2604_18780_b200 as scrf
    from paper_2604_18780_b200 import streaming as S
    from paper_2604_18780_b200.instances import CONFIGS

    cfg = CONFIGS[sys.argv[1]]
    T = int(sys.argv[2])
    _, params, cum = scrf.equivalence_instance(0, T=T, K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
    prob = S.DeviceProblem.from_host(cum, params)
    v = S.device_viterbi(prob)
    torch.cuda.synchronize()
    dt = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        v = S.device_viterbi(prob)
        torch.cuda.synchronize()
        dt = min(dt, time.perf_counter() - t0)
    segs = S._segments_to_host(v)
    sc = v.score.cpu().numpy()
    sys.stdout.buffer.write(pickle.dumps((dt, sc, [s.segments if hasattr(s, "segments") else tuple(s) for s in segs])))
    sys.exit(0)

cfg, T = sys.argv[1], sys.argv[2]
res = {}
for tag, env in (("new", {}), ("old", {"SCRF_VIT_OLD": "1"})):
    r = subprocess.run([sys.executable, __file__, cfg, T, "child"], env=dict(os.environ, **env), capture_output=True,
                       timeout=600)
    if r.returncode != 0:
        print(tag, "FAILED", r.stderr.decode()[-800:])
        sys.exit(1)
    res[tag] = pickle.loads(r.stdout)
dn, sn, gn = res["new"]
do, so, go = res["old"]
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

B = CONFIGS[cfg]["B"]
same_sc = np.array_equal(sn, so)
same_seg = gn == go
print(f"{cfg} T={T}: new {dn * 1e3:.1f} ms ({B * int(T) / dn / 1e6:.2f} M pos/s), old {do * 1e3:.1f} ms "
      f"({B * int(T) / do / 1e6:.2f} M pos/s); scores identical {same_sc}, segments identical {same_seg}")
