"""Time the fused posterior (sweep kernel + whole step) of a config at a given T, no parity.

    python tools/time_cfg.py c4 8000 [repeats]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import _lib  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
T = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
_, params, cum = scrf.equivalence_instance(0, T=T, K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
prob = scrf.DeviceProblem.from_host(cum, params)
f, b = S.device_posterior(prob)
torch.cuda.synchronize()
lib = _lib.load()
best = None
for _ in range(reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for ev in e:
        ev.record()
    torch.cuda.synchronize()
    lib.scrf_profile_events(e[1].cuda_event, e[2].cuda_event)
    e[0].record()
    f, b = S.device_posterior(prob)
    e[3].record()
    lib.scrf_profile_events(None, None)
    torch.cuda.synchronize()
    sweep, tot = e[1].elapsed_time(e[2]), e[0].elapsed_time(e[3])
    if best is None or sweep < best[0]:
        best = (sweep, tot)
sweep, tot = best
zb = S.device_beta_logz(prob, f, b)
print(f"{sys.argv[1]} T={T} {os.environ.get('TAG', '')}: sweep {sweep:.2f} ms ({sweep * 1e6 / T:.0f} ns/pos), "
      f"step {tot:.2f} ms, {cfg['B'] * T / tot * 1e3 / 1e6:.2f} M pos/s, |logZ a-b| {float((f.logZ - zb).abs().max()):.1e}",
      flush=True)
