"""Wall-clock phases of the numpy posterior API at config 4 (host staging, device, copies back)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

cfg = CONFIGS["c4"]
_, params, cum = scrf.equivalence_instance(0, T=cfg["T"], K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
for it in range(4):
    t = [time.perf_counter()]
    S._check_labels(cum, params)
    t.append(time.perf_counter())
    prob = S.DeviceProblem.from_host(cum, params)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    fwd, bw = S.device_posterior(prob)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    S._raise_if_dead(fwd)
    g = S._grads_to_host(bw)
    m = S._marg_to_host(bw, cum)
    t.append(time.perf_counter())
    r = scrf.posterior(cum, params)
    t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"iter {it}: check {d[0]:.1f} ms, H2D {d[1]:.1f}, device {d[2]:.1f}, D2H {d[3]:.1f}; full posterior() {d[4]:.1f} ms")
