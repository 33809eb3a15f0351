"""Quick GPU parity + timing check of the fused posterior against the golden fixtures.

    python tools/quick_parity.py [fp32|fp64] [timing-config T]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_io  # noqa: E402
import parity  # noqa: E402
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
S.set_precision(prec)
worst = {}
fails = 0
for i, params, cum, delta, up, exp in golden_io.small_cases():
    logZ, grads, marg = scrf.posterior(cum, params, delta, up)
    try:
        errs = parity.compare_posterior(logZ, grads, marg, exp, prec)
    except AssertionError as e:
        fails += 1
        if fails <= 3:
            print("small case", i, "FAIL", str(e)[:600])
        continue
    for k, v in errs.items():
        worst[k] = max(worst.get(k, 0.0), v)
print("small cases worst:", {k: f"{v:.2e}" for k, v in worst.items()}, "fails", fails, flush=True)
for name in ["c1", "c1rp", "shmax", "c2", "c3s", "c4s", "c5s"]:
    case = golden_io.equiv_case(name)
    if case is None:
        continue
    params, cum, delta, exp = case
    try:
        logZ, grads, marg = scrf.posterior(cum, params, delta)
        errs = parity.compare_posterior(logZ, grads, marg, exp, prec)
        print(name, "ok", {k: f"{v:.1e}" for k, v in errs.items()}, flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "FAIL", str(e)[:800], flush=True)

if len(sys.argv) > 3:
    cfg = CONFIGS[sys.argv[2]]
    T = int(sys.argv[3])
    _, params, cum = scrf.equivalence_instance(0, T=T, K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
    prob = scrf.DeviceProblem.from_host(cum, params)
    S.device_posterior(prob)
    torch.cuda.synchronize()
    lib = scrf._lib.load() if hasattr(scrf, "_lib") else None
    from paper_2604_18780_b200 import _lib
    lib = _lib.load()
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
    sweep = e[1].elapsed_time(e[2])
    tot = e[0].elapsed_time(e[3])
    print(f"{sys.argv[2]} T={T}: sweep {sweep:.2f} ms ({sweep*1e6/T:.0f} ns/pos), step {tot:.2f} ms, "
          f"{cfg['B']*T/tot*1e3/1e6:.2f} M pos/s", flush=True)
    zb = S.device_beta_logz(prob, f, b)
    print("logZ alpha vs beta:", float((f.logZ - zb).abs().max()), flush=True)
