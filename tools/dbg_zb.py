import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import golden_io, paper_2604_18780_b200 as scrf
from paper_2604_18780_b200 import streaming as S
for name in ["c1rp", "c2", "c3s", "c4s", "c5s"]:
    params, cum, delta, exp = golden_io.equiv_case(name)
    prob = scrf.DeviceProblem.from_host(cum, params)
    f, b = S.device_posterior(prob, delta)
    zb = S.device_beta_logz(prob, f, b).cpu().numpy()
    print(name, np.abs(zb - exp["logZ"]).max(), np.abs(f.logZ.cpu().numpy() - exp["logZ"]).max(), cum.S.shape)
