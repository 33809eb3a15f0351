"""fp32 vs fp64 instantiation at a full BASELINE config (default c4): every output in the
reference metric max|d|/max(1,|ref|), the error profile along t, and device time of both.

    python tools/c4_precision.py [--config c4] [--B 8] [--out gpurun_out/prec.json]
"""
import argparse
import json
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--B", type=int, default=0)
ap.add_argument("--T", type=int, default=0)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--precs", default="fp32,fp64")
ap.add_argument("--out", default="")
args = ap.parse_args()
cfg = dict(CONFIGS[args.config])
if args.B:
    cfg["B"] = args.B
if args.T:
    cfg["T"] = args.T
B, T, K, C = cfg["B"], cfg["T"], cfg["K"], cfg["C"]
_, params, cum = scrf.equivalence_instance(args.seed, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
res = {}
outs = {}
for prec in args.precs.split(","):
    fwd, bw = S.device_posterior(prob, precision=prec)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fwd, bw = S.device_posterior(prob, precision=prec)
    b.record()
    torch.cuda.synchronize()
    res[prec + "_ms"] = a.elapsed_time(b)
    outs[prec] = {
        "logZ": fwd.logZ.cpu().numpy(),
        "logZb": S.device_beta_logz(prob, fwd, bw).cpu().numpy(),
        "grad_S": bw.grad_S.cpu().numpy(), "grad_T": bw.grad_T.cpu().numpy(), "grad_B": bw.grad_B.cpu().numpy(),
        "position_marginals": bw.position_marginals.cpu().numpy(),
        "boundary_posterior": bw.boundary_posterior.cpu().numpy(),
        "expected_segment_count": bw.expected_segment_count.cpu().numpy(),
    }
    del fwd, bw
precs = args.precs.split(",")
if len(precs) >= 2:
    g, w = outs[precs[0]], outs[precs[1]]
    errs = {}
    for k in g:
        d = np.abs(g[k] - w[k])
        if k in ("logZ", "logZb"):
            errs[k] = float(np.max(d / np.maximum(1.0, np.abs(w[k]))))
        else:
            errs[k] = float(d.max() / max(1.0, np.abs(w[k]).max()))
    res["errors"] = errs
    # error profile along t (max over b, c) in 20 bins
    d = np.abs(g["position_marginals"] - w["position_marginals"]).max(axis=(0, 2))
    res["pm_err_profile"] = [float(x.max()) for x in np.array_split(d, 20)]
    d = np.abs(g["boundary_posterior"] - w["boundary_posterior"]).max(axis=0)
    res["bp_err_profile"] = [float(x.max()) for x in np.array_split(d, 20)]
    # uniform (log) error of the alpha+beta frame at each boundary: sum_c E / sum_c E_ref
    res["pm_rowsum_dev"] = float(np.abs(g["position_marginals"].sum(-1) - 1.0).max())
    res["pm_rowsum_dev_ref"] = float(np.abs(w["position_marginals"].sum(-1) - 1.0).max())
res["config"] = dict(cfg, seed=args.seed)
print(json.dumps(res, indent=1))
if args.out:
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)

# drift of the uniform (alpha+beta frame) error: eps_t = bp32/bp64 - 1 (boundary mass = sum_c A)
if len(precs) >= 2:
    g, w = outs[precs[0]], outs[precs[1]]
    bp32, bp64 = g["boundary_posterior"], w["boundary_posterior"]
    ok = bp64 > 1e-3
    eps = np.where(ok, bp32 / np.where(ok, bp64, 1.0) - 1.0, np.nan)
    drift = {"eps_absmax": float(np.nanmax(np.abs(eps)))}
    for lag in (1, 16, 64, 256, 1024, 4096):
        if eps.shape[1] > 2 * lag:
            d = eps[:, lag:] - eps[:, :-lag]
            drift[f"lag{lag}_absmax"] = float(np.nanmax(np.abs(d)))
            drift[f"lag{lag}_std"] = float(np.nanstd(d))
    drift["eps_profile_b0"] = [float(np.nanmean(x)) for x in np.array_split(eps[0], 20)]
    print(json.dumps(drift, indent=1))
    if args.out:
        with open(args.out.replace(".json", "_drift.json"), "w") as fh:
            json.dump(drift, fh, indent=1)
