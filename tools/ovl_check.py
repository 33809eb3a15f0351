"""Overlapped full-mode posterior passes: timing and equivalence at a BASELINE config.

SCRF_OVERLAP=1 (windows concurrent with the sweeps), 0 (the same windows after the sweeps) and
-1 (one pass after the sweeps, the pre-overlap path). 1 and 0 must agree bit for bit; -1 differs
by rounding only (log Z reference of the masses).

    python tools/ovl_check.py [config] [window sizes...]
"""
import json
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
sizes = [int(x) for x in sys.argv[2:]] or [8192]
cfg = dict(CONFIGS[name])
B, T, K, C = cfg["B"], cfg["T"], cfg["K"], cfg["C"]
_, params, cum = scrf.equivalence_instance(0, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN)
prob = S.DeviceProblem.from_host(cum, params)
torch.cuda.synchronize()


lib = scrf._lib.load()


def run(mode, ws, n=4):
    os.environ["SCRF_OVERLAP"] = str(mode)
    os.environ["SCRF_OVL_WS"] = str(ws)
    for _ in range(2):
        r = S.device_posterior(prob, memory="full")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sw = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for x, y in sw:  # create the underlying events (lazily made on first record)
        x.record()
        y.record()
    a.record()
    for i in range(n):
        lib.scrf_profile_events(sw[i][0].cuda_event, sw[i][1].cuda_event)
        r = S.device_posterior(prob, memory="full")
    b.record()
    lib.scrf_profile_events(None, None)
    torch.cuda.synchronize()
    run.sweep_ms = sum(x.elapsed_time(y) for x, y in sw) / n
    fwd, bw = r
    outs = {"logZ": fwd.logZ, "grad_S": bw.grad_S, "grad_T": bw.grad_T, "grad_B": bw.grad_B,
            "pos": bw.position_marginals, "bnd": bw.boundary_posterior, "cnt": bw.expected_segment_count}
    return a.elapsed_time(b) / n, {k: v.clone() for k, v in outs.items()}


res = {"config": name}
ms_ref, ref = run(-1, 8192)
res["single_pass_ms"] = ms_ref
res["single_pass_sweep_ms"] = run.sweep_ms
for ws in sizes:
    ms1, o1 = run(1, ws)
    sw1 = run.sweep_ms
    ms0, o0 = run(0, ws)
    same = {k: bool(torch.equal(o1[k], o0[k])) for k in o1}
    diff = {k: float(((o1[k] - ref[k]).abs().max() / ref[k].abs().max().clamp(min=1.0)).item()) for k in o1}
    res[str(ws)] = {"overlap_ms": ms1, "overlap_sweep_ms": sw1, "sequential_windows_ms": ms0, "bit_identical_1_vs_0": same,
                    "max_rel_vs_single_pass": diff, "launches": scrf._lib.launches()}
print(json.dumps(res, indent=1))
