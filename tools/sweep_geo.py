"""Time device_forward / device_backward on a config for a grid of launch geometries.

    python tools/sweep_geo.py c4 "G=8,TPL=32" "G=8,TPL=64" ...

Each setting runs in a fresh subprocess (the geometry is read from SCRF_G / SCRF_TPL).
Prints one JSON line per setting with forward and backward kernel ms (CUDA events).
"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2604_18780_b200 as scrf
from paper_2604_18780_b200 import streaming as S
from paper_2604_18780_b200.instances import CONFIGS
cfg = CONFIGS[os.environ["CFG"]]
T = int(os.environ.get("TOVR", cfg["T"]))
_, params, cum = scrf.equivalence_instance(0, T=T, K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
prob = scrf.DeviceProblem.from_host(cum, params)
bwd = os.environ.get("BWD", "1") == "1"
def run():
    f = S.device_forward(prob)
    b = S.device_backward(prob, f) if bwd else None
    return f, b
run(); torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record(); f = S.device_forward(prob); e[1].record()
if bwd: S.device_backward(prob, f)
e[2].record(); torch.cuda.synchronize()
fm = e[0].elapsed_time(e[1]); bm = e[1].elapsed_time(e[2])
print(json.dumps({"setting": os.environ["SETTING"], "T": T, "fwd_ms": fm, "bwd_ms": bm,
                  "fwd_ns_per_pos": fm * 1e6 / T, "bwd_ns_per_pos": bm * 1e6 / T}), flush=True)
'''

cfg = sys.argv[1]
for setting in sys.argv[2:]:
    env = dict(os.environ, ROOT=ROOT, CFG=cfg, SETTING=setting)
    for kv in setting.split(","):
        k, v = kv.split("=")
        env[{"G": "SCRF_G", "TPL": "SCRF_TPL"}.get(k, k)] = v
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    out = r.stdout.strip().splitlines()
    print(out[-1] if out else json.dumps({"setting": setting, "error": r.stderr[-400:]}), flush=True)
