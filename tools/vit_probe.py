"""Viterbi on random shapes: head + tails kernel vs the label-sliced kernel (SCRF_VIT_OLD=1),
bit-identical scores and segments; one subprocess per run with a timeout.

    python tools/vit_probe.py C,K,B,T [C,K,B,T ...]
"""
import os
import pickle
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, pickle
sys.path.insert(0, os.environ["ROOT"])
import paper_2604_18780_b200 as scrf
C, K, B, T = (int(v) for v in os.environ["SHAPE"].split(","))
_, params, cum = scrf.equivalence_instance(1, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN, ragged=True)
segs, sc = scrf.decode(cum, params)
sys.stdout.buffer.write(pickle.dumps(([tuple(s) for s in segs], sc.tolist())))
'''
for spec in sys.argv[1:]:
    res = []
    for old in ("0", "1"):
        env = dict(os.environ, ROOT=ROOT, SHAPE=spec, SCRF_VIT_OLD=old if old == "1" else "")
        try:
            r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, timeout=120)
            res.append(pickle.loads(r.stdout) if r.returncode == 0 else ("ERR", r.stderr.decode()[-200:]))
        except subprocess.TimeoutExpired:
            res.append(("TIMEOUT",))
    same = res[0] == res[1] and res[0][0] not in ("ERR", "TIMEOUT")
    print(spec, "identical" if same else f"DIFF/ERR {str(res[0])[:120]} | {str(res[1])[:120]}", flush=True)
