"""Aggregate an ncu source-page CSV (tools/ncu_head.sh) by head role: stall samples per reason.

    python tools/head_stalls.py gpurun_out/ncu_head_source.csv.gz
Line ranges refer to csrc/scrf_sweep.cuh at the profiled revision; inlined helpers are
attributed by their own source lines (edge_* -> edge, lse5/gemv_exact -> chain).
"""
import collections
import csv
import gzip
import io
import sys

ROLES = [("edge helpers", 740, 849), ("chain (+lse5)", 850, 1123), ("near", 1124, 1235), ("source", 1236, 1334),
         ("edge role", 1335, 1357), ("output role", 1358, 1375), ("head_main", 1376, 1459), ("tails", 1460, 99999)]
rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]), encoding="utf-8")))
hdr = None
curfile = None
agg = collections.defaultdict(lambda: collections.Counter())
lines = collections.defaultdict(lambda: collections.Counter())
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        curfile = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None or not r[0]:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    role = curfile
    if curfile == "scrf_sweep.cuh":
        role = next((n for n, a, b in ROLES if a <= ln <= b), "sweep other")
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and i < len(r) and r[i].isdigit():
            agg[role][h[6:]] += int(r[i])
            lines[(curfile, ln)][h[6:]] += int(r[i])
    if len(r) > 7 and r[7].isdigit():
        agg[role]["#instr"] += int(r[7])
        lines[(curfile, ln)]["#instr"] += int(r[7])
for role, c in sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "#instr")):
    tot = sum(v for k, v in c.items() if k != "#instr")
    top = ", ".join(f"{k} {v}" for k, v in c.most_common(8) if k != "#instr")
    print(f"{role:16s} samples {tot:8d} instr {c['#instr']:10d} | {top}")
print()
for (f, ln), c in sorted(lines.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "#instr"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    if f != "scrf_sweep.cuh" or ln >= 1460:
        continue
    tot = sum(v for k, v in c.items() if k != "#instr")
    top = ", ".join(f"{k} {v}" for k, v in c.most_common(5) if k != "#instr")
    print(f"{f}:{ln:5d} {tot:7d} | {top}")
