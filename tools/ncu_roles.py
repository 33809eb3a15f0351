"""Per-role stall breakdown of the sweep kernel from an ncu source capture.

SASS rows are sorted by address; each row belongs to the role function (head_chain, head_near,
...) whose source lines own the nearest preceding attributed row, so inlined helpers (mbarrier
waits, shuffles) count towards their caller.

    python tools/ncu_roles.py report.ncu-rep [detail-role]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
detail = sys.argv[2] if len(sys.argv) > 2 else None
src_path = "paper_2604_18780_b200/csrc/scrf_sweep.cuh"
code = open(src_path).read().split("\n")
ROLES = ["head_chain", "head_near", "head_src", "head_edge_role", "edge_batch", "tail_loop_blocked", "tail_loop",
         "tail_main", "head_main", "gemv_exact", "lse5", "ring_lse", "ring_exact"]
ranges = []
for name in ROLES:
    for i, l in enumerate(code):
        if re.search(r"\b" + name + r"\(", l) and ("__device__" in l or "__device__" in code[i - 1]):
            depth, started = 0, False
            for j in range(i, len(code)):
                depth += code[j].count("{") - code[j].count("}")
                if "{" in code[j]:
                    started = True
                if started and depth == 0:
                    ranges.append((i + 1, j + 1, name))
                    break
            break


def owner(line):
    best = None
    for lo, hi, n in ranges:
        if lo <= line <= hi and (best is None or hi - lo < best[1] - best[0]):
            best = (lo, hi, n)
    return best[2] if best else None


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, cur, f = None, None, None
sass = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = ["Line No", "LSource", "Address", "Source"] + r[4:]
        continue
    if r[0] == "Function Name" or len(r) < 4:
        continue
    if r[0].isdigit():
        cur = (f, int(r[0]), r[1])
        continue
    if r[2].startswith("0x") and cur:
        d = dict(zip(hdr, r))
        st = collections.Counter({k[6:]: int(v) for k, v in d.items()
                                  if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v)})
        ex = d.get("Instructions Executed", "0")
        sass.append((int(r[2], 16), cur, st, int(ex) if ex.isdigit() else 0, r[3]))
sass.sort()
agg = collections.defaultdict(collections.Counter)
inst = collections.Counter()
own = None
lines = collections.defaultdict(collections.Counter)
for addr, (fi, ln, sr), st, ex, sa in sass:
    if fi == "scrf_sweep.cuh":
        o = owner(ln)
        if o:
            own = o
    key = own or "?"
    agg[key] += st
    inst[key] += ex
    if detail and key == detail:
        lines[(fi, ln, sr[:60])] += st
for k, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
    tot = sum(c.values())
    print(f"{k:20s} samples {tot:7d} instr {inst[k]:11d}  " + ", ".join(f"{n} {v / tot:.0%}" for n, v in c.most_common(6)))
if detail:
    for k, c in sorted(lines.items(), key=lambda kv: -sum(kv[1].values()))[:40]:
        print(f"  {k[0]}:{k[1]:5d} {sum(c.values()):6d} {k[2]:60s} {c.most_common(3)}")
