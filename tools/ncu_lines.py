"""Summarise an ncu report per CUDA source line: instructions executed and stall samples.

    python tools/ncu_lines.py report.ncu-rep [kernel-index] [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-id", f"::regex:.*:{kidx + 1}"], capture_output=True, text=True).stdout
if not out.strip():
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = collections.defaultdict(lambda: [0, 0, ""])
curfile, curline, cursrc = None, None, ""
fn_seen = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        curfile = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn_seen += 1
        continue
    if r[0] == "Line No":
        continue
    if r[0]:
        try:
            curline = (curfile, int(r[0]))
            cursrc = r[1]
        except ValueError:
            pass
    if len(r) > 7 and r[2]:
        try:
            agg[curline][0] += int(r[7] or 0)
            agg[curline][1] += int(r[4] or 0)
            agg[curline][2] = cursrc
        except ValueError:
            pass
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {ti}  total stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"stall {v[1] / ts * 100:5.1f}%  instr {v[0] / ti * 100:5.1f}%  {k[0]}:{k[1]}  {v[2].strip()[:90]}")
