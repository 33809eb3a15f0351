"""Per-SASS stall breakdown for a source-line range of one file in an ncu report.

    python tools/ncu_sass_range.py report.ncu-rep scrf_sweep.cuh 745 826 [min_samples]
"""
import csv
import io
import subprocess
import sys

rep, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
mins = int(sys.argv[5]) if len(sys.argv) > 5 else 5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
cur = None
tot = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        curfile = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = ["Line No", "LSource", "Address", "Source"] + r[4:]
        continue
    if r[0] == "Function Name" or len(r) < 4:
        continue
    if r[0].isdigit():
        cur = (curfile, int(r[0]), r[1])
        continue
    if r[2].startswith("0x"):
        if cur and cur[0] == fname and lo <= cur[1] <= hi:
            d = dict(zip(hdr, r))
            try:
                smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            except ValueError:
                smp = 0
            tot += smp
            if smp >= mins:
                st = sorted(((int(v or 0), k[6:]) for k, v in d.items()
                             if k.startswith("stall_") and "Not Issued" not in k and (v or "0").isdigit()), reverse=True)[:3]
                print(f"{cur[1]:5d} {smp:6d} {d.get('Source','')[:60]:60s} {st}")
print("total samples in range", tot)
