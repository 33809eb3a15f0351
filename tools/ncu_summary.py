"""Summarise an ncu --set full report: key throughput / pipe / memory metrics per kernel, and
write the sweep's DRAM bytes per launch for bench.py.

    python tools/ncu_summary.py report.ncu-rep [out.txt] [--traffic-json profiles/r02_sweep_traffic.json]
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
idx = {h: i for i, h in enumerate(hdr)}
lines = []
traffic = None
for r in data:
    name = r[idx["Kernel Name"]]
    lines.append(name[:90])
    vals = {}
    for w in want:
        if w in idx:
            lines.append(f"  {w} = {r[idx[w]]} {units[idx[w]]}")
            vals[w] = r[idx[w]]
    if "sweep_kernel" in name and traffic is None:
        def num(k):
            v = vals.get(k, "0").replace(",", "")
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[idx[k]], 1)
            return float(v) * mult
        traffic = {"bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
                   "executed": {"xu_pipe_pct": vals.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                                "fma_pipe_pct": vals.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                                "issue_active_pct": vals.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                "warps_active_pct": vals.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                                "source": rep}}
text = "\n".join(lines)
print(text)
if out:
    open(out, "w").write(text + "\n")
if tj and traffic:
    json.dump(traffic, open(tj, "w"), indent=1)
