#!/bin/bash
# Head-CTA stall attribution: one ncu --set full capture of the c4 sweep at T = 8000 with source
# correlation; the per-line source page (with stall-reason columns) and the raw page are
# exported for offline aggregation by role (tools/head_stalls.py).
mkdir -p gpurun_out
T=${1:-8000}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o /tmp/ncu_head -f \
  python tools/time_cfg.py c4 $T 1 > gpurun_out/ncu_head.log 2>&1
ncu -i /tmp/ncu_head.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/ncu_head_source.csv.gz
ncu -i /tmp/ncu_head.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/ncu_head_raw.csv.gz
ls -la gpurun_out/ncu_head*
