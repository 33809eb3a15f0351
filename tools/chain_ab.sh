#!/bin/bash
# A/B of the sweep at config 4 (T = $1) across library builds in paper_2604_18780_b200/
# (libscrf_base.so = the previous build, libscrf_v*.so = experiment variants).
D=$PWD/paper_2604_18780_b200
for rep in 1 2; do
  for v in base v1 v2 v3; do
    [ -f $D/libscrf_$v.so ] || continue
    echo -n "$v: "; SCRF_LIB=$D/libscrf_$v.so timeout 120 python tools/time_cfg.py c4 ${1:-8000} 3 2>&1 | tail -1
  done
done
