#!/bin/bash
# A/B of the sweep at config 4 (T = $1): libscrf_base.so (round-2 head) vs the current build.
D=$PWD/paper_2604_18780_b200
for rep in 1 2; do
  echo -n "base: "; SCRF_LIB=$D/libscrf_base.so timeout 120 python tools/time_cfg.py c4 ${1:-8000} 3 2>&1 | tail -1
  echo -n "new:  "; timeout 120 python tools/time_cfg.py c4 ${1:-8000} 3 2>&1 | tail -1
  echo -n "new identity placement:  "; SCRF_WPERM=01234567 timeout 120 python tools/time_cfg.py c4 ${1:-8000} 3 2>&1 | tail -1
done
