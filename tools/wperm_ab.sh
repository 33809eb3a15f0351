#!/bin/bash
# Head warp placement A/B (SCRF_WPERM: digit i = role of physical warp i; c4 roles:
# 0 chain, 1-4 near groups, 5 source, 6 edge, 7 output). Sweep ms at config 4, T = 8000.
for rep in 1 2; do
for p in 01234567 01237564 01235467 01236574; do
  echo -n "wperm $p: "; SCRF_WPERM=$p python tools/time_cfg.py c4 ${1:-8000} 3 2>&1 | tail -1
done
done
