#!/bin/bash
# Sweep A/B on full-length c4 across library builds: the current libscrf.so and any
# paper_2604_18780_b200/libscrf_v*.so experiment variants (tools/e2e_breakdown.py: posterior()
# wall, MODE 0 and MODE 3-open sweep times).
D=$PWD/paper_2604_18780_b200
for lib in $D/libscrf.so $D/libscrf_v*.so; do
  echo "$(basename $lib):"; SCRF_LIB=$lib timeout 300 python tools/e2e_breakdown.py 2>&1 | grep -v "Warn\|^wall 2"
done
