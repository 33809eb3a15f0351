#!/bin/bash
# Sweep A/B across library builds on full-length c4 (tools/e2e_breakdown.py: posterior() wall,
# MODE 0 and MODE 3-open sweeps): libscrf_base.so (previous build) vs the current libscrf.so
echo "base:"; SCRF_LIB=$PWD/paper_2604_18780_b200/libscrf_base.so timeout 300 python tools/e2e_breakdown.py 2>&1 | grep -v Warn
echo "current:"; timeout 300 python tools/e2e_breakdown.py 2>&1 | grep -v Warn
