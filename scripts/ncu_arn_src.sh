#!/bin/bash
# Source-level ncu of one mid-solve Arnoldi launch at a config (SASS + stall samples as CSV).
set -u
O=gpurun_out/${1:-arnsrc}; CFG=${2:-2d256}; SKIP=${3:-60}; mkdir -p $O
CMD="python scripts/one_solve.py $CFG 2"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_arnoldi -s $SKIP -c 1 -o $O/arn $CMD > $O/ncu.log 2>&1; echo "rc=$?"
ncu -i $O/arn.ncu-rep --page source --csv > $O/src.csv 2>/dev/null
ncu -i $O/arn.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
rm -f $O/arn.ncu-rep
