#!/bin/bash
# Source-level ncu (SASS + stall samples, raw metrics) of one launch of a kernel, as CSV.
# usage: bash scripts/ncu_src.sh TAG CONFIG REGEX SKIP
set -u
O=gpurun_out/$1; CFG=$2; RE=$3; SKIP=${4:-20}; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$RE" -s $SKIP -c 1 -o $O/k python scripts/one_solve.py $CFG 1 > $O/ncu.log 2>&1; echo "rc=$?"
ncu -i $O/k.ncu-rep --page source --csv > $O/src.csv 2>/dev/null
ncu -i $O/k.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
rm -f $O/k.ncu-rep
