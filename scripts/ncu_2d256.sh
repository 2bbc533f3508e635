#!/bin/bash
# 2d256: launch list of one solve + ncu --set full of one mid-solve Arnoldi launch (CSV out).
set -u
O=gpurun_out/${1:-n256}; mkdir -p $O
CMD="python scripts/one_solve.py 2d256 2"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv $CMD > $O/ncu1.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:k_arnoldi -s 60 -c 1 -o $O/arn $CMD > $O/ncu2.log 2>&1; echo "full rc=$?"
ncu -i $O/arn.ncu-rep --page raw --csv > $O/arn_raw.csv 2>/dev/null; rm -f $O/arn.ncu-rep
timeout 600 ncu --set full --clock-control none -k regex:k_fwd -s 60 -c 1 -o $O/fwd $CMD > $O/ncu3.log 2>&1; echo "full fwd rc=$?"
ncu -i $O/fwd.ncu-rep --page raw --csv > $O/fwd_raw.csv 2>/dev/null; rm -f $O/fwd.ncu-rep
