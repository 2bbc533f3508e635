#!/bin/bash
# Full ncu capture of the fused SP level-0 kernels (one launch each, steady state), exported as CSV.
set -u
O=gpurun_out/${1:-ncusp}; mkdir -p $O
for k in k_spf_apply k_spf_restrict k_spf_prolong_post; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 20 -c 1 -o $O/$k python scripts/one_solve.py saddle 1 > $O/ncu_$k.log 2>&1; echo "$k rc=$?"
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/raw_$k.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv > $O/src_$k.csv 2>/dev/null
  rm -f $O/$k.ncu-rep
done
