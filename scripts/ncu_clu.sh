#!/bin/bash
# Full ncu capture of the real ns=8 wavefront block, halo vs cluster kernel.
set -u
O=gpurun_out/${1:-cluncu}; mkdir -p $O
for c in 0 1; do
  AAC_WAVE_CLUSTER=$c timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_waver<\(int\)8, \(int\)128, \(int\)8, \(bool\)0' -c 1 -o $O/w_c$c python scripts/one_solve.py headline 1 > $O/ncu_c$c.log 2>&1; echo "ncu c=$c rc=$?"
done
for c in 0 1; do
  ncu -i $O/w_c$c.ncu-rep --page raw --csv > $O/raw_c$c.csv 2>/dev/null
  ncu -i $O/w_c$c.ncu-rep --page details --csv > $O/det_c$c.csv 2>/dev/null
  rm -f $O/w_c$c.ncu-rep
done
