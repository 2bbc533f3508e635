#!/bin/bash
# Cluster wavefront A/B: halo kernel vs cluster kernel (default lib and variants/*.so), timed
# solves and the serialised ncu per-launch times of the wavefront kernels.
set -u
O=gpurun_out/${1:-clu}; mkdir -p $O
LIB=paper_2506_03947_b200/libaac.so
cp $LIB /tmp/_keep.so
timeout 600 python -m pytest tests -m gpu -x -q -k "cluster or sweep_organisations" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for so in /tmp/_keep.so variants/*.so; do
  cp $so $LIB
  for c in 0 1; do
    echo "== $so AAC_WAVE_CLUSTER=$c"; AAC_WAVE_CLUSTER=$c timeout 300 python scripts/one_solve.py headline 5 2>&1 | tail -2
  done
  n=$(basename $so .so)
  AAC_WAVE_CLUSTER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_waver -c 6 --csv --log-file $O/wave_$n.csv python scripts/one_solve.py headline 1 > /dev/null 2>&1
done
cp /tmp/_keep.so $LIB
