#!/bin/bash
# Cluster wavefront diagnostics: the halo kernel launched in clusters (scheduling cost), and the
# serialised per-launch times (ncu) of the halo vs the cluster kernel.
set -u
O=gpurun_out/${1:-clu}; mkdir -p $O
for v in "AAC_WAVE_CLUSTER=0" "AAC_WAVE_CLUSTER=0 AAC_WAVE_CLDIM=2" "AAC_WAVE_CLUSTER=0 AAC_WAVE_CLDIM=8" "AAC_WAVE_CLUSTER=1"; do
  echo "== $v"; env $v timeout 300 python scripts/one_solve.py headline 5 2>&1 | tail -2
done
for c in 0 1; do
  AAC_WAVE_CLUSTER=$c timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__cluster_dim_x --clock-control none -k regex:k_waver -c 12 --csv --log-file $O/wave_c$c.csv python scripts/one_solve.py headline 1 > $O/ncu_c$c.log 2>&1; echo "ncu c=$c rc=$?"
done
