#!/bin/bash
# A/B of the traversal-direction masks (AAC_REV) on a config: ms per solve, last of N solves.
# usage: bash scripts/ab_rev.sh CONFIG "mask mask ..."
set -u
CFG=${1:-headline}; MASKS=${2:-"0 2 18 20 5 10 31"}
O=gpurun_out/ab_rev; mkdir -p $O
for m in $MASKS; do
  echo "== AAC_REV=$m"
  AAC_REV=$m timeout 300 python scripts/one_solve.py $CFG 8 2>&1 | tail -4 | tee -a $O/$CFG.$m.log
done
