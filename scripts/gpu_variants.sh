#!/bin/bash
# Build variants (extra nvcc -D flags) and time a config with each.
# usage: bash scripts/gpu_variants.sh TAG CONFIG "FLAGS1;FLAGS2;..." [ENV]
set -u
TAG=$1; CFG=$2; VARIANTS=$3; ENVV=${4:-}
O=gpurun_out/$TAG; mkdir -p $O
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  echo "== $v"
  AAC_EXTRA_NVCC="$v" python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; continue; }
  env $ENVV timeout 300 python scripts/one_solve.py $CFG 4 2>&1 | tail -2
done
