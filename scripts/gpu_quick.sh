#!/bin/bash
# Quick GPU check: build, a pytest selection, timed solves of a config under env variants.
# usage: bash scripts/gpu_quick.sh TAG "PYTEST -k expr" CONFIG "ENV1;ENV2;..."
set -u
TAG=$1; KEXPR=$2; CFG=$3; VARIANTS=$4
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }
if [ -n "$KEXPR" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
fi
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  echo "== $v"
  env $v timeout 300 python scripts/one_solve.py $CFG 4 2>&1 | tail -2
done
