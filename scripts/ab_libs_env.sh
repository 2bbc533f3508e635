#!/bin/bash
# A/B prebuilt libraries x env settings on one config (alternating rounds, separate processes).
# usage: bash scripts/ab_libs_env.sh CONFIG ROUNDS "ENV;ENV2" A.so B.so ...
set -u
CFG=$1; R=$2; ENVS=$3; shift 3
LIB=paper_2506_03947_b200/libaac.so
cp $LIB /tmp/_keep.so
IFS=';' read -ra VS <<< "$ENVS"
for i in $(seq $R); do
  for so in "$@"; do
    cp $so $LIB
    for v in "${VS[@]}"; do
      echo "== $so [$v] $(env $v timeout 300 python scripts/one_solve.py $CFG 5 2>&1 | tail -1)"
    done
  done
done
cp /tmp/_keep.so $LIB
