#!/bin/bash
# A/B several prebuilt libraries on one config (alternating rounds, separate processes).
# usage: bash scripts/ab_multi.sh CONFIG ROUNDS A.so B.so ...
set -u
CFG=$1; R=$2; shift 2
LIB=paper_2506_03947_b200/libaac.so
cp $LIB /tmp/_keep.so
for i in $(seq $R); do
  for so in "$@"; do
    cp $so $LIB
    echo "== $so $(timeout 300 python scripts/one_solve.py $CFG 4 2>&1 | tail -1)"
  done
done
cp /tmp/_keep.so $LIB
