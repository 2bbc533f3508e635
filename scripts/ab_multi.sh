#!/bin/bash
# Time one config with several prebuilt libraries (separate processes, ROUNDS passes).
# usage: bash scripts/ab_multi.sh CONFIG ROUNDS LIB1.so LIB2.so ...
set -u
CFG=$1; R=$2; shift 2
LIB=paper_2506_03947_b200/libaac.so
cp $LIB /tmp/_keep.so
for i in $(seq $R); do
  for v in "$@"; do
    cp $v $LIB
    echo "== $v $(timeout 300 python scripts/one_solve.py $CFG 4 2>&1 | tail -1)"
  done
done
cp /tmp/_keep.so $LIB
