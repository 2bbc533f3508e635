#!/bin/bash
# A/B several prebuilt libraries on one config (alternating rounds, separate processes).
# usage: bash scripts/ab_multi.sh CONFIG ROUNDS A.so B.so ...
set -u
CFG=$1; R=$2; shift 2
LIB=paper_2506_03947_b200/libaac.so
cp $LIB /tmp/_keep.so
# (snapshot every library first: one of them may be $LIB itself)
n=0; snaps=()
for so in "$@"; do cp $so /tmp/_ab_$n.so; snaps+=("/tmp/_ab_$n.so:$so"); n=$((n+1)); done
for i in $(seq $R); do
  for sp in "${snaps[@]}"; do
    so=${sp#*:}
    cp ${sp%%:*} $LIB
    echo "== $so $(timeout 300 python scripts/one_solve.py $CFG 4 2>&1 | tail -1)"
  done
done
cp /tmp/_keep.so $LIB
