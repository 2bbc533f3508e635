#!/bin/bash
# A/B two prebuilt libraries on one config (alternating, separate processes).
# usage: bash scripts/ab_so.sh OLD.so NEW.so CONFIG [ROUNDS]
set -u
A=$1; B=$2; CFG=$3; R=${4:-2}
LIB=paper_2506_03947_b200/libaac.so
cp $LIB /tmp/_keep.so
cp $A /tmp/_ab_A.so; cp $B /tmp/_ab_B.so      # (either may be $LIB itself)
for i in $(seq $R); do
  for v in A B; do
    cp /tmp/_ab_$v.so $LIB
    echo "== $v"; timeout 300 python scripts/one_solve.py $CFG 4 2>&1 | tail -2
  done
done
cp /tmp/_keep.so $LIB
