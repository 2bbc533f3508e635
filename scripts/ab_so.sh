#!/bin/bash
# A/B two prebuilt libraries on one config (alternating, separate processes).
# usage: bash scripts/ab_so.sh OLD.so NEW.so CONFIG [ROUNDS]
set -u
A=$1; B=$2; CFG=$3; R=${4:-2}
LIB=paper_2506_03947_b200/libaac.so
cp $LIB /tmp/_keep.so
for i in $(seq $R); do
  for v in A B; do
    if [ $v = A ]; then cp $A $LIB; else cp $B $LIB; fi
    echo "== $v"; timeout 300 python scripts/one_solve.py $CFG 4 2>&1 | tail -2
  done
done
cp /tmp/_keep.so $LIB
