#!/bin/bash
# ncu capture of one config: plain run, launch list, then a full capture of a kernel range.
# usage: bash scripts/prof.sh TAG CONFIG REGEX SKIP COUNT [NSOLVES]
set -u
TAG=$1; CFG=$2; KRE=$3; SKIP=$4; CNT=$5; NS=${6:-2}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }
CMD="python scripts/one_solve.py $CFG $NS"
timeout 600 $CMD > $O/plain.log 2>&1; rc=$?; echo "plain rc=$rc"; cat $O/plain.log | tail -4
[ $rc -eq 0 ] || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv $CMD > $O/ncu1.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c $CNT -o $O/prof $CMD > $O/ncu2.log 2>&1; echo "ncu full rc=$?"
tail -3 $O/ncu2.log
