#!/bin/bash
# One GPU call: parity tests, bench (headline), launch list + one full ncu capture.
# usage: bash scripts/gpu_round.sh TAG [ncu-kernel-regex] [ncu-skip]
set -u
TAG=${1:-run}; KRE=${2:-k_sweep}; SKIP=${3:-40}
O=gpurun_out/$TAG; mkdir -p $O
if [ -z "${SKIPBUILD:-}" ]; then python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }; fi
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 600 $O/bench.json
CMD="python scripts/one_solve.py headline 2"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv $CMD > $O/ncu1.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 3 -o $O/prof $CMD > $O/ncu2.log 2>&1; echo "ncu full rc=$?"
ls -la $O
