#!/bin/bash
# Round bench: every BASELINE config through bench.py, then the headline launch list (of one solve
# and of the bench command itself) and one ncu --set full capture of one GMRES iteration.
set -u
TAG=${1:-bench}
O=gpurun_out/$TAG; mkdir -p $O
if [ -z "${SKIPBUILD:-}" ]; then python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }; fi
timeout 600 python bench.py > $O/b_head.json 2> $O/b_head.err; echo "head rc=$?"
for c in saddle 2d256 1d; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/b_$c.json 2> $O/b_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config 3d --maxit 20 --steps 2 --no-cpu-baseline > $O/b_3d.json 2> $O/b_3d.err; echo "3d rc=$?"
timeout 900 python bench.py --impl reference --steps 2 > $O/b_ref.json 2> $O/b_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config paper500 --steps 3 > $O/b_paper500.json 2> $O/b_paper500.err; echo "paper500 rc=$?"
timeout 600 python bench.py --config paper500 --method exact --steps 3 --no-cpu-baseline > $O/b_paper500_exact.json 2> $O/b_paper500_exact.err; echo "paper500 exact rc=$?"
CMD="python scripts/one_solve.py headline 2"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv $CMD > $O/ncu1.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu bench launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_wave|k_fwd|k_arnoldi|k_matvec|k_inverse" -s 40 -c 5 -o $O/prof $CMD > $O/ncu2.log 2>&1; echo "ncu full rc=$?"
