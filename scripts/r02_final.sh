#!/bin/bash
# Round-2 final GPU pass: the whole -m gpu suite, smoke(), every bench config, the headline and
# saddle launch lists, one ncu --set full capture of a headline iteration and of the SP K1 kernel.
set -u
O=gpurun_out/r02_final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
SKIPBUILD=1 bash scripts/gpu_bench_all.sh r02_final/bench
B=$O/bench
CMD="python scripts/one_solve.py saddle 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $B/saddle_launches.csv $CMD > $B/ncu_saddle.log 2>&1; echo "ncu saddle launches rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"k_spf_apply_tma" -s 20 -c 1 -o $B/sp_k1 $CMD > $B/ncu_sp_k1.log 2>&1; echo "ncu sp k1 rc=$?"
ncu -i $B/sp_k1.ncu-rep --page raw --csv > $B/sp_k1_raw.csv 2>/dev/null; rm -f $B/sp_k1.ncu-rep
python scripts/ncu_summary.py $B/prof.ncu-rep > $B/ncu_full_summary.txt 2>&1
ncu -i $B/prof.ncu-rep --page raw --csv 2>/dev/null | gzip > $B/ncu_full_raw.csv.gz; rm -f $B/prof.ncu-rep
ls -la $B | head -40
