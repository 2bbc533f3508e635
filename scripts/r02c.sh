O=gpurun_out/r02c; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "sp_ or saddle" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for e in "X=1" "AAC_PDL=0" "AAC_SP_FUSED=0"; do echo "== $e"; env $e timeout 300 python scripts/one_solve.py saddle 4 2>&1 | tail -2; done
CMD="python scripts/one_solve.py saddle 2"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_saddle.csv $CMD > $O/ncu1.log 2>&1; echo "ncu rc=$?"
