O=gpurun_out/r02f; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline > $O/b_head.json 2> $O/b_head.err; echo "head rc=$?"
CMD="python scripts/one_solve.py headline 2"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_arnoldi|k_fwd_upd" -c 30 --csv --log-file $O/ar.csv $CMD > $O/ncu1.log 2>&1; echo "ncu rc=$?"
