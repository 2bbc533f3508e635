O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "matvec or gmres_parity or headline" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for e in "X=1" "AAC_MATVEC_TILE=0"; do echo "== $e"; env $e timeout 300 python scripts/one_solve.py headline 5 2>&1 | tail -1; done
CMD="python scripts/one_solve.py headline 2"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_matvec -c 10 --csv --log-file $O/mv.csv $CMD > $O/ncu1.log 2>&1; echo "ncu rc=$?"
timeout 300 python bench.py --no-cpu-baseline > $O/b_head.json 2> $O/b_head.err; echo "head rc=$?"
