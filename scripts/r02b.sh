O=gpurun_out/r02b; mkdir -p $O
timeout 300 python bench.py --no-cpu-baseline > $O/b_head.json 2> $O/b_head.err; echo "head rc=$?"
timeout 300 python bench.py --config saddle --no-cpu-baseline > $O/b_saddle.json 2> $O/b_saddle.err; echo "saddle rc=$?"
CMD="python scripts/one_solve.py saddle 2"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_saddle.csv $CMD > $O/ncu1.log 2>&1; echo "ncu rc=$?"
