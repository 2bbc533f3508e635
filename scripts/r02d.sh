O=gpurun_out/r02d; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline > $O/b_head.json 2> $O/b_head.err; echo "head rc=$?"
timeout 300 python bench.py --config saddle --no-cpu-baseline > $O/b_saddle.json 2> $O/b_saddle.err; echo "saddle rc=$?"
