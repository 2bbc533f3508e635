O=gpurun_out/r02h; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "multirank or nccl or wave" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
