#!/bin/bash
# A/B of the cluster wavefront: parity tests, then alternating timed headline solves.
set -u
O=gpurun_out/${1:-clu}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "${2:-cluster or sweep_organisations or headline_full_size_apply}" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for r in 1 2; do for c in 0 1; do
  echo "== AAC_WAVE_CLUSTER=$c"; AAC_WAVE_CLUSTER=$c timeout 300 python scripts/one_solve.py ${3:-headline} 6 2>&1 | tail -3
done; done
