#!/bin/bash
# A/B of the calA apply: k_matvec (AAC_MATVEC_ROWS=0) vs the row-marching k_matvec_rows at several
# rows-per-thread settings (stencil_probe: back to back, graph replay), then the headline bench.
set -u
O=gpurun_out/ab_mvr; mkdir -p $O
echo "== k_matvec"; AAC_MATVEC_ROWS=0 timeout 300 python scripts/stencil_probe.py 2>&1 | tail -2
echo "== rows default"; timeout 300 python scripts/stencil_probe.py 2>&1 | tail -2
for ry in 2 4 8 16 32 64; do echo "== rows RY=$ry"; AAC_MATVEC_RY=$ry timeout 300 python scripts/stencil_probe.py 2>&1 | tail -2; done
