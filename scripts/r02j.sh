#!/bin/bash
# Row-marching calA apply: bit-identity + parity tests, stencil A/B sweep, headline bench both ways,
# then the ncu traffic capture of one headline iteration.
set -u
O=gpurun_out/r02j; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "matvec or gmres_parity or headline or multirank" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
bash scripts/ab_matvec_rows.sh > $O/ab.log 2>&1; cat $O/ab.log
timeout 600 python bench.py --no-cpu-baseline > $O/b_rows.json 2> $O/b_rows.err; echo "bench rows rc=$?"
AAC_MATVEC_ROWS=0 timeout 600 python bench.py --no-cpu-baseline > $O/b_old.json 2> $O/b_old.err; echo "bench old rc=$?"
python - <<'P'
import json
for c in ("rows","old"):
    try:
        d=json.load(open(f"gpurun_out/r02j/b_{c}.json")); k=d["config"]["kernels"]["matvec"]
        print(c, round(d["value"],1), "stencil%", round(d["config"]["stencil_pct_of_peak"],1), "in-solve%", round(d["config"]["stencil_pct_of_peak_in_solve"],1), "matvec ms/solve", round(k["ms_per_step"],3))
    except Exception as e: print(c, "ERR", e)
P
bash scripts/ncu_traffic_r02.sh
