#!/bin/bash
# SP quick check: parity tests of the SP path, timed saddle solves, serialised per-kernel times.
set -u
O=gpurun_out/${1:-spq}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "sp_ or saddle" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 300 python scripts/one_solve.py saddle 4 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_spf -s 60 -c 30 --csv --log-file $O/spf.csv python scripts/one_solve.py saddle 1 > /dev/null 2>&1
python - <<PY
import csv, collections
rows = list(csv.reader(open("$O/spf.csv")))
h = None; acc = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r: h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum": acc[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
for k, v in acc.items(): print(k, len(v), "mean us", sum(v) / len(v) / 1e3)
PY
