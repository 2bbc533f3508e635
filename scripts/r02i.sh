#!/bin/bash
# Re-entry check of the restored tree: the whole -m gpu suite, smoke(), headline / saddle / 2d256 bench lines.
set -u
O=gpurun_out/r02i; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/b_headline.json 2> $O/b_headline.err; echo "head rc=$?"
for c in saddle 2d256; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/b_$c.json 2> $O/b_$c.err; echo "$c rc=$?"
done
python - <<'P'
import json
for c in ("headline","saddle","2d256"):
    try:
        d=json.load(open(f"gpurun_out/r02i/b_{c}.json")); print(c, round(d["value"],1), d["e2e"]["value"], d["clocks"])
    except Exception as e: print(c, "ERR", e)
P
