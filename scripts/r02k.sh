#!/bin/bash
# Re-entry pass with the traversal-direction default (AAC_REV = 5): the whole -m gpu suite,
# smoke(), the headline / saddle / 2d256 bench lines.
set -u
O=gpurun_out/r02k; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
for c in headline saddle 2d256; do
  timeout 600 python bench.py --config $c > $O/b_$c.json 2> $O/b_$c.err; echo "bench $c rc=$?"
  python -c "import json,sys; d=json.loads(open('$O/b_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])"
done
