#!/bin/bash
# A/B SP library variants: "lib:ENV" pairs; timed saddle solves + serialised k_spf_* times.
set -u
O=gpurun_out/${1:-absp}; shift; mkdir -p $O
LIB=paper_2506_03947_b200/libaac.so
cp $LIB /tmp/_keep.so
for spec in "$@"; do
  so=${spec%%:*}; ev=${spec#*:}
  [ "$so" = default ] && so=/tmp/_keep.so
  cp $so $LIB
  echo "== $spec"; env $ev timeout 300 python scripts/one_solve.py saddle 4 2>&1 | tail -1
  n=$(echo "$spec" | tr -c 'a-zA-Z0-9' '_')
  env $ev timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_spf -s 60 -c 30 --csv --log-file $O/$n.csv python scripts/one_solve.py saddle 1 > /dev/null 2>&1
  python - $O/$n.csv <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
h = None; acc = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r: h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum": acc[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
print("   ", "  ".join(f"{k.replace('void ','')}: {sum(v)/len(v)/1e3:.1f}us x{len(v)}" for k, v in acc.items()))
PY
done
cp /tmp/_keep.so $LIB
