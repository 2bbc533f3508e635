#!/bin/bash
# DRAM bytes of the kernels of one headline GMRES iteration with the L2 left as the previous
# kernel left it (--cache-control none, one counter pass: no replay), forward traversal
# (AAC_REV=0) against the default direction mask: what the hand-over through L2 saves.
set -u
O=gpurun_out/ncu_l2; mkdir -p $O
CMD="python scripts/one_solve.py headline 1"
export MASKS=${MASKS:-"0 5 21"}
for m in $MASKS; do
  AAC_REV=$m timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --cache-control none --clock-control none \
    -k regex:"k_fwd_upd|k_waver|k_inverse|k_matvec|k_arnoldi" -s 60 -c 20 --csv --log-file $O/rev$m.csv $CMD > $O/rev$m.log 2>&1
  echo "ncu rev=$m rc=$?"
done
python - <<'P'
import csv, collections
import os
for m in os.environ.get("MASKS", "0 5 21").split():
    rows = [r for r in csv.reader(open(f"gpurun_out/ncu_l2/rev{m}.csv")) if len(r) > 10]
    h = rows[0]; ik = h.index("Kernel Name"); im = h.index("Metric Name"); iv = h.index("Metric Value"); iid = h.index("ID")
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault((r[iid], r[ik].split("(")[0][:40]), {})[r[im]] = float(r[iv].replace(",", ""))
    print(f"== AAC_REV={m}")
    tot = 0.0
    for (i, k), d in per.items():
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        tot += b
        print(f"  {i:>4} {k:42s} rd {d.get('dram__bytes_read.sum',0)/1e6:8.1f} MB  wr {d.get('dram__bytes_write.sum',0)/1e6:8.1f} MB  {d.get('gpu__time_duration.sum',0)/1e3:8.1f} us")
    print(f"  total {tot/1e6:.1f} MB over {len(per)} launches")
P
