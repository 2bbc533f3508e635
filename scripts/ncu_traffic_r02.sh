#!/bin/bash
# ncu --set full of one headline GMRES iteration (j = 6 of the first solve): k_fwd_upd, the six
# k_waver launches of the preconditioner apply, k_inverse_exact, k_matvec, k_arnoldi -- the DRAM
# bytes per launch that bench.py reports as roofline.traffic (profiles/ncu_traffic.json).
set -u
O=gpurun_out/ncu_traffic; mkdir -p $O
CMD="python scripts/one_solve.py headline 1"
timeout 300 $CMD > $O/plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_fwd_upd|k_waver|k_inverse_exact|k_matvec|k_arnoldi" -s 60 -c 10 -o $O/it $CMD > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/it.ncu-rep --page raw --csv > $O/it_raw.csv 2>/dev/null
python scripts/ncu_summary.py $O/it.ncu-rep > $O/it_summary.txt 2>&1
gzip -f $O/it_raw.csv; rm -f $O/it.ncu-rep
cat $O/it_summary.txt
