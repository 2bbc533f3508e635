# ncu --set full of kernels matching a regex on the headline solve; usage: bash scripts/ncu_one.sh TAG REGEX [SKIP] [COUNT]
T=${1:-r2_x}; KRE=$2; SKIP=${3:-4}; CNT=${4:-1}; O=gpurun_out/$T; mkdir -p $O
CMD="python scripts/one_solve.py headline 2"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c $CNT -o $O/prof $CMD > $O/ncu.log 2>&1; echo "ncu rc=$?"
