# Headline solve time under several environment settings (no tests).
# usage: bash scripts/ab_env.sh TAG "ENV1" "ENV2" ...   (each ENVk: space-separated VAR=VAL, or "-")
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
i=0
for envs in "$@"; do
  i=$((i+1))
  if [ "$envs" = "-" ]; then envs=""; fi
  env $envs timeout 300 python scripts/one_solve.py headline 5 > $O/solve_$i.log 2>&1; echo "[$envs] $(tail -1 $O/solve_$i.log)"
done
