# A/B of wavefront variants: parity (wave-related GPU tests) + headline solve times + bench line.
# usage: bash scripts/ab_wave.sh TAG "ENV1" "ENV2" ...   (each ENVk: space-separated VAR=VAL, or "-")
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paper.py -x -q -k "wave or organisation or precond or gmres or paper" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
i=0
for envs in "$@"; do
  i=$((i+1))
  if [ "$envs" = "-" ]; then envs=""; fi
  env $envs timeout 300 python scripts/one_solve.py headline 6 > $O/solve_$i.log 2>&1; echo "[$envs]"; tail -1 $O/solve_$i.log
done
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['roofline']['frac'], d['config']['kernels']['cheb_sweep'])"
