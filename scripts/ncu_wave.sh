# ncu --set full of the wavefront kernel (new, then old) on the headline; usage: bash scripts/ncu_wave.sh TAG
T=${1:-r2_w}; O=gpurun_out/$T; mkdir -p $O
CMD="python scripts/one_solve.py headline 2"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_waver -s 4 -c 1 -o $O/prof_new $CMD > $O/ncu_new.log 2>&1; echo "ncu new rc=$?"
AAC_WAVE_OLD=1 timeout 300 $CMD > $O/plain_old.log 2>&1 && \
AAC_WAVE_OLD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 4 -c 1 -o $O/prof_old $CMD > $O/ncu_old.log 2>&1; echo "ncu old rc=$?"
