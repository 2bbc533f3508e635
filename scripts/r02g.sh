O=gpurun_out/r02g; mkdir -p $O
CMD="python scripts/one_solve.py saddle 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spf_apply|k_spf_prolong_post|k_spf_restrict" -s 30 -c 6 -o $O/prof $CMD > $O/ncu.log 2>&1; echo "ncu rc=$?"
