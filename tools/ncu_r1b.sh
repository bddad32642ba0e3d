CMD="python tools/sweep.py --quick --ops rotsum,ntt"
$CMD > gpurun_out/sweep_r1b.jsonl 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_ks_inner_hoisted|ntt_pass" -s 8 -c 6 -o gpurun_out/prof_r1b $CMD > gpurun_out/ncu_r1b.log 2>&1
tail -2 gpurun_out/ncu_r1b.log
