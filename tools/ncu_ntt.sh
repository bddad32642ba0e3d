# quick primitive sweep, then a full ncu capture of the big batched NTT passes
python tools/sweep.py --quick > gpurun_out/sweep_quick.jsonl 2> gpurun_out/sweep_quick.err
CMD="python tools/sweep.py --quick --ops ntt"
$CMD > gpurun_out/plain_ntt.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ntt_pass -s 4 -c 4 -o gpurun_out/prof_ntt2 $CMD > gpurun_out/ncu_ntt2.log 2>&1
tail -2 gpurun_out/ncu_ntt2.log
