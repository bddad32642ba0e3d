set -x
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --cpu-iters 0 --profile-steps 1 --no-graph"
$CMD > gpurun_out/plain3.json 2> gpurun_out/plain3.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 700 --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ntt_pass -s 600 -c 4 -o gpurun_out/prof_ntt $CMD > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_modup|k_ks_inner|k_moddown" -s 300 -c 4 -o gpurun_out/prof_ks $CMD > gpurun_out/ncu_k.log 2>&1
ls -la gpurun_out/
