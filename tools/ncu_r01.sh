# Round-1 evidence: full bench line, reference arm, one-step ncu launch list
# with DRAM bytes, launch list of the bench command, full captures of the top kernels.
set -x
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_r01.json 2> gpurun_out/bench_ref_r01.err
python tools/profile_step.py > gpurun_out/pstep.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/step_launches_r01.csv python tools/profile_step.py > gpurun_out/ncu_step.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --cpu-iters 0 --profile-steps 1"
$B > gpurun_out/bshort.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/bench_launches_r01.csv $B > gpurun_out/ncu_bl.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_ks_inner_hoisted|k_moddown_conv|k_modup|k_mdr_conv" -c 8 -o gpurun_out/prof_ks_r01 python tools/profile_step.py > gpurun_out/ncu_ks.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"ntt_pass" -c 6 -o gpurun_out/prof_ntt_r01 python tools/profile_step.py > gpurun_out/ncu_ntt.log 2>&1
ls gpurun_out
