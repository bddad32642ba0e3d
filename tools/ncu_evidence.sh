# Profile evidence for profiles/: (1) one-step launch list with DRAM bytes,
# (2) launch list of the bench command (gpu__time_duration only),
# (3) --set full captures of the top kernels of one step.
# Usage: bash tools/ncu_evidence.sh TAG
TAG=${1:-r01}
set -x
python tools/profile_step.py > gpurun_out/pstep_$TAG.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/step_launches_$TAG.csv python tools/profile_step.py > gpurun_out/ncu_step_$TAG.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --cpu-iters 0 --profile-steps 1"
$B > gpurun_out/bshort_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/bench_launches_$TAG.csv $B > gpurun_out/ncu_bl_$TAG.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"ntt_pass|k_ks_inner_hoisted|k_moddown_final|k_modup|k_moddown_conv" -c 12 -f -o gpurun_out/full_$TAG python tools/profile_step.py > gpurun_out/ncu_full_$TAG.log 2>&1
ls gpurun_out | grep $TAG
