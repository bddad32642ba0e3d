# r3b: bootstrap GPU tests + ncu of the TMA vs plain NTT passes (microbench, 112 fp64 limbs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bootstrap.py -q -m gpu > gpurun_out/r3b_boot.log 2>&1; tail -5 gpurun_out/r3b_boot.log
for t in 0 1; do
  HELR_NTT_TMA=$t timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:ntt_pass \
     -o /tmp/r3b_ntt_tma$t -f python tools/ntt_micro.py --once > gpurun_out/r3b_ncu$t.log 2>&1
  tail -1 gpurun_out/r3b_ncu$t.log
  python tools/ncu_brief.py /tmp/r3b_ntt_tma$t.ncu-rep > gpurun_out/r3b_brief$t.txt 2>&1
done
