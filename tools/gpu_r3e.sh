mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bootstrap.py -q -m gpu -s > gpurun_out/r3e_boot.log 2>&1; grep -E "max .dw|passed|failed|^E  " gpurun_out/r3e_boot.log | head -20
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r3e_parity.log 2>&1; tail -2 gpurun_out/r3e_parity.log
