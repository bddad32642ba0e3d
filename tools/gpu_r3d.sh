# r3d: mixed-ring parity + bootstrap after the ModDown fix; ncu of the hoisted inner product
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mixed_p60" > gpurun_out/r3d_mixed.log 2>&1; tail -3 gpurun_out/r3d_mixed.log
timeout 900 python -m pytest tests/test_gpu_bootstrap.py -q -m gpu > gpurun_out/r3d_boot.log 2>&1; tail -5 gpurun_out/r3d_boot.log
bash tools/ncu_hoist.sh
