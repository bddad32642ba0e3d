# r3c: hoisted inner product with the prefetch interleaved into the MAC block
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q -m gpu > gpurun_out/r3c_tests.log 2>&1; tail -3 gpurun_out/r3c_tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 > gpurun_out/r3c_bench.json 2> gpurun_out/r3c_bench.err
python -c "import json;d=json.load(open('gpurun_out/r3c_bench.json'));print(round(d['value'],2),round(d['ms_per_step'],3));print({k:round(v['ms'],3) for k,v in d['kernels'].items()})"
timeout 900 python -m pytest tests/test_gpu_bootstrap.py -q -m gpu > gpurun_out/r3c_boot.log 2>&1; tail -5 gpurun_out/r3c_boot.log
