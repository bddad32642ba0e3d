python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q -m gpu > gpurun_out/q_tests.log 2>&1; tail -1 gpurun_out/q_tests.log
for cfg in ""; do
python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 $cfg > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python -c "import json;d=json.load(open('gpurun_out/q_bench.json'));print('$cfg', round(d['value'],2),round(d['ms_per_step'],3), d['gpu_launches']/d['steps']);print({k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
