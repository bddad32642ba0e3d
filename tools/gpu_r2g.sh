#!/bin/bash
# pipelined hoisted inner product: parity + step A/B
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_trainer_residue.py -x -q -m gpu > gpurun_out/r2g_tests.log 2>&1; tail -2 gpurun_out/r2g_tests.log
for hp in 0 1; do
HELR_HOIST_PIPE=$hp timeout 600 python bench.py --steps 200 --warmup 5 --no-e2e --cpu-iters 0 > gpurun_out/r2g_bench_$hp.json 2> gpurun_out/r2g_bench_$hp.err
python -c "import json;d=json.load(open('gpurun_out/r2g_bench_$hp.json'));print('pipe=$hp', round(d['value'],2),round(d['ms_per_step'],3));print({k:round(v['ms'],3) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/r2g_bench_$hp.err
done
