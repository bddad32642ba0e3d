#!/bin/bash
# fused basis conversions: parity + A/B
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2l_tests.log 2>&1; tail -3 gpurun_out/r2l_tests.log
for fc in 0 1; do
HELR_FUSE_CONV=$fc timeout 600 python bench.py --steps 200 --warmup 5 --no-e2e --cpu-iters 0 > gpurun_out/r2l_bench_$fc.json 2> gpurun_out/r2l_bench_$fc.err
python -c "import json;d=json.load(open('gpurun_out/r2l_bench_$fc.json'));print('fuse=$fc', round(d['value'],2),round(d['ms_per_step'],3), d['gpu_launches']/d['steps']);print({k:round(v['ms'],3) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/r2l_bench_$fc.err
done
