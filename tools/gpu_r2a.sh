#!/bin/bash
# round-2 quick check: full GPU suite + short bench
python -m pytest tests -x -q -m gpu > gpurun_out/r2a_tests.log 2>&1; tail -3 gpurun_out/r2a_tests.log
python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
python -c "import json;d=json.load(open('gpurun_out/r2a_bench.json'));print(round(d['value'],2),round(d['ms_per_step'],3), d['gpu_launches']/d['steps']);print({k:round(v['ms'],3) for k,v in d['kernels'].items()})"
tail -3 gpurun_out/r2a_bench.err
