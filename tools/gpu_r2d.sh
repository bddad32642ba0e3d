#!/bin/bash
# cluster NTT: parity + microbench + step A/B
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trainer_residue.py -x -q -m gpu > gpurun_out/r2d_tests.log 2>&1; tail -5 gpurun_out/r2d_tests.log
for cl in 0 1; do
  for bk in 0 1; do
    HELR_NTT_CLUSTER=$cl HELR_NTT_BULK=$bk timeout 300 python tools/ntt_micro.py --batch 16 > gpurun_out/r2d_micro_$cl$bk.json 2>&1; echo "cl=$cl bulk=$bk"; cat gpurun_out/r2d_micro_$cl$bk.json | cut -c1-600
  done
done
for cl in 0 1; do
HELR_NTT_CLUSTER=$cl timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 > gpurun_out/r2d_bench_$cl.json 2> gpurun_out/r2d_bench_$cl.err
python -c "import json;d=json.load(open('gpurun_out/r2d_bench_$cl.json'));print('cluster=$cl', round(d['value'],2),round(d['ms_per_step'],3));print({k:round(v['ms'],3) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/r2d_bench_$cl.err
done
