# r3a: TMA NTT path — parity (forced on every N=2^16 launch), microbench and step A/B
mkdir -p gpurun_out
HELR_NTT_TMA_MIN_TILES=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q -m gpu > gpurun_out/r3a_tests.log 2>&1; tail -3 gpurun_out/r3a_tests.log
for t in 0 1; do
  echo "ntt_micro TMA=$t"; HELR_NTT_TMA=$t timeout 300 python tools/ntt_micro.py --batch 16 2>&1 | tail -1
done
for t in 0 1; do
  HELR_NTT_TMA=$t timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 > gpurun_out/r3a_bench_$t.json 2> gpurun_out/r3a_bench_$t.err
  python -c "import json;d=json.load(open('gpurun_out/r3a_bench_$t.json'));print('TMA=$t', round(d['value'],2),round(d['ms_per_step'],3));print({k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
