# parity of the touched paths + short bench lines (HELR_HOIST_NB A/B)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q -m gpu > gpurun_out/q_tests.log 2>&1; tail -2 gpurun_out/q_tests.log
for nb in 2 4 8; do
HELR_HOIST_NB=$nb python tools/sweep.py --quick --ops rotsum > gpurun_out/q_sweep_$nb.jsonl 2>&1; cat gpurun_out/q_sweep_$nb.jsonl
HELR_HOIST_NB=$nb python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 > gpurun_out/q_bench_$nb.json 2> gpurun_out/q_bench_$nb.err
python -c "import json;d=json.load(open('gpurun_out/q_bench_$nb.json'));print($nb, d['value'],d['ms_per_step']);print({k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
