python -m pytest tests -x -q -m gpu > gpurun_out/f_tests.log 2>&1; tail -1 gpurun_out/f_tests.log
python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
python -c "import json;d=json.load(open('gpurun_out/f_bench.json'));print(round(d['value'],2),round(d['ms_per_step'],3), d['gpu_launches']/d['steps'], d['config']['K']);print({k:round(v['ms'],3) for k,v in d['kernels'].items()})"
python tools/accuracy.py toy medium paper_mini paper_full > gpurun_out/f_acc.jsonl 2> gpurun_out/f_acc.err
python -c "
import json
for l in open('gpurun_out/f_acc.jsonl'):
    d=json.loads(l); print(d['workload'], d['dnum'], d['refresh_bits'], d['iterations'], '%.3e'%d['max_abs_dw'], '%.3e'%d['max_abs_dauc'], round(d['seconds'],1))
"
