#!/bin/bash
# full default bench line (C1-C3 CPU baselines) + paper_full line
nproc
timeout 1500 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
python -c "import json;d=json.load(open('gpurun_out/r2k_bench.json'));print(round(d['value'],2),round(d['ms_per_step'],3), d['e2e']['value'], json.dumps(d['roofline']), json.dumps(d['cpu_baseline']))" || tail -5 gpurun_out/r2k_bench.err
timeout 900 python bench.py --workload paper_full --steps 3 --warmup 3 --cpu-iters 0 > gpurun_out/r2k_full.json 2> gpurun_out/r2k_full.err
python -c "import json;d=json.load(open('gpurun_out/r2k_full.json'));print(d['value'],d['ms_per_step'], d['e2e'], json.dumps(d['roofline']))" || tail -5 gpurun_out/r2k_full.err
