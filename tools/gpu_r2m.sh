#!/bin/bash
# r02 evidence: default bench line, reference arm, paper_full line, ncu launch lists + full captures (text briefs only)
nproc
timeout 1500 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
python -c "import json;d=json.load(open('gpurun_out/r2m_bench.json'));print(round(d['value'],2),round(d['ms_per_step'],3), d['e2e']['value'], json.dumps(d['roofline']));print({k:round(v['ms'],3) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/r2m_bench.err
timeout 600 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/r2m_bench_ref.json 2> gpurun_out/r2m_bench_ref.err; tail -c 300 gpurun_out/r2m_bench_ref.json
timeout 900 python bench.py --workload paper_full --steps 3 --warmup 3 --cpu-iters 0 > gpurun_out/r2m_full.json 2> gpurun_out/r2m_full.err
python -c "import json;d=json.load(open('gpurun_out/r2m_full.json'));print(d['value'],d['ms_per_step'], d['e2e'])" || tail -5 gpurun_out/r2m_full.err
bash tools/ncu_evidence.sh r02 > gpurun_out/evidence_r02.log 2>&1
python tools/ncu_brief.py gpurun_out/full_r02.ncu-rep > gpurun_out/full_r02.txt 2>&1
python tools/ncu_table.py gpurun_out/full_r02.ncu-rep --md gpurun_out/full_table_r02.md > /dev/null 2>&1
rm -f gpurun_out/full_r02.ncu-rep
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; tail -1 gpurun_out/smoke_r02.log
du -sh gpurun_out
