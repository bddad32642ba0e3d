python -m pytest tests -x -q -m gpu > gpurun_out/f_tests.log 2>&1; tail -1 gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
python tools/accuracy.py toy medium paper_mini paper_full > gpurun_out/f_acc.jsonl 2> gpurun_out/f_acc.err
python -c "
import json
for l in open('gpurun_out/f_acc.jsonl'):
    d=json.loads(l); print(d['workload'], d['dnum'], d['refresh_bits'], d['iterations'], '%.3e'%d['max_abs_dw'], '%.3e'%d['max_abs_dauc'], round(d['seconds'],1))
"
