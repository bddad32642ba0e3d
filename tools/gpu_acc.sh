python -m pytest tests/test_gpu_train.py -x -q -m gpu > gpurun_out/acc_tests.log 2>&1; tail -1 gpurun_out/acc_tests.log
python tools/accuracy.py toy medium paper_mini paper_full > gpurun_out/accuracy8.jsonl 2> gpurun_out/accuracy8.err
python -c "
import json
for l in open('gpurun_out/accuracy8.jsonl'):
    d=json.loads(l); print(d['workload'], d['dnum'], d['refresh_bits'], d['iterations'], '%.3e'%d['max_abs_dw'], '%.3e'%d['max_abs_dauc'], round(d['seconds'],1))
"
