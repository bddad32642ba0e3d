#!/bin/bash
# precision sweep: refresh_bits (W/V scale after refresh) vs whole-run error
python tools/accuracy.py medium:47 medium:44 medium:42 paper_mini:44 paper_mini:42 > gpurun_out/r2c_acc.jsonl 2> gpurun_out/r2c_acc.err
python -c "
import json
for l in open('gpurun_out/r2c_acc.jsonl'):
    d=json.loads(l); print(d['workload'], d['refresh_bits'], '%.3e'%d['max_abs_dw'], '%.2e'%d['max_abs_dauc'], round(d['seconds'],1))
"
tail -3 gpurun_out/r2c_acc.err
