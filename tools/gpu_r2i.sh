#!/bin/bash
# precision: W/V re-entry scale after the refresh stand-in (refresh_bits)
python tools/accuracy.py paper_mini:48 paper_mini:49 paper_mini:50 medium:49 > gpurun_out/r2i_acc.jsonl 2> gpurun_out/r2i_acc.err
python -c "
import json
for l in open('gpurun_out/r2i_acc.jsonl'):
    d=json.loads(l); print(d['workload'], d['refresh_bits'], '%.3e'%d['max_abs_dw'], '%.2e'%d['max_abs_dauc'], round(d['seconds'],1))
"
tail -3 gpurun_out/r2i_acc.err
