#!/bin/bash
# ncu full capture: pipelined hoisted inner product (first launch of one step) + the per-thread kernel for contrast
python tools/profile_step.py > gpurun_out/pstep.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_ks_inner_pipe" -c 1 -o /tmp/hpipe python tools/profile_step.py > gpurun_out/ncu_hpipe.log 2>&1
tail -1 gpurun_out/ncu_hpipe.log
python tools/ncu_brief.py /tmp/hpipe.ncu-rep > gpurun_out/r2h_brief.txt 2>&1
ncu -i /tmp/hpipe.ncu-rep --page source --csv --print-source sass > gpurun_out/r2h_src.csv 2>/dev/null; gzip -f gpurun_out/r2h_src.csv
ncu -i /tmp/hpipe.ncu-rep --page details --csv > gpurun_out/r2h_details.csv 2>/dev/null
cat gpurun_out/r2h_brief.txt
