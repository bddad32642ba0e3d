#!/bin/bash
# ncu full capture of the cluster NTT (fwd + inv, one call each)
export HELR_NTT_BULK=0
python tools/ntt_micro.py --once && \
ncu --profile-from-start off --set full --clock-control none --import-source on -o /tmp/ntt_cl python tools/ntt_micro.py --once > gpurun_out/r2e_ncu.log 2>&1; tail -2 gpurun_out/r2e_ncu.log
python tools/ncu_brief.py /tmp/ntt_cl.ncu-rep > gpurun_out/r2e_brief.txt 2>&1
for i in 0 1; do
  ncu -i /tmp/ntt_cl.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > gpurun_out/r2e_src_$i.csv 2>/dev/null
done
ncu -i /tmp/ntt_cl.ncu-rep --page details --csv > gpurun_out/r2e_details.csv 2>/dev/null
gzip -f gpurun_out/r2e_src_*.csv
cat gpurun_out/r2e_brief.txt
