# full ncu capture of the first hoisted inner-product launch of one paper_mini step, reduced to text on the box
python tools/profile_step.py > gpurun_out/pstep.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_ks_inner_hoisted" -c 1 -o /tmp/hoist python tools/profile_step.py > gpurun_out/ncu_hoist.log 2>&1
tail -2 gpurun_out/ncu_hoist.log
python tools/ncu_brief.py /tmp/hoist.ncu-rep > gpurun_out/hoist_brief.txt 2>&1
ncu -i /tmp/hoist.ncu-rep --page source --csv --print-source sass > gpurun_out/hoist_src.csv 2>/dev/null; gzip -f gpurun_out/hoist_src.csv
ncu -i /tmp/hoist.ncu-rep --page details --csv > gpurun_out/hoist_details.csv 2>/dev/null
