# full ncu capture of the 4 NTT passes of one fp64 forward + inverse call (tools/ntt_micro.py --once);
# the report is reduced to text on the box (it embeds the module: too large to bring back)
python tools/ntt_micro.py --once && \
ncu --profile-from-start off --set full --clock-control none --import-source on -o /tmp/ntt_full python tools/ntt_micro.py --once > gpurun_out/ncu_ntt.log 2>&1; tail -2 gpurun_out/ncu_ntt.log
python tools/ncu_brief.py /tmp/ntt_full.ncu-rep > gpurun_out/ntt_brief.txt 2>&1
for i in 0 1 2 3; do
  ncu -i /tmp/ntt_full.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > gpurun_out/ntt_src_$i.csv 2>/dev/null
done
gzip -f gpurun_out/ntt_src_*.csv
