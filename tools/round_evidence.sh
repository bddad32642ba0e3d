# Full bench line + reference arm + profile evidence (tools/ncu_evidence.sh) for TAG
TAG=${1:-r01}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
bash tools/ncu_evidence.sh $TAG > gpurun_out/evidence_$TAG.log 2>&1
# brief of the full captures (the .ncu-rep embeds the whole module; keep the text)
python tools/ncu_brief.py gpurun_out/full_$TAG.ncu-rep > gpurun_out/full_$TAG.txt 2>&1
rm -f gpurun_out/full_$TAG.ncu-rep
tail -c 600 gpurun_out/bench_$TAG.json
# every launch of one step under --set full -> per-kernel pipe / issue / occupancy table
python tools/profile_step.py > /dev/null 2>&1 && \
ncu -f --profile-from-start off --set full --clock-control none -o /tmp/fullstep_$TAG python tools/profile_step.py > gpurun_out/ncu_fullstep_$TAG.log 2>&1
python tools/ncu_table.py /tmp/fullstep_$TAG.ncu-rep --md gpurun_out/full_table_$TAG.md > /dev/null 2>&1
python tools/ncu_brief.py /tmp/fullstep_$TAG.ncu-rep > gpurun_out/full_brief_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
