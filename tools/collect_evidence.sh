#!/bin/bash
# Copy one round_evidence.sh run from gpurun_out/ into profiles/ (tracked) and
# regenerate the summaries bench.py reads.  Usage: tools/collect_evidence.sh r02
TAG=${1:-r02}
G=gpurun_out; P=profiles
cp $G/bench_$TAG.json $P/${TAG}_bench.json
cp $G/bench_ref_$TAG.json $P/${TAG}_bench_reference.json
[ -s $G/bench_paper_full_$TAG.json ] && cp $G/bench_paper_full_$TAG.json $P/${TAG}_bench_paper_full.json
cp $G/step_launches_$TAG.csv $P/${TAG}_step_launches.csv
[ -s $G/step_launches_warm_$TAG.csv ] && cp $G/step_launches_warm_$TAG.csv $P/${TAG}_step_launches_warm.csv
cp $G/bench_launches_$TAG.csv $P/${TAG}_bench_launches.csv
python tools/ncu_summary.py $P/${TAG}_step_launches.csv --md $P/${TAG}_step_launches.md --traffic $P/ncu_traffic.json \
    --warm $P/${TAG}_step_launches_warm.csv \
    --title "$TAG: one Paper-mini iteration, every launch (ncu gpu__time_duration + DRAM bytes)" > /dev/null
python tools/ncu_summary.py $P/${TAG}_bench_launches.csv --md $P/${TAG}_bench_launches.md \
    --title "$TAG: launch list of python bench.py --steps 2 --warmup 3 (ncu gpu__time_duration)" > /dev/null
cp $G/full_table_$TAG.md $P/${TAG}_full_table.md
cp $G/full_$TAG.txt $P/${TAG}_top_kernels_brief.txt
cp $G/smoke_$TAG.log $P/${TAG}_smoke.log
[ -s $G/accuracy_$TAG.jsonl ] && cp $G/accuracy_$TAG.jsonl $P/${TAG}_accuracy.jsonl
[ -s $G/ntt_micro_$TAG.json ] && tail -1 $G/ntt_micro_$TAG.json > $P/${TAG}_ntt_micro.json
ls -la $P | grep ${TAG}_ | awk '{print $5, $9}'
