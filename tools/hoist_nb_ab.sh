for nb in 4 2 8; do
HELR_HOIST_NB=$nb python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 --profile-steps 1 > gpurun_out/nb$nb.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/nb$nb.json'));print($nb, round(d['value'],2), round(d['kernels']['ks_inner']['ms'],3))"
done
