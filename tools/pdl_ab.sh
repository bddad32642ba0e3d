# A/B: programmatic dependent launch on (default) / off
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_train.py tests/test_gpu_shard.py -x -q 2>&1 | tail -1
for v in 1 0; do
HELR_PDL=$v python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 --profile-steps 1 > gpurun_out/pdl$v.json 2>gpurun_out/pdl$v.err
python - <<PY
import json; d=json.load(open("gpurun_out/pdl$v.json")); print("PDL=$v", round(d["value"], 2), {k: round(x["ms"], 3) for k, x in d["kernels"].items()})
PY
done
