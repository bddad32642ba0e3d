# Build-time knob sweep on the GPU box: rebuild with each HELR_NVCC_DEFS and time 100 steps
for defs in "-DHELR_NTT_EPI_UNROLL=8" "-DHELR_NTT_EPI_UNROLL=2" ""; do
  HELR_NVCC_DEFS="$defs" python -m paper_2406_13221_b200.build --force > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 --profile-steps 1 > gpurun_out/knob.json 2>/dev/null
  python - "$defs" <<'PY'
import json, sys; d = json.load(open("gpurun_out/knob.json"))
print(repr(sys.argv[1]), round(d["value"], 2), round(d["kernels"]["ntt"]["ms"], 3))
PY
done
