# hoisted-kernel knobs after the interleaved prefetch (bench only)
mkdir -p gpurun_out
for defs in "-DHELR_HOIST_STAGES=2" "-DHELR_HOIST_STAGES=4" "-DHELR_HOIST_MINB=2" "-DHELR_HOIST_MINB=4"; do
  HELR_NVCC_DEFS="$defs" python -c "from paper_2406_13221_b200 import build; build.build(force=True)" > gpurun_out/knob_build.log 2>&1 || { echo "build failed: $defs"; tail -5 gpurun_out/knob_build.log; continue; }
  echo "== defs: [$defs]"
  timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
