# usage: bash tools/knob_ab.sh "<nvcc defs A>" "<nvcc defs B>" ...   (run on the GPU box: rebuilds per variant)
mkdir -p gpurun_out
for defs in "$@"; do
  HELR_NVCC_DEFS="$defs" python -c "from paper_2406_13221_b200 import build; build.build(force=True)" > gpurun_out/knob_build.log 2>&1 || { echo "build failed: $defs"; tail -5 gpurun_out/knob_build.log; continue; }
  echo "== defs: [$defs]"
  timeout 300 python tools/ntt_micro.py --batch 16 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print({k:(v['us_per_limb'] if isinstance(v,dict) else v) for k,v in d.items()})"
  timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
# restore the default build
python -c "from paper_2406_13221_b200 import build; build.build(force=True)" > /dev/null 2>&1
