mkdir -p gpurun_out
HELR_NVCC_DEFS="-DHELR_HOIST_MINB=5" python -c "from paper_2406_13221_b200 import build; build.build(force=True)" > gpurun_out/knob_build.log 2>&1
echo "== MINB=5"; timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
python -c "from paper_2406_13221_b200 import build; build.build(force=True)" > gpurun_out/knob_build.log 2>&1
echo "== default (MINB=4)"; timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_ntt_tma.py tests/test_gpu_fused.py -q -m gpu -s 2>&1 | grep -E "max .dw|passed|failed|^E  " | head
for o in "--work-levels 7" "--work-levels 14 --dnum 6"; do echo "== $o"; timeout 900 python tools/bootstrap_train_bench.py $o 2>&1 | tail -1; done
