for v in ckks keyreg; do
echo "== $v"; HELR_LIB=$PWD/paper_2406_13221_b200/libhelr_$v.so timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
HELR_LIB=$PWD/paper_2406_13221_b200/libhelr_keyreg.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q -m gpu -x 2>&1 | tail -3
