#!/bin/bash
# cluster NTT variants: parity (ntt) + microbench
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "ntt or rotsum or mul_relin" > gpurun_out/r2f_tests.log 2>&1; tail -2 gpurun_out/r2f_tests.log
for v in "0 0 0" "1 0 0" "1 0 1" "1 1 1"; do
  set -- $v
  HELR_NTT_CLUSTER=$1 HELR_NTT_BULK=$2 HELR_NTT_XASYNC=$3 timeout 300 python tools/ntt_micro.py --batch 16 > gpurun_out/r2f_micro.json 2>&1
  echo "cl=$1 bulk=$2 xasync=$3 $(python -c "import json;d=json.load(open('gpurun_out/r2f_micro.json'));print({k:v['us_per_limb'] for k,v in d.items() if isinstance(v,dict)})")"
done
