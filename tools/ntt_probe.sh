# NTT microbenchmark, then tests + quick bench
python tools/ntt_micro.py > gpurun_out/ntt_micro.json 2>&1; cat gpurun_out/ntt_micro.json
bash tools/gpu_quick.sh
