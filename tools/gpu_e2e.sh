python -m pytest tests/test_gpu_train.py -x -q -m gpu -k "host_streamed or toy" > gpurun_out/e2e_tests.log 2>&1; tail -2 gpurun_out/e2e_tests.log
python bench.py --steps 200 --cpu-iters 100 > gpurun_out/e2e_bench.json 2> gpurun_out/e2e_bench.err
python -c "import json;d=json.load(open('gpurun_out/e2e_bench.json'));print(d['value'],d['ms_per_step'],d['e2e'], d['cpu_baseline'])"
