python bench.py --steps 100 --warmup 5 --cpu-iters 0 --profile-steps 1 > gpurun_out/e2e_new.json 2>gpurun_out/e2e_new.err
python -c "import json;d=json.load(open('gpurun_out/e2e_new.json'));print(round(d['value'],2), round(d['e2e']['value'],2))"
python -m pytest tests/test_gpu_train.py -x -q 2>&1 | tail -1
