python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/shard_tests.log 2>&1; tail -3 gpurun_out/shard_tests.log
python bench.py --workload paper_full --steps 2 --warmup 3 --no-e2e --cpu-iters 0 --profile-steps 1 > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; tail -c 1500 gpurun_out/full_bench.json; tail -3 gpurun_out/full_bench.err
