#!/bin/bash
# round-2: new parity tests on the GPU
python -m pytest tests/test_gpu_dropin.py tests/test_gpu_trainer_residue.py -q -m gpu -rA 2>&1 | tail -40 > gpurun_out/r2b_dropin.log
python -m pytest tests/test_gpu_train.py -q -m gpu -s 2>&1 | grep -E "max \||passed|failed|Error" > gpurun_out/r2b_train.log
cat gpurun_out/r2b_dropin.log | tail -15; cat gpurun_out/r2b_train.log
