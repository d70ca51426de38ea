#!/bin/bash
mkdir -p gpurun_out/r02
bash scripts/sanitize.sh > gpurun_out/r02/v_sanitize.txt 2>&1
MMA_RANDOM_CASES=2000 MMA_RANDOM_SEED=99 MMA_SPIN_TIMEOUT_MS=8000 timeout 1800 python -m pytest tests/test_gpu_random.py -q -x > gpurun_out/r02/v_soak.log 2>&1; echo "rc=$?" >> gpurun_out/r02/v_soak.log
MMA_MULTI_CASES=500 MMA_SPIN_TIMEOUT_MS=8000 timeout 1800 python -m pytest tests/test_gpu_multi.py -q -x -k random > gpurun_out/r02/v_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02/v_multi.log
cat gpurun_out/r02/v_sanitize.txt; tail -3 gpurun_out/r02/v_soak.log; tail -3 gpurun_out/r02/v_multi.log
