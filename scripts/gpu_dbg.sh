#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
for seed in 1001 1002 1003 1004 1005; do
  MMA_RANDOM_CASES=2000 MMA_RANDOM_SEED=$seed timeout 1200 python -m pytest tests/test_gpu_random.py -q -x > gpurun_out/r02/x_soak_$seed.log 2>&1; echo "seed $seed rc=$?"
done
for seed in 2001 2002; do
  MMA_MULTI_CASES=1000 MMA_RANDOM_SEED=$seed timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k random > gpurun_out/r02/x_multi_$seed.log 2>&1; echo "multi seed $seed rc=$?"
done
MMA_RELAY_BULK=1 MMA_RANDOM_CASES=1000 MMA_RANDOM_SEED=3001 timeout 1200 python -m pytest tests/test_gpu_random.py -q -x > gpurun_out/r02/x_soak_bulk.log 2>&1; echo "bulk soak rc=$?"
