#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_gpu_numa.py tests/test_gpu_random.py -q -x > gpurun_out/r02/d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02/d_tests.log
for lanes in 1 2; do MMA_HOP_LANES=$lanes timeout 900 python scripts/sweep_group.py 0 4194304 8388608 >> gpurun_out/r02/sweep_lanes.jsonl 2>> gpurun_out/r02/sweep_lanes.err; done
tail -5 gpurun_out/r02/d_tests.log; tail -3 gpurun_out/r02/sweep_lanes.err
