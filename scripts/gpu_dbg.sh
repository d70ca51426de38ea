#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=60000
timeout 1500 compute-sanitizer --tool racecheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r02/i_race_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02/i_race_multi.log
export MMA_SPIN_TIMEOUT_MS=8000
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02/i_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02/i_all.log
tail -5 gpurun_out/r02/i_race_multi.log; tail -8 gpurun_out/r02/i_all.log
