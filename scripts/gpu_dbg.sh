#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
MMA_MULTI_CASES=300 timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r02/o_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02/o_multi.log
tail -25 gpurun_out/r02/o_multi.log
