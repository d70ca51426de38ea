#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r02/e_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02/e_multi.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02/e_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02/e_all.log
tail -30 gpurun_out/r02/e_multi.log; tail -15 gpurun_out/r02/e_all.log
