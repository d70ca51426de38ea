#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 1500 python -m pytest tests/test_gpu_forward_log.py tests/test_gpu_parity.py tests/test_gpu_serialized.py tests/test_gpu_fault.py -q -x > gpurun_out/r02/p_fwd.log 2>&1; echo "rc=$?" >> gpurun_out/r02/p_fwd.log
tail -25 gpurun_out/r02/p_fwd.log
