#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
MMA_TRACE=1 MMA_FAKE_HOST_NODES=2 MMA_FAKE_PATH_NODES=0,0,0,0,1,1,1,1 timeout 600 python scripts/probe_issue_paths.py 7 > gpurun_out/r02/pi_numa.jsonl 2> gpurun_out/r02/probe_issue_numa.err
timeout 1500 python -m pytest tests/test_gpu_numa.py tests/test_gpu_random.py -q -x > gpurun_out/r02/s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02/s_tests.log
cat gpurun_out/r02/pi_numa.jsonl; grep "\[mma\]" gpurun_out/r02/probe_issue_numa.err | tail -2; tail -3 gpurun_out/r02/s_tests.log
