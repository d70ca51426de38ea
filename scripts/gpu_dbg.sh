#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
MMA_TRACE=1 timeout 600 python scripts/probe_issue_paths.py 7 1 > gpurun_out/r02/pi.jsonl 2> gpurun_out/r02/probe_issue_trace3.err
timeout 1500 python -m pytest tests/test_gpu_segments.py tests/test_gpu_logs.py tests/test_gpu_random.py tests/test_gpu_graph.py tests/test_gpu_numa.py -q -x > gpurun_out/r02/r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02/r_tests.log
cat gpurun_out/r02/pi.jsonl; grep "\[mma\]" gpurun_out/r02/probe_issue_trace3.err | tail -3; tail -3 gpurun_out/r02/r_tests.log
