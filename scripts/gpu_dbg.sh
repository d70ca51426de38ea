#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_gpu_logs.py tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_trace.py tests/test_gpu_fault.py tests/test_gpu_segments.py -q -x -s > gpurun_out/r02/c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02/c_tests.log
timeout 600 python scripts/sweep_ring.py > gpurun_out/r02/c_sweep_ring.jsonl 2> gpurun_out/r02/c_sweep_ring.err
tail -30 gpurun_out/r02/c_tests.log; cat gpurun_out/r02/c_sweep_ring.jsonl
