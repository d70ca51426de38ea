#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_random.py -q -x > gpurun_out/r02/k_graph.log 2>&1; echo "rc=$?" >> gpurun_out/r02/k_graph.log
tail -15 gpurun_out/r02/k_graph.log
