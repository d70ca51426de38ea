#!/bin/bash
# round 2, call B: the new tests and the modules touched by the waves / capture lanes
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=${MMA_SPIN_TIMEOUT_MS:-8000}
timeout 1500 python -m pytest tests/test_gpu_serialized.py tests/test_gpu_validate.py tests/test_gpu_graph.py \
  tests/test_gpu_parity.py tests/test_gpu_trace.py tests/test_gpu_fault.py -q -s > gpurun_out/r02/b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02/b_tests.log
timeout 600 python scripts/sweep_ring.py > gpurun_out/r02/b_sweep_ring.jsonl 2> gpurun_out/r02/b_sweep_ring.err
tail -25 gpurun_out/r02/b_tests.log; cat gpurun_out/r02/b_sweep_ring.jsonl | head -40
