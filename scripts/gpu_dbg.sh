#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_gpu_dynamic.py -q -x > gpurun_out/r02/l_dyn.log 2>&1; echo "rc=$?" >> gpurun_out/r02/l_dyn.log
timeout 600 python scripts/probe_background.py > gpurun_out/r02/probe_background.jsonl 2>&1
tail -5 gpurun_out/r02/l_dyn.log; cat gpurun_out/r02/probe_background.jsonl
