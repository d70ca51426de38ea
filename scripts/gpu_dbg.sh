#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 300 ./scripts/probe/probe_relay bulk > gpurun_out/r02/probe_relay_bulk.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_bulk.py -q -x > gpurun_out/r02/u_bulk.log 2>&1; echo "rc=$?" >> gpurun_out/r02/u_bulk.log
cat gpurun_out/r02/probe_relay_bulk.txt; tail -15 gpurun_out/r02/u_bulk.log
