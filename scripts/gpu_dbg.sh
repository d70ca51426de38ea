#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02/q_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02/q_all.log
tail -8 gpurun_out/r02/q_all.log
