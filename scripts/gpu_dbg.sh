#!/bin/bash
mkdir -p gpurun_out/r02
SWEEP_C=1048576,2097152 SWEEP_S=8,16,32 timeout 900 python scripts/sweep_group.py 8388608 > gpurun_out/r02/sweep_S.jsonl 2>&1
SWEEP_C=1048576 SWEEP_S=8,32 MMA_NO_BATCH_MEMOP=1 timeout 900 python scripts/sweep_group.py 8388608 > gpurun_out/r02/sweep_nobatch.jsonl 2>&1
cat gpurun_out/r02/sweep_S.jsonl gpurun_out/r02/sweep_nobatch.jsonl | grep -v "^\[" | cut -c1-150
