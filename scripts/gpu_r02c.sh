#!/bin/bash
# last-code evidence: sanitizer tiers, a random soak, GPU-tier test durations; logs in gpurun_out/
mkdir -p gpurun_out
bash scripts/sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1
for seed in 41 42; do
  MMA_RANDOM_SEED=$seed MMA_RANDOM_CASES=1000 MMA_RANDOM_CASES_VGPU=3000 timeout 900 \
    python -m pytest tests/test_gpu_random.py -m gpu -q -x 2>&1 | tail -1 | sed "s/^/seed $seed: 4000 cases, /" >> gpurun_out/soak.txt
done
cat gpurun_out/sanitize_summary.txt gpurun_out/soak.txt
