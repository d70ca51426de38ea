#!/bin/bash
# compute-sanitizer over the relay / zero-copy / dynamic / multi-process paths (small cases);
# logs in gpurun_out/
mkdir -p gpurun_out
export MMA_SPIN_TIMEOUT_MS=60000 MMA_RANDOM_CASES=${MMA_RANDOM_CASES:-40} MMA_RANDOM_CASES_VGPU=${MMA_RANDOM_CASES_VGPU:-40}
SEL='test_h2d_contiguous and (3158073 or 2101248) or test_d2h_contiguous and 3158073 or test_misaligned or test_dynamic or test_kv_fetch_h2d and 272 or test_kv_offload_d2h and 272 or test_random or test_two_processes or test_share_through or test_ring_kinds or test_two_fetches or test_mixed_directions or peer or across_gpus or two_targets or test_joint_plan or behind_its_own'
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_dynamic.py tests/test_gpu_segments.py \
      tests/test_gpu_random.py tests/test_gpu_mp.py tests/test_gpu_multi.py tests/test_gpu_peer.py -m gpu -q -x -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3
done
