#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_preload.py tests/test_gpu_hostmem.py tests/test_gpu_ledger.py -q > gpurun_out/r02/f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02/f_tests.log
timeout 900 python bench.py > gpurun_out/r02/f_bench.json 2> gpurun_out/r02/f_bench.err
timeout 600 python bench.py --workload contention --steps 3 --warmup 1 > gpurun_out/r02/f_contention.json 2> gpurun_out/r02/f_contention.err
tail -15 gpurun_out/r02/f_tests.log; tail -c 1500 gpurun_out/r02/f_bench.json; tail -3 gpurun_out/r02/f_bench.err; cat gpurun_out/r02/f_contention.json; tail -3 gpurun_out/r02/f_contention.err
