#!/bin/bash
# round 2, call A: serialised-launch tests, smoke under ncu, then the whole GPU tier
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=${MMA_SPIN_TIMEOUT_MS:-8000}
timeout 900 python -m pytest tests/test_gpu_serialized.py -q -x > gpurun_out/r02/serialized.log 2>&1; echo "rc=$?" >> gpurun_out/r02/serialized.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/smoke_ncu.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r02/smoke_ncu.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_gpu.log
tail -3 gpurun_out/r02/serialized.log gpurun_out/r02/smoke_ncu.log; tail -30 gpurun_out/r02/pytest_gpu.log
