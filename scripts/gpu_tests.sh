#!/bin/bash
# Run the GPU tier under hard timeouts; results land in gpurun_out/.
mkdir -p gpurun_out
export MMA_SPIN_TIMEOUT_MS=${MMA_SPIN_TIMEOUT_MS:-8000}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${GPU_TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/smoke.log; tail -40 gpurun_out/pytest_gpu.log
