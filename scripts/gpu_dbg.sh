#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/n_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02/n_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02/n_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02/n_all.log
tail -2 gpurun_out/r02/n_smoke.log; tail -6 gpurun_out/r02/n_all.log
