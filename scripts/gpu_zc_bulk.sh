#!/bin/bash
# the cp.async.bulk zero-copy kernel (MMA_ZC_BULK=1): parity modules, duplex probe, bench; gpurun_out/
mkdir -p gpurun_out
export MMA_SPIN_TIMEOUT_MS=8000
MMA_ZC_BULK=1 timeout 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_dynamic.py tests/test_gpu_logs.py -m gpu -q -x > gpurun_out/zcbulk_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/zcbulk_tests.log
for v in 0 1; do
  MMA_ZC_BULK=$v timeout 600 python scripts/probe_duplex_grid.py ${GRIDS:-16,24} > gpurun_out/zcbulk_duplex_$v.jsonl 2>> gpurun_out/zcbulk_duplex.err; echo "probe $v rc=$?"; cat gpurun_out/zcbulk_duplex_$v.jsonl
done
MMA_ZC_BULK=1 timeout 900 python bench.py > gpurun_out/bench_zcbulk.json 2> gpurun_out/bench_zcbulk.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_zcbulk.json'));print(d['value'],d['per_direction'],d['roofline']['frac'],d['roofline']['kernel'],d['duplex'],d['e2e']['value'])"
