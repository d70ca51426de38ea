#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02/t_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02/t_all.log
timeout 900 python bench.py > gpurun_out/r02/t_bench.json 2> gpurun_out/r02/t_bench.err
tail -4 gpurun_out/r02/t_all.log
python -c "
import json
d=json.loads(open('gpurun_out/r02/t_bench.json').read().strip().splitlines()[-1])
print(d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('error'), d['engine'])"
