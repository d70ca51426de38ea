#!/bin/bash
mkdir -p gpurun_out/r02
timeout 900 python bench.py > gpurun_out/r02/y_bench.json 2> gpurun_out/r02/y_bench.err
python -c "
import json
d=json.loads(open('gpurun_out/r02/y_bench.json').read().strip().splitlines()[-1])
print(d.get('value'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('host_cpu'), d.get('error'))"
tail -2 gpurun_out/r02/y_bench.err
