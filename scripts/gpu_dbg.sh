#!/bin/bash
mkdir -p gpurun_out/r02
for cfg in "MMA_ZC_CTAS=16" "MMA_ZC_CTAS=4" "MMA_ZC_CTAS=8" "MMA_ZC_CTAS=32" "MMA_UNIT_BYTES=2097152" "MMA_UNIT_BYTES=131072" "MMA_ZC_CTAS=4 MMA_UNIT_BYTES=4194304"; do
  env $cfg timeout 600 python bench.py --quick --no-verify --steps 5 --warmup 3 > gpurun_out/r02/w.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/r02/w.json').read().strip().splitlines()[-1])
print('$cfg', d.get('value'), d['per_direction'], (d.get('roofline') or {}).get('frac'))"
done
