#!/bin/bash
mkdir -p gpurun_out/r02
timeout 1200 python bench.py --workload wake --steps 3 --warmup 3 > gpurun_out/r02/m_wake.json 2> gpurun_out/r02/m_wake.err
timeout 900 python bench.py --workload contention --steps 3 --warmup 3 > gpurun_out/r02/m_contention.json 2> gpurun_out/r02/m_contention.err
timeout 1500 python scripts/sweep_sizes.py > gpurun_out/r02/m_sweep_sizes.jsonl 2> gpurun_out/r02/m_sweep_sizes.err
for f in gpurun_out/r02/m_wake.json gpurun_out/r02/m_contention.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('value'), d.get('ms_per_step'), d.get('native'), d.get('per_call_ledger'), d.get('error'))"; done
wc -l gpurun_out/r02/m_sweep_sizes.jsonl; tail -3 gpurun_out/r02/m_sweep_sizes.err
