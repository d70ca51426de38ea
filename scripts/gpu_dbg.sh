#!/bin/bash
mkdir -p gpurun_out/r02
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/j_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02/j_smoke.log
for i in 1 2; do timeout 900 python bench.py > gpurun_out/r02/j_bench_$i.json 2> gpurun_out/r02/j_bench_$i.err; done
timeout 600 python bench.py --impl reference > gpurun_out/r02/j_ref.json 2> gpurun_out/r02/j_ref.err
timeout 900 python bench.py --workload contig --bytes 67108864 --chunk 1048576 --loopback 1 --hop 1 --steps 20 --warmup 3 > gpurun_out/r02/j_config1_loopback.json 2> gpurun_out/r02/j_config1.err
tail -2 gpurun_out/r02/j_smoke.log
for f in gpurun_out/r02/j_bench_1.json gpurun_out/r02/j_bench_2.json gpurun_out/r02/j_ref.json gpurun_out/r02/j_config1_loopback.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('error'))"; done
