#!/bin/bash
# bench A/B of the direct zero-copy kernel form on one box (MMA_ZC_BULK=0 vector, 1 bulk)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 1 0; do
    MMA_ZC_BULK=$v timeout 900 python bench.py > gpurun_out/bench_ab_${v}_$rep.json 2> gpurun_out/bench_ab_${v}_$rep.err
    python -c "import json;d=json.load(open('gpurun_out/bench_ab_${v}_$rep.json'));print('bulk=$v rep $rep', d['value'],d['per_direction']['h2d_gbps'],d['per_direction']['d2h_gbps'],d['roofline']['kernel'],d['roofline']['frac'],d['duplex']['gbps'],d['e2e']['value'],d['path_roofline']['pcie_solo'],d['path_roofline']['cpu_dram_read_gbps'])"
  done
done
