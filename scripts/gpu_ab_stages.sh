#!/bin/bash
# bench + duplex probe of the bulk zero-copy kernel's stage count on one box
# (variants/libmma_st{3,4}.so built with -DMMA_ZC_STAGES=n; the default build has 6)
L=paper_2512_16056_b200/libmma.so
cp $L /tmp/st6.so
for rep in 1 2; do for v in 6 4 3; do
  if [ $v = 6 ]; then cp /tmp/st6.so $L; else cp variants/libmma_st$v.so $L; fi
  timeout 600 python bench.py --steps 3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('stages=$v', d['value'],d['per_direction']['h2d_gbps'],d['per_direction']['d2h_gbps'],d['duplex']['gbps'])"
  timeout 400 python scripts/probe_duplex_grid.py 16 2>/dev/null | tail -1 | sed "s/^/stages=$v /"
done; done
cp /tmp/st6.so $L
