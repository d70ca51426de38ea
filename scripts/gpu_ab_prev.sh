#!/bin/bash
# bench A/B of the current libmma.so against variants/libmma_prevbulk.so (the previous
# commit's zerocopy.cu compiled against the current objects: nvcc -c <old zerocopy.cu>, then
# link with paper_2512_16056_b200/build/*.o minus zerocopy.o, as in scripts/gpu_ab_group.sh)
L=paper_2512_16056_b200/libmma.so
cp $L /tmp/new.so
for rep in 1 2; do for v in new prev; do
  if [ $v = new ]; then cp /tmp/new.so $L; else cp variants/libmma_prevbulk.so $L; fi
  timeout 600 python bench.py --steps 3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['value'],d['per_direction']['h2d_gbps'],d['per_direction']['d2h_gbps'],d['duplex']['gbps'],d['path_roofline']['pcie_solo'])"
done; done
cp /tmp/new.so $L
