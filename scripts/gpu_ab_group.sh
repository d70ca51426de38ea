#!/bin/bash
# A/B of piece grouping in the zero-copy kernels (variants/libmma_nogroup.so: built with
# -DMMA_NO_GROUP) under duplex load; rows in gpurun_out/ab.jsonl
mkdir -p gpurun_out
L=paper_2512_16056_b200/libmma.so
cp $L /tmp/new.so
for rep in 1 2; do
  for v in new old; do
    if [ $v = new ]; then cp /tmp/new.so $L; G=${GRIDS_NEW:-16,32}; else cp variants/libmma_nogroup.so $L; G=${GRIDS_OLD:-16,32}; fi
    echo "## $v rep $rep" >> gpurun_out/ab.jsonl
    timeout 600 python scripts/probe_duplex_grid.py $G >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
  done
done
cp /tmp/new.so $L
cat gpurun_out/ab.jsonl
