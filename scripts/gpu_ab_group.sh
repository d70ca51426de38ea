#!/bin/bash
# A/B of piece grouping in the zero-copy kernels (variants/libmma_nogroup.so: built with
# -DMMA_NO_GROUP) under duplex load; rows in gpurun_out/ab.jsonl. Build the variant first
# (after the default build, from the repo root):
#   R=paper_2512_16056_b200; mkdir -p variants
#   nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I include \
#     --expt-relaxed-constexpr --extended-lambda -DMMA_NO_GROUP -c $R/csrc/kernels/zerocopy.cu -o variants/zc.o
#   nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o variants/libmma_nogroup.so \
#     $(ls $R/build/*.o | grep -v '/zerocopy.o$') variants/zc.o -ldl -lpthread -lrt
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
