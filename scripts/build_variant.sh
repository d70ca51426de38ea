#!/bin/bash
# Build a variant of libmma.so with extra nvcc defines for relay.cu (probe use only):
#   scripts/build_variant.sh OUT.so -DMACRO=VALUE ...   (after the default build: reuses build/*.o)
set -e
out=$1; shift
R=paper_2512_16056_b200
mkdir -p $(dirname $out)
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I include \
    --expt-relaxed-constexpr --extended-lambda "$@" -c $R/csrc/kernels/relay.cu -o $out.relay.o
objs=$(ls $R/build/*.o | grep -v '/relay.o$')
nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o $out $objs $out.relay.o -ldl -lpthread -lrt
rm -f $out.relay.o
