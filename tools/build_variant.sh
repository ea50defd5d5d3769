#!/bin/bash
# build paper_1611_03029_b200/libfem_$1.so: kernels_stencil.cu recompiled with the given -D flags, the
# other objects from the main build (development aid for A/B timing)
set -e
cd "$(dirname "$0")/.."
P=paper_1611_03029_b200
T=$1; shift
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr "$@" -I include -c $P/csrc/kernels_stencil.cu -o /tmp/ks_$T.o
objs=$(ls $P/build/*.o | grep -v kernels_stencil)
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs /tmp/ks_$T.o -o $P/libfem_$T.so -lcudart -ldl
