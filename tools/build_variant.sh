#!/bin/bash
# build paper_1611_03029_b200/libfem_$1.so: csrc/$SRC.cu (default kernels_stencil) recompiled with the
# given -D flags, the other objects from the main build (development aid for A/B timing)
set -e
cd "$(dirname "$0")/.."
P=paper_1611_03029_b200
S=${SRC:-kernels_stencil}
T=$1; shift
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr "$@" -I include -c $P/csrc/$S.cu -o /tmp/${S}_$T.o
objs=$(ls $P/build/*.o | grep -v "/$S.o")
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs /tmp/${S}_$T.o -o $P/libfem_$T.so -lcudart -ldl
