#!/bin/bash
# libfem_$1.so with hdg.cu recompiled with the given -D flags (development aid)
set -e
cd "$(dirname "$0")/.."
P=paper_1611_03029_b200
T=$1; shift
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr "$@" -I include -c $P/csrc/hdg.cu -o /tmp/hdg_$T.o
objs=$(ls $P/build/*.o | grep -v '/hdg.o')
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs /tmp/hdg_$T.o -o $P/libfem_$T.so -lcudart -ldl
