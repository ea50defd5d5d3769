#!/bin/bash
# stencil parity tests with the main lib, then apply / smoother / solve probes of each lib variant
mkdir -p gpurun_out
TAG=${TAG:-ab}
timeout 600 python -m pytest ${TESTS:-tests/test_gpu_stencil.py} -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
: > gpurun_out/ab_$TAG.log
for L in ${LIBS}; do
  echo "== $L" >> gpurun_out/ab_$TAG.log
  FEM_LIB=paper_1611_03029_b200/$L PROBE_SMOOTH=1 PROBE_SOLVE=${PROBE_SOLVE:-1} timeout 300 python tools/probe.py ${PROBES:-C4} >> gpurun_out/ab_$TAG.log 2>&1
done
