#!/bin/bash
# A/B apply timings of libfem variants (FEM_LIB) on configs, plus optional ncu of each
mkdir -p gpurun_out
: > gpurun_out/ab.log
for L in ${LIBS:-paper_1611_03029_b200/libfem.so}; do
  for V in ${VARIANTS:-"X=1"}; do
    echo "== $L $V" >> gpurun_out/ab.log
    env $V FEM_LIB=$L PROBE_SOLVE=${PROBE_SOLVE:-0} timeout 300 python tools/probe.py ${PROBES:-C4} >> gpurun_out/ab.log 2>&1
  done
  if [ -n "$NCU" ]; then
    T=$(basename $L .so)
    env FEM_LIB=$L timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
      -k regex:"${NCU_K:-stencil2}" -o gpurun_out/${TAG:-ab}_$T -f python tools/ncu_apply.py ${NCU_C:-C4} 2 > gpurun_out/ncu_$T.log 2>&1
  fi
done
