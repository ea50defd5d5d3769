#!/bin/bash
# K1t: apply/smoother probe, then one ncu --set full capture (with source) of MODE 0 and MODE 1 on C4
mkdir -p gpurun_out
TAG=${TAG:-r02c}
: > gpurun_out/probe_$TAG.log
for V in ${VARIANTS:-"X=1"}; do
  echo "== $V" >> gpurun_out/probe_$TAG.log
  env $V PROBE_SMOOTH=1 PROBE_SOLVE=${PROBE_SOLVE:-1} timeout 300 python tools/probe.py ${PROBES:-C4} >> gpurun_out/probe_$TAG.log 2>&1
done
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
  -k regex:stencil2 -o gpurun_out/${TAG}_m0 -f python tools/ncu_apply.py C4 2 > gpurun_out/ncu_${TAG}_m0.log 2>&1
NCU_SMOOTH=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 -s 1 \
  -k regex:stencil2 -o gpurun_out/${TAG}_m1 -f python tools/ncu_apply.py C4 1 > gpurun_out/ncu_${TAG}_m1.log 2>&1
fi
