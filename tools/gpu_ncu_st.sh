#!/bin/bash
# K1t stencil: parity tests, apply probe, one ncu --set full capture of the C4 apply kernel
mkdir -p gpurun_out
TAG=${TAG:-r02a}
timeout 400 python -m pytest ${TESTS:-tests/test_gpu_stencil.py} -m gpu -x -q -p no:cacheprovider --timeout 120 > gpurun_out/pytest_quick.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_quick.log
: > gpurun_out/probe.log
for V in ${VARIANTS:-"X=1"}; do
  echo "== $V" >> gpurun_out/probe.log
  env $V PROBE_SOLVE=${PROBE_SOLVE:-0} timeout 200 python tools/probe.py ${PROBES:-C4} >> gpurun_out/probe.log 2>&1
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
    -k regex:"${NCU_K:-stencil2}" -o gpurun_out/${TAG}_apply_C4 -f python tools/ncu_apply.py C4 2 \
    > gpurun_out/ncu_${TAG}.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_${TAG}.log
fi
