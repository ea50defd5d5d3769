#!/bin/bash
# quick check: selected GPU tests + apply timings (probe) for a few configs under env variants
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_cg.py} -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_quick.log
: > gpurun_out/probe.log
for V in ${VARIANTS:-"X=1"}; do
  echo "== $V" >> gpurun_out/probe.log
  env $(echo $V | tr , " ") PROBE_SOLVE=${PROBE_SOLVE:-0} timeout 600 python tools/probe.py ${PROBES:-C2} >> gpurun_out/probe.log 2>&1
done
