#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for V in FEM_PDL=1 FEM_PDL=0; do
  echo "== $V" >> gpurun_out/probe.log
  env $V timeout 300 python tools/probe_levels.py >> gpurun_out/probe.log 2>&1
  env $V PROBE_SOLVE=1 timeout 600 python tools/probe.py C2 C3 C4 >> gpurun_out/probe.log 2>&1
done
