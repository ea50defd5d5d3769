#!/bin/bash
# HDG parity tests, HDG layout probes (LIBS), then compute-sanitizer memcheck / racecheck / synccheck
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hdg.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_hdg2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hdg2.log
: > gpurun_out/hdg_probe2.log
for L in ${LIBS:-libfem.so}; do
  FEM_LIB=paper_1611_03029_b200/$L timeout 300 python tools/hdg_probe.py 64:4 50:5 84:3 42:6 126:2 31:8 >> gpurun_out/hdg_probe2.log 2>&1
done
if [ -z "$NO_SAN" ]; then
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$T.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$T.log
done
fi
