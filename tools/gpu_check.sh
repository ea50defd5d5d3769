#!/bin/bash
# One GPU verification pass: parity tests, bench line.  TESTS overrides the test selection.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest ${TESTS:-tests} -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
fi
