#!/bin/bash
# FP64 DFMA / DMMA peaks and compute-sanitizer runs (memcheck, racecheck, synccheck)
mkdir -p gpurun_out
./tools/fp64_peak.bin > gpurun_out/fp64_peak.json 2>&1
./tools/dmma_peak.bin > gpurun_out/dmma_peak.json 2>&1
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$T.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$T.log
done
