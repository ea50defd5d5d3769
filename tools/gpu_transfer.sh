#!/bin/bash
# node-grid CG transfers: parity tests, A/B timing of the register-cap variants against the
# element form (finest C4 / C2 transfers and the solves), one ncu --set full of each new kernel
mkdir -p gpurun_out
python -m pytest tests/test_gpu_cg.py tests/test_gpu_slabs.py -m gpu -x -q -k "transfer" > gpurun_out/pytest_transfer.log 2>&1
tail -3 gpurun_out/pytest_transfer.log
: > gpurun_out/transfer.log
for L in ${LIBS:-libfem}; do
  echo "== $L" >> gpurun_out/transfer.log
  FEM_LIB=paper_1611_03029_b200/$L.so PROBE_TRANSFER=1 PROBE_SOLVE=1 timeout 300 python tools/probe.py C4 C2 >> gpurun_out/transfer.log 2>&1
done
echo "== element form" >> gpurun_out/transfer.log
FEM_GT_MIN_CELLS=1000000000 PROBE_TRANSFER=1 PROBE_SOLVE=1 timeout 300 python tools/probe.py C4 C2 >> gpurun_out/transfer.log 2>&1
for M in ${MINS:-512 32768}; do
  echo "== libfem FEM_GT_MIN_CELLS=$M" >> gpurun_out/transfer.log
  FEM_GT_MIN_CELLS=$M PROBE_SOLVE=1 timeout 300 python tools/probe.py C4 C2 >> gpurun_out/transfer.log 2>&1
done
cat gpurun_out/transfer.log
if [ -n "$NCU" ]; then
  PROBE_TRANSFER=1 PROBE_SOLVE=0 timeout 600 ncu --set full --clock-control none --import-source on -c 2 \
    -k regex:grid_kernel -s 2 -o gpurun_out/${TAG:-r02l}_gt -f python tools/probe.py C4 > gpurun_out/ncu_gt.log 2>&1
fi
