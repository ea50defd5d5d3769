#!/bin/bash
# round-2 profile set: bench line, ncu launch list of the bench command, one ncu --set full
# capture of the C4 apply kernel (K1t MODE 0) and of the fused Chebyshev launch (MODE 1),
# solve timings of C2, C3, C5
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv \
  --log-file gpurun_out/${TAG}_launches_bench_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
  -k regex:stencil2 -o gpurun_out/${TAG}_apply_C4 -f python tools/ncu_apply.py C4 2 > gpurun_out/${TAG}_ncu_apply.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled \
  -k regex:"stencil2_kernel<\(int\)4, \(int\)1" -c 1 -o gpurun_out/${TAG}_cheb_C4 -f python tools/solve_breakdown.py C4 \
  > gpurun_out/${TAG}_ncu_cheb.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
  -k regex:dg_apply -o gpurun_out/${TAG}_apply_C5 -f python tools/ncu_apply.py C5 2 > gpurun_out/${TAG}_ncu_c5.log 2>&1
PROBE_SOLVE=1 timeout 600 python tools/probe.py C2 C3 C5 > gpurun_out/${TAG}_probe.log 2>&1
