#!/bin/bash
# end-of-round evidence: bench line, ncu launch list of the bench (C4 only), one ncu --set full of
# the K1t apply (traffic) and the fused smoother step, C4 solve breakdown
mkdir -p gpurun_out
TAG=${TAG:-r02f}
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --others "" --no-hdg > gpurun_out/bench_pre_ncu.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/${TAG}_launches_bench_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --others "" --no-hdg > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
  -k regex:stencil2 -o gpurun_out/${TAG}_m0 -f python tools/ncu_apply.py C4 2 > gpurun_out/ncu_${TAG}_m0.log 2>&1
NCU_SMOOTH=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 -s 1 \
  -k regex:stencil2 -o gpurun_out/${TAG}_m1 -f python tools/ncu_apply.py C4 1 > gpurun_out/ncu_${TAG}_m1.log 2>&1
python tools/solve_breakdown.py C4 > gpurun_out/bd_C4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/bd_C4.csv python tools/solve_breakdown.py C4 >> gpurun_out/bd_C4.log 2>&1
