#!/bin/bash
# bench line + ncu launch list of the bench + full ncu captures of the apply kernels.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pre_ncu.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/${TAG}_launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launch.log 2>&1
for C in ${CONFIGS:-C2 C3 C4}; do
  python tools/ncu_apply.py $C 3 > gpurun_out/apply_$C.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
    -k regex:'apply|cart' -o gpurun_out/${TAG}_apply_$C -f python tools/ncu_apply.py $C 3 \
    >> gpurun_out/apply_$C.log 2>&1
done
ls -la gpurun_out
