mkdir -p gpurun_out
for C in C2 C3; do
python tools/solve_breakdown.py $C > gpurun_out/bd_$C.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/bd_$C.csv python tools/solve_breakdown.py $C >> gpurun_out/bd_$C.log 2>&1
done
