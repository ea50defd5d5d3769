#!/bin/bash
# one full ncu capture of one kernel (NCU_K: regex on the mangled name) under ncu_apply.py
mkdir -p gpurun_out
python tools/ncu_apply.py ${NCU_C:-C4} 1 > gpurun_out/ncu_one_pre.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base mangled -k regex:"${NCU_K}" -s ${NCU_SKIP:-0} -c 1 \
  -o gpurun_out/${TAG:-one} -f python tools/ncu_apply.py ${NCU_C:-C4} 1 > gpurun_out/ncu_${TAG:-one}.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_${TAG:-one}.log
