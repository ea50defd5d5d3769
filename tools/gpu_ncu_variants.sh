#!/bin/bash
# full ncu capture of one finest-level apply of $CFG under each env variant in $VARIANTS
mkdir -p gpurun_out
CFG=${CFG:-C2}
for V in $VARIANTS; do
  tag=$(echo $V | tr '=' '_')
  env $V python tools/ncu_apply.py $CFG 3 > gpurun_out/ncu_$tag.log 2>&1 && \
  env $V timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
    -k regex:'apply|cart|plane|dline|dg_|stencil' -o gpurun_out/${TAG:-v}_${CFG}_$tag -f python tools/ncu_apply.py $CFG 3 >> gpurun_out/ncu_$tag.log 2>&1
done
