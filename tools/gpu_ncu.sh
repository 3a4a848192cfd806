#!/bin/bash
# ncu --set full of named kernels: SPEC="target:regex:skip:count ..."
mkdir -p gpurun_out
for spec in $SPEC; do
  IFS=: read t rx sk ct <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s ${sk:-0} -c ${ct:-2} -o gpurun_out/full_${t}_${rx} -f \
      python tools/prof_target.py $t 2 > gpurun_out/ncu_${t}_${rx}.log 2>&1
done
ls -la gpurun_out
