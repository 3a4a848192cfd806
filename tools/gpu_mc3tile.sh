#!/bin/bash
# 3-MC block-kernel tile size sweep (GPM_MC3_TILE keys per CTA tile)
mkdir -p gpurun_out
for t in 1024 2048 4096 8192; do
  GPM_MC3_TILE=$t GPM_TRACE=1 timeout 600 python tools/prof_target.py mc3 2 > gpurun_out/trace_mc3_$t.log 2>&1
done
