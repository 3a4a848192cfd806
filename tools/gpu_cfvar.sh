#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2; do
  GPM_CF_VARIANT=$v GPM_TRACE=1 timeout 300 python tools/prof_target.py cf4 5 > gpurun_out/trace_cf4_v$v.log 2>&1
done
