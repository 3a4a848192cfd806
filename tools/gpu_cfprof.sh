#!/bin/bash
# cf4 local-row kernels: timeline (GPM_TRACE) + ncu --set full of the two kernels
mkdir -p gpurun_out
GPM_TRACE=1 timeout 300 python tools/prof_target.py cf4 3 > gpurun_out/trace_cf4.log 2>&1
SPEC="cf4:local_small:1:1 cf4:local_big:1:1" bash tools/gpu_ncu.sh
for f in gpurun_out/full_cf4_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>&1; done
