#!/bin/bash
# A/B library variants (paper_1911_06969_b200/libgpm_<V>.so) on one workload:
# VARS="A B" TGT=mc4 bash tools/gpu_variants.sh
mkdir -p gpurun_out
for v in ${VARS:-A B}; do
  for r in 1 2; do
    GPM_LIB_VARIANT=libgpm_$v.so timeout 300 python tools/prof_target.py ${TGT:-mc4} 3 >> gpurun_out/var_$v.log 2>&1
  done
done
tail -n 3 gpurun_out/var_*.log
