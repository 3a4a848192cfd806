#!/bin/bash
# A/B of library variants through bench.py (L2 flush, CUDA events): VARS="OLD NEW" APP=cf4
mkdir -p gpurun_out
for r in 1 2; do
  for v in ${VARS:-OLD NEW}; do
    GPM_LIB_VARIANT=libgpm_$v.so timeout 300 python bench.py --app ${APP:-cf4} --no-sub --no-cpu-baseline --steps ${STEPS:-20} > gpurun_out/ab_${v}_$r.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_${v}_$r.json')); print('$v', d['ms_per_step'], d['step_stats']['median_ms'], d['parity']['match'])"
  done
done
