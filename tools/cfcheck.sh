#!/bin/bash
# CF kernel variants: parity tests + cf4/tc timings per GPM_CF_LONG / GPM_CF_STREAM
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in ${VARIANTS:-"GPM_CF_STREAM=1" "GPM_CF_LONG=2" "GPM_CF_LONG=4" "GPM_CF_LONG=8" "GPM_CF_LONG=16"}; do
  for app in ${CFAPPS:-cf4 tc}; do
    env $m timeout 300 python bench.py --app $app --no-sub --no-cpu-baseline > gpurun_out/bench_${app}_${m}.json 2>&1
  done
done
