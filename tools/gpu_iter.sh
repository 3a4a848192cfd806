#!/bin/bash
# iteration run: full GPU test suite + bench lines of the named apps (no CPU baseline)
mkdir -p gpurun_out
timeout ${PYT:-1500} python -m pytest tests -m gpu -q ${PYK:+-k "$PYK"} ${PYX:--x} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for spec in ${RUNS:-"cf4" "tc" "fsm"}; do
  IFS=: read app envs <<< "$spec"
  env $envs timeout 600 python bench.py --app $app --no-sub --no-cpu-baseline > "gpurun_out/bench_${app}_${envs}.json" 2>&1
done
