#!/bin/bash
# iteration pass: GPU tests (optionally -k), then one workload's bench line
mkdir -p gpurun_out
timeout ${PYT:-1200} python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for app in ${APPS:-mc4}; do
  timeout 900 python bench.py --app $app --no-sub --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/bench_$app.json 2> gpurun_out/bench_$app.err
  echo "rc=$?" >> gpurun_out/bench_$app.err
done
[ -n "$TRACE" ] && GPM_TRACE=1 timeout 300 python tools/prof_target.py $TRACE 2 > gpurun_out/trace.log 2>&1
ls gpurun_out
