#!/bin/bash
# quick GPU iteration: parity tests + timings of the named workloads
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for t in ${TARGETS:-}; do timeout 300 python tools/prof_target.py $t 3 > gpurun_out/t_$t.txt 2>&1; done
for a in ${APPS:-}; do
  timeout 900 python bench.py --app $a ${BENCHARGS:-} > gpurun_out/bench_$a.json 2> gpurun_out/bench_$a.err; echo "rc=$?" >> gpurun_out/bench_$a.err
done
