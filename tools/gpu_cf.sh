#!/bin/bash
# CF iteration: GPU parity tests touching k-CL + cf4 bench (local rows vs level-by-level) + trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
GPM_TRACE=1 timeout 300 python tools/prof_target.py cf4 3 > gpurun_out/trace_cf4.log 2>&1
timeout 600 python bench.py --app cf4 --no-sub --no-cpu-baseline > gpurun_out/bench_cf4_local.json 2>&1
