#!/bin/bash
# One GPU session: parity tests, smoke, the default bench line (cf4 + sub-records), reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout ${PYT:-1500} python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -z "$NOBENCH" ]; then
timeout 1500 python bench.py ${BENCHARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
fi
if [ -n "$REFARM" ]; then
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
fi
ls -la gpurun_out
