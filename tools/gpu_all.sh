#!/bin/bash
# One GPU session: parity tests, smoke, bench of every workload, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for a in ${APPS:-cf4 tc mc3 mc4 fsm}; do
  timeout 900 python bench.py --app $a > gpurun_out/bench_$a.json 2> gpurun_out/bench_$a.err; echo "rc=$?" >> gpurun_out/bench_$a.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cf4.csv \
    python bench.py --app cf4 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
