#!/bin/bash
# Profiling recipe (B200_PROFILING.md) — run under gpurun.  Outputs in gpurun_out/.
set -x
APP=${1:-cf4}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${APP}.csv \
    python bench.py --app $APP --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:extend -c ${2:-3} -o gpurun_out/prof_${APP} -f \
    python bench.py --app $APP --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
