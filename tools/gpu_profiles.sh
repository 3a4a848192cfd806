#!/bin/bash
# Round profiling pass (B200_PROFILING.md recipe): launch list of the headline
# bench command + one ncu --set full capture of each workload's dominant kernel.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cf4.csv \
    python bench.py --app cf4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for spec in "cf4:edge_chunk:0:1" "tc:edge_chunk:0:1" "mc3:mc3_warp:0:1" "mc3:mc3_block:0:1" "mc4:mc4_last:0:1" "fsm:eextend:4:1"; do
  IFS=: read t rx sk ct <<< "$spec"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c $ct -o gpurun_out/full_${t}_${rx} -f \
      python tools/prof_target.py $t 1 > gpurun_out/ncu_${t}_${rx}.log 2>&1
done
ls -la gpurun_out
