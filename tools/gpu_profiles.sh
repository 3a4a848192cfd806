#!/bin/bash
# Round profiling pass (B200_PROFILING.md recipe): launch list of the headline
# bench command + one ncu --set full capture of each workload's dominant kernel.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cf4.csv \
    python bench.py --app cf4 --steps 2 --warmup 3 --no-cpu-baseline --no-sub > /dev/null 2>&1
# target : kernel regex (demangled name) : launches to skip : count
for spec in "cf4:local_warp_kernel.*int.64:1:1" "tc:edge_lane_kernel:0:1" "mc3:mc3_warp:0:1" "mc3:mc3_block:0:1" \
            "mc4:mc4_roots:0:1" "fsm:efan_kernel:0:1"; do
  IFS=: read t rx sk ct <<< "$spec"
  tag=$(echo "$rx" | sed 's/[^A-Za-z0-9_]//g' | cut -c1-24)
  timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$rx" \
      -s $sk -c $ct -o gpurun_out/full_${t}_${tag} -f python tools/prof_target.py $t 2 > gpurun_out/ncu_${t}_${tag}.log 2>&1
done
ls -la gpurun_out
