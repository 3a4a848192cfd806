#!/bin/bash
# racecheck re-run, cf4 ncu capture, FSM / cf4 traces, cf4 e2e phases
mkdir -p gpurun_out/sanitizer
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 200 --error-exitcode 9 \
    python tools/sanitize_target.py > gpurun_out/sanitizer/racecheck.log 2>&1; echo "exit=$?" >> gpurun_out/sanitizer/racecheck.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'local_warp_kernel.*int.64' \
    -s 1 -c 1 -o gpurun_out/full_cf4_local_warp -f python tools/prof_target.py cf4 2 > gpurun_out/ncu_cf4_local_warp.log 2>&1
GPM_TRACE=1 timeout 300 python tools/prof_target.py fsm 2 > gpurun_out/trace_fsm.log 2>&1
GPM_TRACE=1 timeout 300 python tools/prof_target.py cf4 4 > gpurun_out/trace_cf4.log 2>&1
GPM_CF_PIPE=1 GPM_TRACE=1 timeout 300 python tools/prof_target.py cf4 4 > gpurun_out/trace_cf4_pipe.log 2>&1
timeout 300 python tools/e2e_phases.py cf4 12 --keep > gpurun_out/e2e_phases_cf4.log 2>&1
