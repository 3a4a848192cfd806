#!/bin/bash
# compute-sanitizer over every kernel path at small size (VERDICT r1 hygiene):
# memcheck, racecheck (shared-memory hazards), synccheck, initcheck.
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_target.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer/$tool.log
done
tail -n 4 gpurun_out/sanitizer/*.log
