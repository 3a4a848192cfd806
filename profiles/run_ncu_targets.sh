#!/bin/bash
# ncu --set full of the dominant extend kernels (one launch each), B200_PROFILING.md recipe
for t in cf4 tc mc3s mc4s fsms; do
  python tools/prof_target.py $t 2
  ncu --set full --clock-control none --import-source on -k regex:"extend" -s 3 -c 3 -o gpurun_out/full_$t -f \
      python tools/prof_target.py $t 2 > /dev/null 2>&1
done
ls -la gpurun_out
