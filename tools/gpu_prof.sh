#!/bin/bash
# ncu --set full of the dominant extend kernel of each workload (B200_PROFILING.md recipe)
mkdir -p gpurun_out
for t in ${TARGETS:-cf4 tc mc3s mc4s fsms}; do
  timeout 120 python tools/prof_target.py $t 2 > gpurun_out/prof_$t.txt 2>&1
  K=$(python - <<PY
import re
s=open("gpurun_out/prof_$t.txt").read().split()
print(s[3] if len(s)>3 else "extend")
PY
)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-extend}" -s ${SKIP:-2} -c ${COUNT:-4} -o gpurun_out/full_$t -f \
      python tools/prof_target.py $t 2 > gpurun_out/ncu_$t.log 2>&1
done
ls -la gpurun_out
