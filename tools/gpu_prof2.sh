#!/bin/bash
# ncu --set full captures: SPEC="target:regex:skip:count[:ENV=VAL] ..." (tools/prof_target.py targets)
mkdir -p gpurun_out
for spec in ${SPEC}; do
  IFS=: read t rx sk ct envs <<< "$spec"
  tag=${t}_${rx}${envs:+_${envs%%=*}}
  env $envs timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s ${sk:-0} -c ${ct:-1} -o gpurun_out/full_${tag} -f \
      python tools/prof_target.py $t 1 > gpurun_out/ncu_${tag}.log 2>&1
done
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${LAUNCHES}.csv \
    python bench.py --app ${LAUNCHES} --steps 2 --warmup 3 --no-cpu-baseline --no-sub > /dev/null 2>&1
fi
ls -la gpurun_out
