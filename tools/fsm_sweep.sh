#!/bin/bash
# FSM min-support sweep (sigma in {100, 300, 1000, 3000}) on the
# Mico-like config; one bench line per sigma, CPU oracle baseline included.
mkdir -p gpurun_out
for s in 100 300 1000 3000; do
  timeout 900 python bench.py --app fsm --sigma $s --steps 3 --warmup 3 > gpurun_out/fsm_sweep_$s.json 2> gpurun_out/fsm_sweep_$s.err
done
