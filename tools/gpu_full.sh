mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
PYX=" " RUNS="cf4 tc fsm mc3 mc4" bash tools/gpu_iter.sh
bash tools/gpu_sanitize.sh
