mkdir -p gpurun_out
GPM_TRACE=1 timeout 300 python tools/prof_target.py fsm 2 > gpurun_out/trace_fsm.log 2>&1
GPM_TRACE=1 timeout 300 python tools/prof_target.py mc4 2 > gpurun_out/trace_mc4.log 2>&1
SPEC="mc4:mc4_last:1:1" bash tools/gpu_ncu.sh
