mkdir -p gpurun_out
for v in G512 G768 G1024; do for r in 1 2; do GPM_LIB_VARIANT=libgpm_$v.so GPM_TRACE=1 timeout 300 python tools/prof_target.py fsm 2 2>&1 | grep "group_qc_L1\|group_domain_L1\|^fsm" | tail -3 | sed "s/^/$v /"; done; done
