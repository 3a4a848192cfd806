#!/bin/bash
# End-of-round GPU pass: parity suite, smoke, default bench line (cf4 + sub-records
# + CPU baseline), reference arm, profiles (launch list + ncu of each dominant
# kernel), compute-sanitizer.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
[ -z "$NOPROF" ] && bash tools/gpu_profiles.sh
[ -z "$NOSAN" ] && bash tools/gpu_sanitize.sh
ls -la gpurun_out
