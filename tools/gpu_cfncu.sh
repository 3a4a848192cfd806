#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
SPEC="cf4:local_warp:2:1" bash tools/gpu_ncu.sh
python tools/ncu_summary.py gpurun_out/full_cf4_local_warp.ncu-rep > gpurun_out/full_cf4_local_warp.txt 2>&1
