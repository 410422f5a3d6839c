#!/bin/bash
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 600 python scripts/gpu_debug.py > gpurun_out/debug.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python scripts/gpu_debug.py golden_radial4 constant single voidcell axis > gpurun_out/memcheck.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:faulthandler > gpurun_out/pytest_full.log 2>&1
echo done
