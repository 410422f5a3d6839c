#!/bin/bash
# Device point-location build (csrc/pbuild.cu) and the PEER brick exchange:
# parity tests, then host vs device build timing on general meshes ->
# gpurun_out/*_TAG*.  CONFIG3=1 also runs radial128/272 (slow).
TAG=${1:-pb1}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_pbuild_gpu.py tests/test_bricks_gpu.py -q -p no:faulthandler -k "not config3" > gpurun_out/pytest_pbuild_$TAG.log 2>&1
echo "small rc=$?" >> gpurun_out/pytest_pbuild_$TAG.log
timeout 900 python scripts/pbuild_timing.py jitter59 radial128 > gpurun_out/pbuild_timing_$TAG.jsonl 2> gpurun_out/pbuild_timing_$TAG.err
echo "timing rc=$?" >> gpurun_out/pbuild_timing_$TAG.err
if [ -n "$CONFIG3" ]; then
timeout 1800 python -m pytest tests/test_pbuild_gpu.py -q -x -p no:faulthandler -k "config3" >> gpurun_out/pytest_pbuild_$TAG.log 2>&1
echo "config3 rc=$?" >> gpurun_out/pytest_pbuild_$TAG.log
timeout 1200 python scripts/pbuild_timing.py radial272 >> gpurun_out/pbuild_timing_$TAG.jsonl 2>> gpurun_out/pbuild_timing_$TAG.err
fi
echo done
