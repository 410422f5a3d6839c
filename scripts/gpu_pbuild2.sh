#!/bin/bash
# Follow-up: PEER brick exchange test, device-walk tests, build timing incl.
# device-walk (jitter59, radial128, radial272) -> gpurun_out/*_TAG*.
TAG=${1:-pb3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bricks_gpu.py tests/test_pbuild_gpu.py -q -p no:faulthandler -k "dist_gpu or device_walk" > gpurun_out/pytest_pbuild_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_pbuild_$TAG.log
timeout 1500 python scripts/pbuild_timing.py jitter59 radial128 radial272 > gpurun_out/pbuild_timing_$TAG.jsonl 2> gpurun_out/pbuild_timing_$TAG.err
echo "timing rc=$?" >> gpurun_out/pbuild_timing_$TAG.err
echo done
