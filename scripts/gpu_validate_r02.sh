#!/bin/bash
# Validation of the device point build with device walk tables (the default):
# the whole GPU suite, smoke, build timing, sanitizer over the build paths.
TAG=${1:-v1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pbuild_gpu.py -q -p no:faulthandler -k "walk_tables_vs_host" -s > gpurun_out/pytest_walkcmp_$TAG.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q -p no:faulthandler > gpurun_out/pytest_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python scripts/pbuild_timing.py radial272 > gpurun_out/pbuild_timing_$TAG.jsonl 2>gpurun_out/pbuild_timing_$TAG.err
timeout 900 python scripts/pbuild_timing.py jitter59 radial128 >> gpurun_out/pbuild_timing_$TAG.jsonl 2>>gpurun_out/pbuild_timing_$TAG.err
timeout 1200 compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py > gpurun_out/sanitizer_$TAG.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck python scripts/sanitize_smoke.py >> gpurun_out/sanitizer_$TAG.log 2>&1
echo done
