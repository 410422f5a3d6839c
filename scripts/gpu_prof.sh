#!/bin/bash
# ncu --set full of the march kernel for one flag setting. -> gpurun_out/prof_$TAG.ncu-rep
TAG=$1; FL=${2:-0}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march -s 2 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu --flags $FL > gpurun_out/ncu_$TAG.log 2>&1
timeout 300 python scripts/gpu_stats.py > gpurun_out/stats_$TAG.log 2>&1
echo done
