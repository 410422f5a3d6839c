#!/bin/bash
# BASELINE config 5: high-resolution frames (multi-chunk) -- parity at 1024^2, timing up to 4096^2.
TAG=${1:-h}
mkdir -p gpurun_out
free -g > gpurun_out/meminfo_$TAG.txt; nproc >> gpurun_out/meminfo_$TAG.txt
timeout 900 python scripts/hires_parity.py > gpurun_out/hires_parity_$TAG.log 2>&1
for sc in 2 4 8; do
  timeout 600 python bench.py --steps 3 --warmup 3 --scale $sc --no-cpu >> gpurun_out/hires_$TAG.jsonl 2>>gpurun_out/hires_$TAG.err
done
echo done
