#!/bin/bash
# Flag variants on several scenes: gpu_flags.sh TAG "scenes" flags...
TAG=$1; SCENES=$2; shift 2
mkdir -p gpurun_out
for sc in $SCENES; do
  for fl in "$@"; do
    timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --scene $sc --flags $fl >> gpurun_out/flags_$TAG.jsonl 2>>gpurun_out/flags_$TAG.err
  done
done
echo done
