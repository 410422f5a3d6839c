#!/bin/bash
# Flag sweep on the default workload -> gpurun_out/sweep_TAG.jsonl
TAG=${1:-sw}
shift
mkdir -p gpurun_out
for f in "$@"; do
  timeout 600 python bench.py --flags $f --steps 10 --warmup 3 --no-cpu --no-e2e --no-traffic ${BENCH_ARGS} >> gpurun_out/sweep_$TAG.jsonl 2>> gpurun_out/sweep_$TAG.err
done
echo done
