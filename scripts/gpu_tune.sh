#!/bin/bash
# Variant timing sweep of flags for the benchmark frame. -> gpurun_out/tune_$TAG.jsonl
TAG=${1:-t}; shift
mkdir -p gpurun_out
for fl in "$@"; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --flags $fl | sed "s/^/$fl /" >> gpurun_out/tune_$TAG.jsonl 2>>gpurun_out/tune_$TAG.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace -s 2 -c 1 \
  -o gpurun_out/prof_trace_$TAG python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1
echo done
