#!/bin/bash
# A/B: each build/ab/<name> library (and the default one) x flags on the
# default workload -> gpurun_out/ab_TAG.jsonl (detail.lib names the build)
TAG=${1:-ab}
shift
FLAGS=${FLAGS:-0}
mkdir -p gpurun_out
for lib in default "$@"; do
  for f in $FLAGS; do
    if [ "$lib" = default ]; then L=""; else L="$PWD/build/ab/$lib/libtetray_b200.so"; fi
    TETRAY_B200_LIB=$L timeout 600 python bench.py --flags $f --steps 10 --warmup 3 --no-cpu --no-e2e --no-traffic ${BENCH_ARGS} 2>> gpurun_out/ab_$TAG.err | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/ab_$TAG.jsonl
  done
done
echo done
