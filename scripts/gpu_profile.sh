#!/bin/bash
# Mode breakdown + one full ncu capture of render_frame_kernel. Outputs -> gpurun_out/
mkdir -p gpurun_out
TAG=${1:-r01}
for m in reference skip skip-adaptive; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --mode $m >> gpurun_out/modes_$TAG.jsonl 2>>gpurun_out/modes_$TAG.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_frame -s 3 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1
echo done
