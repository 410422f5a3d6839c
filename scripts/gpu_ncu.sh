#!/bin/bash
# ncu captures for profiles/: both march launches of one radial59 frame (the
# auto lane width launches G=4 and G=16; one returns at once), the trace pass,
# and the march of radial272 (the DRAM-bound regime).
TAG=${1:-ncu}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_sm -s 6 -c 2 \
  -o gpurun_out/prof_march_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace -s 3 -c 1 \
  -o gpurun_out/prof_trace_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_sm -s 2 -c 2 \
  -o gpurun_out/prof_march272_$TAG python bench.py --scene radial272 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
echo done
