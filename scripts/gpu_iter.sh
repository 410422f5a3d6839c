#!/bin/bash
# Iteration loop on the GPU box: parity sweep, modes bench, optional pytest/ncu. -> gpurun_out/
TAG=${1:-it}
mkdir -p gpurun_out
timeout 600 python scripts/gpu_debug.py > gpurun_out/debug_$TAG.log 2>&1
for m in reference skip skip-adaptive; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --mode $m >> gpurun_out/modes_$TAG.jsonl 2>>gpurun_out/modes_$TAG.err
done
for fl in 0x40 0x1 0x41 0x100 0x300 0x500; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --flags $fl >> gpurun_out/groups_$TAG.jsonl 2>>gpurun_out/modes_$TAG.err
done
if [ "$2" == "full" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -p no:faulthandler > gpurun_out/pytest_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:march -s 2 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
fi
echo done
timeout 300 python scripts/gpu_stats.py > gpurun_out/stats_$TAG.log 2>&1
