#!/bin/bash
# Iteration loop on the GPU box -> gpurun_out/
#   gpu_iter.sh TAG [quick|std|full] [flags...]
#   quick: modes bench + flag variants; std: + parity sweep; full: + pytest, ncu, launch list
TAG=${1:-it}
MODE=${2:-std}
shift 2
FLAGS=${@:-0x40 0x300}
mkdir -p gpurun_out
if [ "$MODE" != "quick" ]; then
  timeout 600 python scripts/gpu_debug.py > gpurun_out/debug_$TAG.log 2>&1
fi
for m in reference skip skip-adaptive; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --mode $m >> gpurun_out/modes_$TAG.jsonl 2>>gpurun_out/modes_$TAG.err
done
for fl in $FLAGS; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --flags $fl >> gpurun_out/groups_$TAG.jsonl 2>>gpurun_out/modes_$TAG.err
done
if [ "$MODE" == "full" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -p no:faulthandler > gpurun_out/pytest_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:march -s 2 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
fi
echo done
