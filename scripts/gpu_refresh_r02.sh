#!/bin/bash
# Short re-measurement after kernel changes -> gpurun_out/*_TAG*: GPU tests,
# the default bench line, modes, the config-2/3/4 lines, launch list and the
# radial272 march ncu capture (the rest of gpu_final_r02.sh unchanged).
TAG=${1:-r02e}
mkdir -p gpurun_out
{ free -g; nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > gpurun_out/box_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > gpurun_out/pytest_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
for m in reference skip; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --mode $m >> gpurun_out/modes_$TAG.jsonl 2>>gpurun_out/bench_$TAG.err
done
for sc in radial59 radial128; do
  for m in skip-adaptive skip reference; do
    timeout 900 python bench.py --scene $sc --mode $m --steps 10 --warmup 3 --no-cpu >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
  done
done
for m in skip-adaptive skip reference; do
  timeout 1500 python bench.py --scene grid585 --mode $m --steps 5 --warmup 3 --no-cpu >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-traffic > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_sm -s 2 -c 2 \
  -o gpurun_out/prof_march272_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-traffic > /dev/null 2>&1
timeout 600 python scripts/e2e_phases.py radial59 radial128 > gpurun_out/e2e_phases_$TAG.txt 2>&1
echo done
