#!/bin/bash
# Round-2 measurement session -> gpurun_out/*_TAG*
#   box info, GPU tests, smoke, the default bench line (radial272: e2e, live
#   ncu traffic, oracle cpu_baseline), the reference arm (stock numba
#   render()), modes, BASELINE configs 2-5, a launch list, ncu --set full of
#   the march (radial272, grid585) and of the interval-list kernels, kernel
#   statistics, compute-sanitizer.
TAG=${1:-r02}
mkdir -p gpurun_out
{ free -g; nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > gpurun_out/box_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > gpurun_out/pytest_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 1800 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
for m in reference skip; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --mode $m >> gpurun_out/modes_$TAG.jsonl 2>>gpurun_out/bench_$TAG.err
done
for sc in radial59 radial128; do
  for m in skip-adaptive skip reference; do
    timeout 900 python bench.py --scene $sc --mode $m --steps 10 --warmup 3 --no-cpu >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
  done
done
timeout 1200 python bench.py --scene radial272 --host-build --steps 10 --warmup 3 --no-cpu --no-traffic >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
for m in skip-adaptive skip reference; do
  timeout 1500 python bench.py --scene grid585 --mode $m --steps 5 --warmup 3 --no-cpu >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
done
for sc in 2 4 8; do
  timeout 900 python bench.py --scene radial59 --scale $sc --steps 5 --warmup 3 --no-cpu --no-traffic >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-traffic > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_sm -s 2 -c 2 \
  -o gpurun_out/prof_march272_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-traffic > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trace|cand_|ray_table|order" -s 5 -c 5 \
  -o gpurun_out/prof_trace272_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-traffic > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:march_sm -s 2 -c 2 \
  -o gpurun_out/prof_march585_$TAG python bench.py --scene grid585 --steps 1 --warmup 1 --no-e2e --no-cpu --no-traffic > /dev/null 2>&1
for sc in radial59 grid272; do timeout 300 python scripts/gpu_stats.py $sc >> gpurun_out/stats_$TAG.log 2>&1; done
timeout 900 python scripts/brick_bench.py radial59 radial128 > gpurun_out/bricks_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
timeout 600 python scripts/shard_timing.py grid272 skip-adaptive > gpurun_out/shard_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
timeout 600 python scripts/shard_timing.py grid272 reference >> gpurun_out/shard_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
timeout 900 python scripts/pbuild_timing.py radial272 > gpurun_out/pbuild_timing_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
timeout 900 python scripts/pbuild_timing.py jitter59 radial128 >> gpurun_out/pbuild_timing_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
timeout 600 python scripts/e2e_phases.py radial59 radial128 > gpurun_out/e2e_phases_$TAG.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py > gpurun_out/sanitizer_$TAG.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck python scripts/sanitize_smoke.py >> gpurun_out/sanitizer_$TAG.log 2>&1
echo done
