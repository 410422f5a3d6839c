#!/bin/bash
# Full measurement session -> gpurun_out/*_TAG*: GPU tests, smoke, bench line,
# reference arm, modes, launch list, ncu captures (radial59 march + trace,
# radial272 march; the candidate raster, sort and trace), kernel statistics, e2e breakdown.
TAG=${1:-r01}
mkdir -p gpurun_out
{ free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > gpurun_out/box_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:faulthandler > gpurun_out/pytest_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
for m in reference skip; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --mode $m >> gpurun_out/modes_$TAG.jsonl 2>>gpurun_out/bench_$TAG.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march_sm -s 6 -c 2 \
  -o gpurun_out/prof_march_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"trace|cand_" -s 9 -c 3 \
  -o gpurun_out/prof_trace_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_sm -s 2 -c 2 \
  -o gpurun_out/prof_march272_$TAG python bench.py --scene radial272 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 python scripts/gpu_stats.py > gpurun_out/stats_$TAG.log 2>&1
{ timeout 300 python scripts/e2e_phases.py; echo; timeout 300 python scripts/e2e_jitter.py 300; } > gpurun_out/e2e_$TAG.log 2>&1
echo done
