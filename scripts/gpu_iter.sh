#!/bin/bash
# One build -> measure iteration -> gpurun_out/*_TAG*: GPU tests, the default
# bench line (radial272) and radial59, modes, and one ncu --set full capture of
# the radial272 march kernel.
TAG=${1:-it}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:faulthandler ${PYTEST_ARGS} > gpurun_out/pytest_$TAG.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
for m in reference skip; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --mode $m >> gpurun_out/bench_$TAG.json 2>> gpurun_out/bench_$TAG.err
done
timeout 600 python bench.py --scene radial59 --steps 20 --warmup 5 --no-cpu --no-traffic >> gpurun_out/bench_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --flags 0x2000000 --steps 10 --warmup 3 --no-cpu --no-e2e --no-traffic >> gpurun_out/bench_$TAG.json 2>> gpurun_out/bench_$TAG.err
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_sm -s 2 -c 2 \
  -o gpurun_out/prof_march272_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-traffic > /dev/null 2>&1
fi
echo done
