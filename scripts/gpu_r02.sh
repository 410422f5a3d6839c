#!/bin/bash
# Round-2 measurement session -> gpurun_out/*_TAG*: GPU tests, smoke, the
# default bench line (radial272, live ncu traffic, oracle cpu_baseline), the
# reference arm (stock numba render()), a radial59 line.
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler ${PYTEST_ARGS} > gpurun_out/pytest_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --scene radial59 --steps 20 --warmup 5 --no-cpu >> gpurun_out/bench_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo done
