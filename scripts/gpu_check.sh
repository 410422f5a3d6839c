#!/bin/bash
# One GPU session: parity tests, smoke, bench, launch list. Outputs -> gpurun_out/
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -60 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1
echo done
