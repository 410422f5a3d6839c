#!/bin/bash
# BASELINE configs beyond the default bench line -> gpurun_out/configs_TAG.jsonl
#   config 2 modes: radial59 reference / skip (skip-adaptive is the default line)
#   config 3: radial128 (1.0e7 tets), radial272 (1.0e8 tets, host build) at 512^2
#   config 4: grid585 (1.0e9 tets, device-generated, 148 GB resident) at 512^2
#   config 5: radial59 at 1024^2 .. 4096^2 (multi-chunk frames), parity at 1024^2 / 1536^2
TAG=${1:-cfg}
mkdir -p gpurun_out
{ free -g; nproc; nvidia-smi --query-gpu=name,memory.total --format=csv; } > gpurun_out/box_$TAG.txt 2>&1
timeout 900 python scripts/hires_parity.py > gpurun_out/hires_parity_$TAG.log 2>&1
for sc in 2 4 8; do
  timeout 600 python bench.py --steps 5 --warmup 3 --scale $sc --no-cpu >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
done
for scene in radial128 radial272; do
  for m in skip-adaptive reference; do
    timeout 1800 python bench.py --steps 5 --warmup 3 --scene $scene --mode $m --cpu-seconds 20 >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
  done
done
for m in skip-adaptive skip reference; do
  timeout 1800 python bench.py --steps 5 --warmup 3 --scene grid585 --mode $m --no-cpu >> gpurun_out/configs_$TAG.jsonl 2>>gpurun_out/configs_$TAG.err
done
echo done
