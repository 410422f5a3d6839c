#!/bin/bash
# Run the skip-adaptive bench with each build/ab/lib_*.so on each scene, twice, interleaved.
TAG=${1:-ab}
mkdir -p gpurun_out
for rep in 1 2; do
  for sc in ${SCENES:-radial59}; do
    for lib in build/ab/lib_*.so; do
      n=$(basename $lib .so)
      for m in ${MODES:-skip-adaptive}; do
        TETRAY_B200_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --mode $m --scene $sc \
          | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$n', '$sc', '$m', round(r['kernel_ms'],3), round(r['frame_kernels_ms'],3))" >> gpurun_out/ab_$TAG.txt 2>&1
      done
    done
  done
done
echo done
