# candidate raster vs BSP walk by frame size (radial59 skip-adaptive) -> gpurun_out/res.jsonl
mkdir -p gpurun_out; rm -f gpurun_out/res.jsonl
for sc in 1 2 4 8; do for fl in 0x1000000 0x800000; do
timeout 600 python bench.py --steps 3 --warmup 2 --scale $sc --no-cpu --no-e2e --flags $fl >> gpurun_out/res.jsonl 2>/dev/null
done; done
