mkdir -p gpurun_out; rm -f gpurun_out/ts_*
timeout 900 python -m pytest tests -m gpu -q -x -p no:faulthandler > gpurun_out/ts_pytest.log 2>&1
for i in 1 2; do
for fl in 0 0x40000; do
timeout 300 python scripts/e2e_jitter.py 200 gc $fl >> gpurun_out/ts_jit.txt 2>&1
TETRAY_B200_STAGED_OUTPUTS=1 timeout 300 python scripts/e2e_jitter.py 200 gc $fl >> gpurun_out/ts_jit_staged.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --flags $fl >> gpurun_out/ts_bench.jsonl 2>&1
done; done
tail -2 gpurun_out/ts_pytest.log
