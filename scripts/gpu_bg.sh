# background-writer A/B on the GPU box -> gpurun_out/bg_*
mkdir -p gpurun_out; rm -f gpurun_out/bg_*
timeout 900 python -m pytest tests -m gpu -q -x -p no:faulthandler > gpurun_out/bg_pytest.log 2>&1
for fl in 0 0x40000 0; do timeout 300 python scripts/e2e_jitter.py 200 gc $fl >> gpurun_out/bg_jit.txt 2>&1; done
TETRAY_B200_STAGED_OUTPUTS=1 timeout 300 python scripts/e2e_jitter.py 200 gc >> gpurun_out/bg_jit.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bg_direct.csv python scripts/e2e_jitter.py 10 > /dev/null 2>&1
tail -2 gpurun_out/bg_pytest.log
