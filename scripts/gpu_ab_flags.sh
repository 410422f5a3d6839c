# A/B of TR_FLAG values on the bench (device-timed frame) -> gpurun_out/abf_$TAG.jsonl
#   SCENES="radial59 radial128" MODES="skip-adaptive skip" bash scripts/gpu_ab_flags.sh TAG flags...
TAG=$1; shift
mkdir -p gpurun_out; rm -f gpurun_out/abf_$TAG.jsonl
for rep in 1 2; do
for sc in ${SCENES:-radial59}; do
for m in ${MODES:-skip-adaptive}; do
for fl in "$@"; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --flags $fl --scene $sc --mode $m >> gpurun_out/abf_$TAG.jsonl 2>/dev/null
done; done; done; done
