#!/bin/bash
# Summarise a gpu_iter.sh run: parity mismatches, per-mode and per-flag timings.
TAG=$1
[ -f gpurun_out/debug_$TAG.log ] && { echo "parity lines not exact:"; grep -v "samples_diff_px=0 rgba_diff_px=0" gpurun_out/debug_$TAG.log | head; }
for f in gpurun_out/modes_$TAG.jsonl gpurun_out/groups_$TAG.jsonl; do
  [ -f $f ] && python -c "
import json
for l in open('$f'):
    d=json.loads(l); r=d['roofline']
    print(f\"{d['config']['mode']:14s} flags={d['config'].get('flags','-'):>8} step={d['ms_per_step']:.3f} march={r['kernel_ms']:.3f} frame={r['frame_kernels_ms']:.3f} frac={r['frac']:.3f}\")
"
done
[ -f gpurun_out/pytest_$TAG.log ] && tail -1 gpurun_out/pytest_$TAG.log
true
[ -f gpurun_out/flags_$TAG.jsonl ] && python -c "
import json
for l in open('gpurun_out/flags_$TAG.jsonl'):
    d=json.loads(l); r=d['roofline']; c=d['config']
    print(f\"{c['scene']:10s} {c['mode']:14s} flags={c.get('flags','-'):>8} march={r['kernel_ms']:.3f} frame={r['frame_kernels_ms']:.3f} frac={r['frac']:.3f} Gs/s={d['value']/1e9:.2f}\")
"
true
