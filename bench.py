#!/usr/bin/env python3
"""Benchmark of the tetray render hot path on B200 (BASELINE.json metric).

Workload (BASELINE config 2): radial59 -- 1,026,895 tets,
default KD partitions (8,192; 4,040 active), the radial16 TF scaled to N=59,
camera [40,26,34]*59/16 -> [29.5]^3, fov 35, 512x512, s1=0.08, s2=0.64, p=2,
termination 0.9999, mode skip-adaptive (the paper's headline mode).

One step = one frame.  Items = samples (point queries, RenderStats.total_samples).
  value   device-timed: scene + epoch resident in HBM, CUDA events around the
          render kernel on its stream, L2 flushed (256 MiB write) between steps
  e2e     through the public render() API: per step the metadata epoch is
          re-uploaded from pinned host memory (H2D) and rgba + samples +
          counters are read back (D2H); wall clock, max over ranks
N > 1: strong scaling -- the frame's 8x4 pixel tiles are interleaved over the
ranks, partial tiles all-gathered and per-partition counts all-reduced
over NCCL (paper_1908_01906_b200/distributed.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
UNIT = "samples/s"
RECORD_BYTES = {0: 128, 1: 104}   # algorithmic bytes per sample (vertex / cell), SURVEY §8d
PIXEL_BYTES = 44                  # rgba f64x4 + samples i64 + visited i32


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scene", default="radial59")
    ap.add_argument("--mode", default="skip-adaptive")
    ap.add_argument("--scale", type=float, default=1.0, help="image size multiplier (512*scale)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0,
                    help="TR_FLAG_* bits (tuning experiments; bits 8-11 = log2 group size)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic():
    """DRAM bytes per render launch from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "r01" / "ncu_dram.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def build_workload(B, args):
    import cases as C
    t0 = time.perf_counter()
    scene = C.build_scene(B, args.scene)
    cam = C.camera(B, args.scene, scale=args.scale)
    par = C.params(B, args.scene)
    return scene, cam, par, time.perf_counter() - t0


def cpu_reference(scene, cam, par, args, budget_s):
    """The oracle port on all host cores, full frames until `budget_s` elapses."""
    from oracle.oracle import OracleScene
    orc = OracleScene(scene)
    threads = os.cpu_count() or 1
    orc.render(cam, args.mode, par, threads=threads, rows=(0, 8))  # warm caches
    t0 = time.perf_counter()
    frames, samples = 0, 0
    while True:
        _, s, _, _ = orc.render(cam, args.mode, par, threads=threads)
        frames += 1
        samples += int(s.sum())
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": samples / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{frames} full {cam.width}x{cam.height} {args.mode} frame(s) of "
                      f"{args.scene} in {dt:.2f} s (oracle/oracle.c, OpenMP over rows)",
            "ms_per_frame": dt * 1000.0 / frames}


def run_reference(args, rank):
    if rank != 0:
        return 0
    import paper_1908_01906_b200 as B
    scene, cam, par, _ = build_workload(B, args)
    from oracle.oracle import OracleScene
    orc = OracleScene(scene)
    threads = os.cpu_count() or 1
    for _ in range(max(args.warmup, 1) if args.warmup else 0):
        orc.render(cam, args.mode, par, threads=threads, rows=(0, cam.height // 8))
    # each step: a bounded row band (1/8 of the frame), so K steps stay within minutes
    band = max(1, cam.height // 8)
    times, samples = [], 0
    for k in range(args.steps):
        r0 = (k * band) % cam.height
        t0 = time.perf_counter()
        _, s, _, _ = orc.render(cam, args.mode, par, threads=threads, rows=(r0, min(r0 + band, cam.height)))
        times.append(time.perf_counter() - t0)
        samples += int(s.sum())
    tot = sum(times)
    v = samples / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot * 1000.0 / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.scene} {cam.width}x{cam.height} {args.mode}",
                       "scene": args.scene, "mode": args.mode, "width": cam.width,
                       "height": cam.height, "n_tets": scene.mesh.n_tets,
                       "n_partitions": scene.n_partitions, "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{args.steps} row bands of {band} rows "
                                       f"(oracle/oracle.c, OpenMP)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import torch.distributed as dist

    import paper_1908_01906_b200 as B
    from paper_1908_01906_b200 import distributed as D
    from paper_1908_01906_b200.device import device_scene_for

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    scene, cam, par, build_s = build_workload(B, args)
    t0 = time.perf_counter()
    dscene = device_scene_for(scene, dev)
    upload_s = time.perf_counter() - t0
    mode_id = {"reference": 0, "skip": 1, "skip-adaptive": 2}[args.mode]
    track = args.mode != "reference"
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    runner = D.ShardedFrame(dscene, scene, cam, mode_id, par, track=track,
                            rank=rank if world > 1 else 0, world=world, flags=args.flags)
    # warm-up
    for _ in range(args.warmup):
        runner.run(stream)
    torch.cuda.synchronize()
    total_samples = runner.total_samples()

    # timed region: K steps, L2 flushed between steps, kernel timed with events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    mev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        time.sleep(0.25)
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            ev[k][0].record(stream)
            runner.run(stream, kernel_events=kev[k], march_events=mev[k])
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        time.sleep(0.1)
    launches_per_step = runner.launches_per_step()   # of the timed frames (not the e2e ones)
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    march_ms = [a.elapsed_time(b) for a, b in mev]
    t_local = sum(step_ms) / 1000.0
    k_local = sum(kern_ms) / len(kern_ms) / 1000.0
    m_local = sum(march_ms) / len(march_ms) / 1000.0
    if world > 1:
        t = torch.tensor([t_local, k_local, m_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max, k_max, m_max = float(t[0]), float(t[1]), float(t[2])
    else:
        t_max, k_max, m_max = t_local, k_local, m_local
    clocks = clk.summary()
    value = total_samples * args.steps / t_max

    # roofline of the dominant kernel (render_frame_kernel), per launch
    hbm, peak_kind = peaks()
    my_samples = runner.local_samples()
    my_pixels = runner.local_pixels()
    alg_bytes = RECORD_BYTES[int(scene.mesh.centering)] * my_samples + PIXEL_BYTES * my_pixels
    achieved = alg_bytes / m_max / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": ncu_traffic(), "peak_kind": peak_kind,
            "kernel": "march_sm_kernel", "kernel_ms": m_max * 1e3,
            "frame_kernels_ms": k_max * 1e3,
            "frame_frac": alg_bytes / k_max / 1e9 / hbm,
            "alg_bytes_per_launch": alg_bytes,
            "alg_bytes_model": f"{RECORD_BYTES[int(scene.mesh.centering)]} B/sample x "
                               f"{my_samples} samples + {PIXEL_BYTES} B/pixel x {my_pixels} pixels"}

    # e2e through render(): epoch H2D + outputs D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        if world > 1:
            e2e = D.bench_e2e_sharded(runner, args.steps, rank, world)
        else:
            fb = None
            for _ in range(max(args.warmup, 3)):
                # hold the previous frame like the timed loop does, so the
                # page-locked result buffers are in the host cache already
                dscene._epochs.clear()
                fb, st = B.render(scene, cam, args.mode, par, device=dev)
            per = []
            e2e_steps = max(args.steps, 20)   # wall-clock: more steps for a stable mean
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                t1 = time.perf_counter()
                dscene._epochs.clear()  # force the per-frame metadata upload
                fb, st = B.render(scene, cam, args.mode, par, device=dev)
                per.append(time.perf_counter() - t1)
            dt = time.perf_counter() - t0
            ep = next(iter(dscene._epochs.values()))
            h2d = ep.h2d_bytes
            d2h = fb.rgba.nbytes + fb.samples.nbytes + 8 * (3 + scene.n_partitions)
            e2e = {"value": st.total_samples * e2e_steps / dt, "unit": UNIT,
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                   "ms_per_step": dt * 1000.0 / e2e_steps, "steps": e2e_steps,
                   "ms_per_step_median": statistics.median(per) * 1000.0,
                   "ms_per_step_min": min(per) * 1000.0}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference(scene, cam, par, args, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max * 1000.0 / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.scene} {cam.width}x{cam.height} {args.mode}",
                       "scene": args.scene, "mode": args.mode, "width": cam.width,
                       "height": cam.height, "n_tets": scene.mesh.n_tets,
                       "n_partitions": scene.n_partitions,
                       "n_active": int(scene.meta_state()[0].sum()),
                       "samples_per_frame": total_samples,
                       "rays_per_s": cam.width * cam.height * args.steps / t_max,
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"pixel tiles interleaved over {world} GPU(s)",
                       "flags": hex(args.flags),
                       "scene_build_s": round(build_s, 3), "upload_s": round(upload_s, 3),
                       "resident_bytes": int(dscene.resident_bytes)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
