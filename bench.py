#!/usr/bin/env python3
"""Benchmark of the tetray render hot path on B200 (BASELINE.json metric).

Workload (BASELINE config 3: headline the >= 1e8-tet scene,
where every sample's tet record is a DRAM miss): radial272 -- 100,618,240
tets, default KD partitions (4,096), the radial16 TF scaled to N=272, camera
[40,26,34]*272/16 -> [136]^3, fov 35, 512x512, s1=0.08, s2=0.64, p=2,
termination 0.9999, mode skip-adaptive (the paper's headline mode).
`--scene radial59` is BASELINE config 2 (1e6 tets).  On the GPU arm a radialN
scene with N >= 128 is generated in HBM (GridScene, csrc/synth.cu) -- the
same scene bit for bit: tests/test_parity_big_gpu.py renders it equal to the
reference's own radial272 frames; `--host-build` uses the general host path.

One step = one frame.  Items = samples (point queries, RenderStats.total_samples).
  value     device-timed: scene + epoch resident in HBM, CUDA events around
            the frame's kernels on their stream, L2 flushed (256 MiB write)
            between steps (the 13 GB of records exceed L2 anyway)
  e2e       the public render() API with host buffers: per step the metadata
            epoch is re-uploaded from pinned host memory (H2D) and rgba +
            samples + counters are read back (D2H)
  roofline  march_sm_kernel (the dominant kernel): SURVEY §8d algorithmic
            bytes (128 B/sample + 44 B/pixel) / its event-timed duration;
            `traffic` = ncu dram__bytes_read.sum + dram__bytes_write.sum of
            that kernel, measured live by an ncu subprocess on this workload
            (null when ncu is unavailable)
  cpu_baseline  the oracle (oracle/oracle.c, a bit-exact C port of the
            numba kernel) on its own scene build, all host cores, a bounded
            sample of whole frames
N > 1 (`--gpus N` re-launches itself under torch.distributed.run when
WORLD_SIZE is unset): one frame's 8x4 pixel tiles interleaved over the
ranks, each rank's tiles gathered to rank 0 and the counters reduced there
over NCCL (paper_1908_01906_b200/distributed.py).  Default `--scaling weak`:
the frame side grows with sqrt(N) (512, 728, 1024, 1448 px at N = 1, 2, 4,
8; same camera), so every GPU keeps ~512^2 rays -- a 512^2 frame split 8
ways leaves 32k rays per B200, under one wave of its march lanes.
`--scaling strong` splits the 512^2 frame itself.

--impl reference: the reference's own render() (pkg/src/tetray/render.py:161-205,
numba, installed under baseline/_ref) with all host threads, on whole frames
of the same workload, rank 0 only.  Its Scene is the stock dataclasses
assembled around the oracle's C restatement of the generator, KD split and
BVH build (oracle/stock_scene.py; the stock Python builders need ~40 min at
1e8 tets).  libtetray_b200.so is never loaded on that path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import csv
import math
import io
import json
import os
import platform
import shutil
import socket
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
MODES = ("reference", "skip", "skip-adaptive")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scene", default="radial272")
    ap.add_argument("--mode", default="skip-adaptive", choices=MODES)
    ap.add_argument("--scale", type=float, default=1.0, help="image size multiplier (512*scale)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = frame side x sqrt(N) (fixed rays per GPU), strong = "
                         "the same frame split N ways")
    ap.add_argument("--host-build", action="store_true",
                    help="build radialN through the general host path, not GridScene")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-traffic", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-budget-s", type=float, default=180.0,
                    help="reference arm: stop timing whole frames after this many seconds")
    ap.add_argument("--shard", default="pixels", choices=["pixels", "records"],
                    help="records: KD-brick record sharding (bricks.py; one brick per rank, "
                         "or --bricks bricks emulated on one GPU)")
    ap.add_argument("--bricks", type=int, default=2, help="--shard records on one GPU: bricks")
    ap.add_argument("--exchange", default="peer", choices=["peer", "sum"],
                    help="--shard records, N > 1: ray states pushed to peer inboxes over NVLink "
                         "(CUDA IPC) or a SUM all-reduce of the state array per round")
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0,
                    help="TR_FLAG_* bits (tuning experiments; bits 8-11 = log2 group size)")
    return ap.parse_args(argv)


def weak_scale(args, world: int) -> None:
    """--scaling weak at N > 1: the frame side x sqrt(N), rounded to whole
    8-pixel tiles, so the rays per GPU stay those of the N = 1 frame."""
    if world > 1 and args.scaling == "weak":
        side = int(round(512 * args.scale * math.sqrt(world) / 8.0)) * 8
        args.scale = side / 512.0


def scene_n(name: str) -> int:
    for pre in ("radial", "grid"):
        if name.startswith(pre) and name[len(pre):].isdigit():
            return int(name[len(pre):])
    return 0


def public_name(name: str) -> str:
    """gridN is radialN generated in HBM: the workload is named radialN."""
    return f"radial{scene_n(name)}" if name.startswith("grid") else name


def workload_config(args, n_tets, n_parts, samples) -> dict:
    """The `config` dict -- identical in both arms for the same workload."""
    w = h = int(512 * args.scale)
    scene = public_name(args.scene)
    return {"workload": f"{scene} {w}x{h} {args.mode}", "scene": scene, "mode": args.mode,
            "width": w, "height": h, "n_tets": int(n_tets), "n_partitions": int(n_parts),
            "samples_per_frame": int(samples)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback"


def mapped_repo_libs() -> list:
    """Shared objects of this repository mapped into the process (/proc/self/maps)."""
    libs = set()
    try:
        for line in Path("/proc/self/maps").read_text().splitlines():
            path = line.split()[-1] if line.split() else ""
            if path.endswith(".so") and str(ROOT) in path:
                libs.add(str(Path(path).relative_to(ROOT)))
    except OSError:
        pass
    return sorted(libs)


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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


# ---------------------------------------------------------------- workloads

def build_gpu_workload(B, args):
    import cases as C
    n = scene_n(args.scene)
    name = args.scene
    if name.startswith("radial") and n >= 128 and not args.host_build:
        name = f"grid{n}"
    t0 = time.perf_counter()
    scene = C.build_scene(B, name)
    cam = C.camera(B, name, scale=args.scale)
    par = C.params(B, name)
    return scene, cam, par, time.perf_counter() - t0


def build_oracle_workload(args):
    """The oracle's own scene (oracle/scene.py), camera and params."""
    import cases as C
    import oracle.scene as OS
    n = scene_n(args.scene)
    if not n or not args.scene.startswith(("radial", "grid")):
        raise SystemExit(f"the oracle builds radialN / gridN scenes only, not {args.scene!r}")
    leaf = 48 if n == 16 else None   # tests/cases.py: radial16 uses KdBuildConfig(48)
    scene = OS.GridScene(n, OS.TF.from_json(C.radial16_tf_doc(n)), max_leaf=leaf)
    return scene, C.camera(OS, public_name(args.scene), scale=args.scale), \
        C.params(OS, public_name(args.scene))


def cpu_reference(args, budget_s):
    """The oracle port on all host cores, on its own scene build: whole
    frames until `budget_s` of rendering has elapsed (>= 1 frame)."""
    from oracle.oracle import OracleScene
    t0 = time.perf_counter()
    scene, cam, par = build_oracle_workload(args)
    orc = OracleScene(scene)
    build_s = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    orc.render(cam, args.mode, par, threads=threads, rows=(0, 8))  # page in
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
            "cpu_model": cpu_model(),
            "sample": f"{frames} whole {cam.width}x{cam.height} {args.mode} frame(s) of "
                      f"{public_name(args.scene)} in {dt:.2f} s (oracle/oracle.c, OpenMP over "
                      f"rows, {threads} threads; scene built by oracle/build.c in {build_s:.1f} s)",
            "ms_per_frame": dt * 1000.0 / frames, "samples_per_frame": samples // frames}


def ncu_traffic(args):
    """DRAM bytes (read + write) per launch of march_sm_kernel on this
    workload, from an `ncu` subprocess (cold caches, --cache-control all);
    the largest of the frame's march launches (the unchosen lane width
    returns at once).  None when ncu is not available."""
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu"
                                  if Path("/usr/local/cuda/bin/ncu").exists() else None)
    if ncu is None or os.environ.get("TETRAY_BENCH_UNDER_NCU"):
        return None, "ncu not available"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:march_sm", "-c", "4", "--csv",
           sys.executable, str(ROOT / "bench.py"), "--scene", args.scene, "--mode", args.mode,
           "--scale", str(args.scale), "--steps", "1", "--warmup", "0", "--no-e2e", "--no-cpu",
           "--no-traffic"] + (["--host-build"] if args.host_build else [])
    env = dict(os.environ, TETRAY_BENCH_UNDER_NCU="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    except (OSError, subprocess.TimeoutExpired) as e:
        return None, f"ncu failed: {e}"
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith('"')]
    per = {}
    for row in csv.DictReader(io.StringIO("\n".join(lines))):
        try:
            v = float(row["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            continue
        unit = row.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                 "GB": 1e9}.get(unit, 1)
        per.setdefault(row["ID"], {})[row["Metric Name"]] = v * scale
    best = None
    for d in per.values():
        t = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        if best is None or t > best:
            best = t
    if best is None:
        return None, f"no march_sm launch in ncu output (rc {res.returncode})"
    return int(best), "ncu dram__bytes_read.sum + dram__bytes_write.sum, this workload"


# ------------------------------------------------------------ reference arm

def run_reference(args, rank, base_scale=None):
    """The stock reference render() on whole frames of the workload (the
    warm-up frames -- numba JIT, page-in -- at the N = 1 frame size)."""
    if rank != 0:
        return 0
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tetray_bench_numba")
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "tetray").exists():
        print(json.dumps({"impl": "reference",
                          "unavailable": "baseline/_ref (pip install --target baseline/_ref "
                                         "of /root/reference/pkg) is missing"}), flush=True)
        return 0
    sys.path.insert(0, str(ref))
    import cases as C
    import tetray
    from oracle.stock_scene import build_stock_scene
    n = scene_n(args.scene)
    t0 = time.perf_counter()
    if n >= 128 or args.scene.startswith("grid"):
        scene = build_stock_scene(tetray, n, C.radial16_tf_doc(n))
    else:
        scene = C.build_scene(tetray, public_name(args.scene))    # the stock Scene.build
    build_s = time.perf_counter() - t0
    cam = C.camera(tetray, public_name(args.scene), scale=args.scale)
    par = C.params(tetray, public_name(args.scene))
    threads = os.cpu_count() or 1
    cam_w = C.camera(tetray, public_name(args.scene),
                     scale=args.scale if base_scale is None else base_scale)
    for _ in range(args.warmup):   # the first frame also JIT-compiles the numba kernels
        tetray.render(scene, cam_w, args.mode, par, threads=threads)
    times, walls, samples = [], [], None
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fb, st = tetray.render(scene, cam, args.mode, par, threads=threads)
        times.append(time.perf_counter() - t0)
        walls.append(st.wall_ms)
        samples = st.total_samples
        if time.perf_counter() - t_start > args.ref_budget_s:
            break
    tot = sum(times)
    v = samples * len(times) / tot
    try:
        import numba
        nthreads = numba.config.NUMBA_NUM_THREADS
    except Exception:   # pragma: no cover
        nthreads = None
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
            "ms_per_step": tot * 1000.0 / len(times), "higher_is_better": True,
            "scaling": "weak" if args.gpus > 1 and args.scaling == "weak" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, scene.mesh.n_tets, len(scene.partitions), samples),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "cpu_model": cpu_model(), "numba_num_threads": nthreads,
                             "sample": f"{len(times)} whole frame(s) through the stock "
                                       f"tetray.render(threads={threads}) (numba)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "detail": {"scene_build_s": round(build_s, 2),
                       "render_wall_ms_median": statistics.median(walls),
                       "repo_libs_mapped": mapped_repo_libs(),
                       "steps_requested": args.steps,
                       "scene": "stock tetray dataclasses around oracle/build.c arrays"
                                if n >= 128 else "stock tetray Scene.build"}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------- record-sharded GPU arm

def run_records(args, world, rank, local):
    """--shard records: the frame over KD bricks (bricks.py):
    one brick per rank (NCCL state exchange per round, no host read between
    the first n rounds), or args.bricks bricks emulated one after another on
    one GPU.  value = samples / device time of the trace + rounds (max over
    ranks); the frame is checked against the one-GPU render() (bit-exact)."""
    import torch
    import torch.distributed as dist

    import cases as C
    import paper_1908_01906_b200 as B
    from paper_1908_01906_b200 import bricks as BR
    dev = dist_setup(local, world)
    name = public_name(args.scene)
    t0 = time.perf_counter()
    scene = C.build_scene(B, name)           # host build: bricks need the mesh arrays
    cam, par = C.camera(B, name, scale=args.scale), C.params(B, name)
    n = world if world > 1 else args.bricks
    br = BR.BrickRenderer(scene, n, max(par.s1, par.s2), device=dev,
                          dist=dist if world > 1 else None, exchange=args.exchange)
    setup_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        br.render(cam, args.mode, par)
    if world > 1:
        dist.barrier()
    ms, st = [], None
    for _ in range(args.steps):
        fb, st = br.render(cam, args.mode, par)
        ms.append(st.device_ms)
    t = torch.tensor([sum(ms) / 1000.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    one = B.render(scene, cam, args.mode, par, device=dev) if rank == 0 else None
    if rank == 0:
        exact = bool(np.array_equal(one[0].rgba, fb.rgba) and
                     np.array_equal(one[0].samples, fb.samples) and
                     one[1].total_samples == st.total_samples)
        value = st.total_samples * args.steps / float(t[0])
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": float(t[0]) * 1000.0 / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(args, scene.mesh.n_tets, scene.n_partitions,
                                          st.total_samples),
                "detail": {"parallelism": f"records: {n} KD bricks over {world} GPU(s)"
                                          + (" (emulated one after another)" if world == 1 else ""),
                           "rounds": br.rounds, "tets_per_brick": br.tets_per_brick,
                           "exact_vs_one_gpu_render": exact,
                           "one_gpu_frame_ms": one[1].device_ms,
                           "exchange": br.exchange if world > 1 else None,
                           "state_exchange_bytes_per_round": int(cam.width * cam.height * 64)
                           if world > 1 and br.exchange == "sum" else None,
                           "setup_s": round(setup_s, 2)}}
        print(json.dumps(line), flush=True)
    if world > 1:
        br.close()
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ GPU arm

def dist_setup(local: int, world: int):
    """The rank's device and process group.  TETRAY_DIST_BACKEND=gloo with
    TETRAY_ONE_DEVICE=1 runs every rank on cuda:0 (tests of the N > 1 path on
    a one-GPU box: NCCL refuses two ranks on one device)."""
    import torch
    import torch.distributed as dist
    one = os.environ.get("TETRAY_ONE_DEVICE") == "1"
    dev = torch.device("cuda", 0 if one else local)
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("TETRAY_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


def relaunch_distributed(argv) -> int:
    """`--gpus N` without a torchrun environment: run N ranks of this script."""
    args = parse(argv)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve())] + list(argv)
    return subprocess.call(cmd)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    base_scale = args.scale
    if args.shard == "pixels":
        weak_scale(args, world)
    if args.impl == "reference":
        return run_reference(args, rank, base_scale)
    if args.shard == "records":
        return run_records(args, world, rank, local)

    import torch
    import torch.distributed as dist

    import paper_1908_01906_b200 as B
    from paper_1908_01906_b200 import distributed as D
    from paper_1908_01906_b200.device import device_scene_for

    dev = dist_setup(local, world)
    nranks = dist.get_world_size() if world > 1 else 1

    scene, cam, par, build_s = build_gpu_workload(B, args)
    t0 = time.perf_counter()
    dscene = device_scene_for(scene, dev)
    upload_s = time.perf_counter() - t0
    mode_id = {"reference": 0, "skip": 1, "skip-adaptive": 2}[args.mode]
    track = args.mode != "reference"
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    runner = D.ShardedFrame(dscene, scene, cam, mode_id, par, track=track,
                            rank=rank if world > 1 else 0, world=world, flags=args.flags)
    for _ in range(args.warmup):
        runner.run(stream)
    torch.cuda.synchronize()
    total_samples = runner.total_samples() if rank == 0 else 0

    # timed region: K steps, L2 flushed between steps, frame timed with events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    mev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(dev.index) as clk:
        time.sleep(0.25)
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            ev[k][0].record(stream)
            runner.run(stream, kernel_events=kev[k], march_events=mev[k])
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        time.sleep(0.1)
    launches_per_step = runner.launches_per_step()
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

    # roofline of the dominant kernel (march_sm_kernel), per launch, rank 0's share
    hbm, peak_kind = peaks()
    my_samples = runner.local_samples()
    my_pixels = runner.local_pixels()
    rb = RECORD_BYTES[int(scene.mesh.centering)]
    alg_bytes = rb * my_samples + PIXEL_BYTES * my_pixels
    achieved = alg_bytes / m_local / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "peak_kind": peak_kind,
            "kernel": "march_sm_kernel", "kernel_ms": m_local * 1e3,
            "frame_kernels_ms": k_local * 1e3,
            "frame_frac": alg_bytes / k_local / 1e9 / hbm,
            "alg_bytes_per_launch": alg_bytes,
            "alg_bytes_model": f"{rb} B/sample x {my_samples} samples + {PIXEL_BYTES} B/pixel x "
                               f"{my_pixels} pixels (SURVEY.md §8d)"}

    # e2e through the public render(): epoch H2D + outputs D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        if world > 1:
            e2e = D.bench_e2e_sharded(scene, cam, args.mode, par, args.steps, dev)
        else:
            fb = None
            for _ in range(max(args.warmup, 10)):
                dscene.mark_epochs_stale()
                fb, st = B.render(scene, cam, args.mode, par, device=dev)
            per = []
            # wall clock: enough steps for a stable mean (~1 s of frames, 20-200)
            frame_s = t_max / args.steps
            e2e_steps = max(args.steps, 20, min(200, int(1.0 / max(frame_s, 1e-6))))
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                t1 = time.perf_counter()
                dscene.mark_epochs_stale()  # every step copies the metadata epoch again
                fb, st = B.render(scene, cam, args.mode, par, device=dev)
                per.append(time.perf_counter() - t1)
            dt = time.perf_counter() - t0
            ep = next(iter(dscene._epochs.values()))
            d2h = fb.rgba.nbytes + fb.samples.nbytes + 8 * (3 + scene.n_partitions)
            e2e = {"value": st.total_samples * e2e_steps / dt, "unit": UNIT,
                   "h2d_bytes_per_step": int(ep.h2d_bytes), "d2h_bytes_per_step": int(d2h),
                   "ms_per_step": dt * 1000.0 / e2e_steps, "steps": e2e_steps,
                   "ms_per_step_median": statistics.median(per) * 1000.0,
                   "ms_per_step_min": min(per) * 1000.0}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference(args, args.cpu_seconds)
        if cpu["samples_per_frame"] != total_samples:
            raise RuntimeError(f"oracle frame has {cpu['samples_per_frame']} samples, the GPU "
                               f"frame {total_samples}")

    if rank == 0 and not args.no_traffic:
        if world > 1:   # the ncu pass profiles a one-GPU frame: N = 1 lines carry it
            roof["traffic_source"] = "not measured at N > 1 (see the N = 1 line)"
        else:
            roof["traffic"], roof["traffic_source"] = ncu_traffic(args)
            if roof["traffic"]:
                roof["traffic_per_sample"] = roof["traffic"] / max(my_samples, 1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max * 1000.0 / args.steps, "higher_is_better": True,
            "scaling": "weak" if world > 1 and args.scaling == "weak" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, scene.mesh.n_tets, scene.n_partitions,
                                      total_samples),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "detail": {"l2": "flushed between steps (256 MiB write)",
                       "rays_per_s": cam.width * cam.height * args.steps / t_max,
                       "n_active": int(scene.meta_state()[0].sum()),
                       "parallelism": f"pixel tiles interleaved over {world} GPU(s)",
                       "scaling_rule": "frame side x sqrt(N) (--scaling weak)"
                       if world > 1 and args.scaling == "weak" else "one frame split N ways",
                       "comm_nranks": nranks, "flags": hex(args.flags),
                       "scene_path": type(scene).__name__,
                       "scene_build_s": round(build_s, 3), "upload_s": round(upload_s, 3),
                       "resident_bytes": int(dscene.resident_bytes)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
