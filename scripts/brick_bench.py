"""Record-sharded (KD-brick) frames, one device emulating n bricks (SURVEY
§8f row f4).  Per config: the one-device frame, the brick frame (all bricks
one after another), rounds, per-brick resident bytes, and the n-GPU critical
path estimate = trace + sum over rounds of the slowest brick's run (plus the
state exchange: rays x 64 B int64 all-reduce per round, not timed here), and
the PEER-exchange estimate: per round the slowest brick's run plus its pushes
(rays it marched x 64 B, each to the one rank of the ray's next run, at
NVLINK_GBS) plus one barrier (BARRIER_MS) -- an upper bound, the stores
overlap the march.
Usage: python scripts/brick_bench.py [scene ...] -> JSON lines."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import torch
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import bricks as BR

NVLINK_GBS = 720.0   # ~80% of NVLink 5's 900 GB/s per direction (nominal; not measured here)
BARRIER_MS = 0.015   # one small NCCL all-reduce over NVSwitch (nominal)

for name in (sys.argv[1:] or ["radial59"]):
    t0 = time.perf_counter()
    sc = C.build_scene(B, name)
    build_s = time.perf_counter() - t0
    cam, par = C.camera(B, name), C.params(B, name)
    for n in (2, 4, 8):
        t0 = time.perf_counter()
        br = BR.BrickRenderer(sc, n, max(par.s1, par.s2))
        setup_s = time.perf_counter() - t0
        for mode in ("reference", "skip-adaptive"):
            one = B.render(sc, cam, mode, par)
            for _ in range(2):
                B.render(sc, cam, mode, par)
                br.render(cam, mode, par)
            one_ms = [B.render(sc, cam, mode, par)[1].device_ms for _ in range(5)]
            fbs = [br.render(cam, mode, par, profile=True) for _ in range(5)]
            fb, st = fbs[-1]
            exact = bool(np.array_equal(fb.rgba, one[0].rgba) and np.array_equal(fb.samples, one[0].samples)
                         and st.total_samples == one[1].total_samples)
            prof = br.profile
            per_round = {}
            for r, b, ms in prof["runs"]:
                per_round.setdefault(r, []).append(ms)
            crit = prof["trace_ms"] + sum(max(v) for v in per_round.values())
            runs = {(r, b): ms for r, b, ms in prof["runs"]}
            push = {(r, b): q * 64 for r, b, q in prof["queued"]}
            rounds_peer = {}
            for (r, b), ms in runs.items():
                t = ms + push.get((r, b), 0) / (NVLINK_GBS * 1e6)
                rounds_peer[r] = max(rounds_peer.get(r, 0.0), t)
            crit_peer = prof["trace_ms"] + sum(rounds_peer.values()) + BARRIER_MS * len(rounds_peer)
            print(json.dumps({
                "scene": name, "n_tets": int(sc.mesh.n_tets), "bricks": n, "mode": mode,
                "exact": exact, "samples": int(st.total_samples), "rounds": br.rounds,
                "one_device_ms": float(np.median(one_ms)),
                "brick_frame_ms_emulated": float(np.median([f[1].device_ms for f in fbs])),
                "trace_ms": prof["trace_ms"], "n_gpu_critical_path_ms": crit,
                "n_gpu_critical_path_peer_ms_est": crit_peer,
                "peer_push_bytes_per_round_max": max(push.values()) if push else 0,
                "round_ms": {str(r): [round(x, 4) for x in v] for r, v in per_round.items()},
                "tets_per_brick": br.tets_per_brick,
                "max_brick_fraction": max(br.tets_per_brick) / sc.mesh.n_tets,
                "resident_bytes_per_brick": list(br.resident_bytes().values()),
                "state_exchange_bytes_per_round": int(512 * 512 * 64),
                "scene_build_s": round(build_s, 2), "brick_setup_s": round(setup_s, 2)}), flush=True)
        del br
        torch.cuda.empty_cache()
