"""Point-location build: host (host_build.cpp + upload) vs device
(csrc/pbuild.cu) on general meshes -- time until the scene is device-resident
and the skip-adaptive / reference frame times on each build.  One JSON line
per (scene, build).  Usage: python scripts/pbuild_timing.py radial128 jitter59 ..."""
import gc
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

import cases as C  # noqa: E402
import paper_1908_01906_b200 as B  # noqa: E402
from paper_1908_01906_b200.device import _CACHE_ATTR, device_scene_for  # noqa: E402


def frame_ms(sc, recipe, mode, n=8):
    cam, par = C.camera(B, recipe), C.params(B, recipe)
    B.render(sc, cam, mode, par)
    ts, tot = [], None
    for _ in range(n):
        _, st = B.render(sc, cam, mode, par)
        ts.append(st.device_ms)
        tot = st.total_samples
    return statistics.median(ts), tot


for recipe in sys.argv[1:]:
    t0 = time.perf_counter()
    sc = C.build_scene(B, recipe)
    scene_s = time.perf_counter() - t0
    res = {}
    for build in ("device", "device-nowalk", "device-hostwalk", "host"):
        getattr(sc, _CACHE_ATTR, {}).clear()
        gc.collect()
        torch.cuda.empty_cache()
        sc.point_build = build
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev = device_scene_for(sc)
        torch.cuda.synchronize()
        ready = time.perf_counter() - t0
        row = {"scene": recipe, "n_tets": int(sc.mesh.n_tets), "build": build,
               "scene_build_s": round(scene_s, 2), "ready_s": round(ready, 3),
               "upload_s": round(getattr(dev, "upload_s", float("nan")), 3),
               "n_leaves": int(dev.desc.n_pleaves), "n_nodes": int(dev.desc.n_pnodes),
               "grid_coverage": round(float(getattr(dev.grid, "coverage", float("nan"))), 4),
               "cell_lists": dev.cells is not None,
               "phases": {k: round(v, 3) for k, v in getattr(dev, "build_phases", {}).items()}}
        for mode in ("skip-adaptive", "reference"):
            ms, tot = frame_ms(sc, recipe, mode)
            row[f"{mode}_ms"] = round(ms, 4)
            row[f"{mode}_samples"] = tot
        res[build] = row
        print(json.dumps(row), flush=True)
    for mode in ("skip-adaptive", "reference"):
        for b in ("device", "device-nowalk", "device-hostwalk"):
            assert res[b][f"{mode}_samples"] == res["host"][f"{mode}_samples"], (recipe, b, mode)
    del sc
    gc.collect()
    torch.cuda.empty_cache()
