#!/usr/bin/env python3
"""Generate the parity fixtures by running the REFERENCE renderer (tetray).

Run in the build container, where /root/reference exists (it is absent on the
GPU box; the fixtures this writes are committed instead):

    python tests/golden/make_golden.py [--big]

The reference is imported from a scratch copy (/tmp/tetray_ref) because its
numba cache must be writable.  For every recipe in tests/cases.py it records
the scene arrays' hashes and, per frame case and mode, the exact outputs of
_kernels.render_frame (pkg/src/tetray/_kernels.py:312-398) called with the
argument list render() assembles (pkg/src/tetray/render.py:183-193):
sha256 of rgba / samples / visited / per-partition samples, the totals, and
(small cases) the full arrays.  Plus point-location, traversal, scalar-formula
and jitter-hash vectors, and the two CLI golden images that
pkg/scripts/make_golden.py would write (absent from the reference tree).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
TESTS = HERE.parent
REF_SRC = Path("/root/reference/pkg")
SCRATCH = Path("/tmp/tetray_ref")


def _import_reference():
    if not REF_SRC.exists():
        sys.exit("the reference tree /root/reference is not present (generate fixtures in "
                 "the build container)")
    if not SCRATCH.exists():
        shutil.copytree(REF_SRC, SCRATCH)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tetray_ref_numba")
    sys.path.insert(0, str(SCRATCH / "src"))
    sys.path.insert(0, str(SCRATCH / "tests"))
    sys.path.insert(0, str(TESTS))
    import tetray  # noqa: F401
    return tetray


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def scene_hashes(scene) -> dict:
    offs = np.cumsum([0] + [len(p.element_ids) for p in scene.partitions])
    ids = np.concatenate([p.element_ids for p in scene.partitions])
    lo = np.stack([p.bounds.lo for p in scene.partitions])
    hi = np.stack([p.bounds.hi for p in scene.partitions])
    vr = np.array([p.value_range for p in scene.partitions])
    active, sigma, tf = scene.meta_state()
    return {"n_tets": int(scene.mesh.n_tets), "n_parts": len(scene.partitions),
            "part_offsets": sha(offs.astype(np.int64)), "part_ids": sha(ids.astype(np.int64)),
            "part_lo": sha(lo), "part_hi": sha(hi), "part_vrange": sha(vr),
            "active": sha(active.astype(np.uint8)), "sigma": sha(sigma),
            "tet_orig": sha(scene.sampler.tet_orig), "tet_inv": sha(scene.sampler.tet_inv),
            "field": sha(scene.mesh.field), "tf_table": sha(tf.table),
            "epsilon": float(scene.traversal_config.epsilon),
            "n_active": int(active.sum()), "n_sigma_lt1": int((sigma < 1).sum())}


def ref_frame(tetray, scene, cam, mode, params, jitter):
    """Direct call of the numba kernel, as render() makes it (R:169-193)."""
    from tetray import _kernels
    from tetray.render import _MODE_IDS
    active, sigma, tf = scene.meta_state()
    w, h = cam.width, cam.height
    right, up, fwd = cam.basis()
    tan_half = math.tan(math.radians(cam.fov_y_deg) / 2.0)
    P = len(scene.partitions)
    track = mode != "reference"
    rgba = np.zeros((h, w, 4))
    samples = np.zeros((h, w), np.int64)
    visited = np.zeros((h, w), np.int32)
    ppart = np.zeros((h, P if track else 1), np.int64)
    _kernels.render_frame(
        cam.position, np.ascontiguousarray(right), np.ascontiguousarray(up),
        np.ascontiguousarray(fwd), tan_half, w / h, w, h, jitter, _MODE_IDS[mode], params.s1,
        params.s2, params.p, params.termination_opacity, scene.traversal_config.epsilon,
        scene.background, tf.table, tf.domain[0], tf.domain[1], scene.mesh.bounds.lo,
        scene.mesh.bounds.hi, *scene.bvh.kernel_args(), active, sigma,
        *scene.sampler.kernel_args(), rgba, samples, visited, ppart, track)
    return rgba, samples, visited, (ppart.sum(axis=0) if track else None)


def frame_record(tetray, scene, cam, mode, params, jitter):
    from tetray.render import render
    rgba, samples, visited, ppart = ref_frame(tetray, scene, cam, mode, params, jitter)
    fb, st = render(scene, cam, mode, params, jitter=jitter)  # the public API agrees
    assert np.array_equal(fb.rgba, rgba) and st.total_samples == int(samples.sum())
    rec = {"rgba": sha(rgba), "samples": sha(samples), "visited": sha(visited),
           "total_samples": int(samples.sum()), "visited_sum": int(visited.sum()),
           "partitions_visited_mean": float(visited.mean()),
           "ppart": None if ppart is None else sha(ppart.astype(np.int64)),
           "ppart_list": None if ppart is None else ppart.astype(np.int64).tolist()
           if len(ppart) <= 1024 else None,
           "rgba_sum": float(rgba.sum())}
    return rec, (rgba, samples, visited, ppart)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also render radial59 (~1 min)")
    args = ap.parse_args()
    tetray = _import_reference()
    import cases as C

    # the bundled TF fixture the radialN recipes scale (T/golden/radial16_tf.json)
    shutil.copy(SCRATCH / "tests" / "golden" / "radial16_tf.json", HERE / "radial16_tf.json")

    out = {"generator": "tests/golden/make_golden.py", "reference": "tetray 0.1.0 (numba)",
           "scenes": {}, "frames": {}}
    arrays = {}
    recipes = sorted({r for _, r, _, _ in C.FRAME_CASES} | ({"radial59"} if args.big else set()))
    scenes = {}
    for r in recipes:
        scenes[r] = C.build_scene(tetray, r)
        out["scenes"][r] = scene_hashes(scenes[r])
        print("scene", r, out["scenes"][r]["n_parts"], "partitions", flush=True)
    cases = C.FRAME_CASES + (C.BIG_CASES if args.big else [])
    for cid, r, modes, jitter in cases:
        sc, cam, par = scenes[r], C.camera(tetray, r), C.params(tetray, r)
        for mode in modes:
            rec, arr = frame_record(tetray, sc, cam, mode, par, jitter)
            out["frames"][f"{cid}/{mode}"] = rec
            if cid in C.FULL_ARRAY_CASES:
                key = f"{cid}/{mode}"
                arrays[key + "/rgba"], arrays[key + "/samples"] = arr[0], arr[1]
                arrays[key + "/visited"] = arr[2]
                if arr[3] is not None:
                    arrays[key + "/ppart"] = arr[3]
            print("frame", cid, mode, rec["total_samples"], flush=True)
    if not args.big:  # keep previously generated big-case records
        old = HERE / "reference_frames.json"
        if old.exists():
            prev = json.loads(old.read_text())
            for k, v in prev.get("frames", {}).items():
                if k.startswith("radial59/"):
                    out["frames"][k] = v
            if "radial59" in prev.get("scenes", {}):
                out["scenes"]["radial59"] = prev["scenes"]["radial59"]
    (HERE / "reference_frames.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    np.savez_compressed(HERE / "reference_small.npz", **arrays)

    # ---- point location (K:93-170)
    from tetray import _kernels
    pts_out = {}
    for r, n in (("golden_radial4", 4000), ("radial16", 4000), ("voidcell", 2000),
                 ("sinus", 2000)):
        sc = scenes[r]
        pts = C.point_set(sc, n, seed=20240817)
        found, vals = sc.sampler.sample_many(pts)
        tet = np.array([sc.sampler.locate(p)[0] for p in pts], dtype=np.int64)
        pts_out[f"{r}/pts"], pts_out[f"{r}/found"] = pts, found
        pts_out[f"{r}/vals"], pts_out[f"{r}/tet"] = vals, tet
    np.savez_compressed(HERE / "reference_points.npz", **pts_out)

    # ---- traversal (K:173-259), scalar formulas (K:20-27), jitter hash (K:300-309)
    misc = {}
    rng = np.random.default_rng(20240817)
    sc = scenes["radial16"]
    active, _, _ = sc.meta_state()
    rays = []
    for _ in range(300):
        o = rng.uniform(-4.0, 20.0, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        ids = np.empty(600, np.int64)
        en = np.empty(600)
        ex = np.empty(600)
        k = _kernels.trace_intervals(o[0], o[1], o[2], d[0], d[1], d[2], 0.0, math.inf,
                                     sc.traversal_config.epsilon, *sc.bvh.kernel_args(), active,
                                     ids, en, ex)
        rays.append({"o": o.tolist(), "d": d.tolist(), "ids": ids[:k].tolist(),
                     "enter": en[:k].tolist(), "exit": ex[:k].tolist()})
    misc["trace_radial16"] = rays
    s1 = rng.uniform(1e-3, 1.0, 2000)
    s2 = s1 + rng.uniform(0.0, 2.0, 2000)
    p = rng.uniform(1.0, 8.0, 2000)
    sig = rng.uniform(0.0, 2.0, 2000)
    alpha = rng.uniform(0.0, 1.0, 2000)
    k = rng.uniform(1.0, 10.0, 2000)
    misc["step_size"] = [[a, b, c, d, float(_kernels.step_size(a, b, c, d))]
                         for a, b, c, d in zip(s1, s2, p, sig)]
    misc["opacity_correction"] = [[a, s * kk, s, float(_kernels.opacity_correction(a, s * kk, s))]
                                  for a, s, kk in zip(alpha, s1, k)]
    hs = [(int(x), int(y)) for x, y in rng.integers(0, 8192, size=(500, 2))]
    hs += [(x, y) for x in range(8) for y in range(8)]
    misc["hash01"] = [[x, y, float(_kernels._hash01(x, y))] for x, y in hs]
    (HERE / "reference_misc.json").write_text(json.dumps(misc) + "\n")

    # ---- the CLI golden images (pkg/scripts/make_golden.py, T/golden_scene.py)
    from golden_scene import write_golden_scene
    from tetray.cli import main as cli_main
    with tempfile.TemporaryDirectory() as tmp:
        scene_path = write_golden_scene(Path(tmp))
        rc = cli_main(["render", "--scene", str(scene_path), "--out",
                       str(HERE / "radial4_skip_adaptive.ppm"), "--heatmap",
                       str(HERE / "radial4_heatmap.ppm")])
        assert rc == 0
    print("wrote fixtures to", HERE)
    return 0


if __name__ == "__main__":
    sys.exit(main())
