"""Reference fixtures for BASELINE configs 3 and 5 -- run the
REFERENCE package (a scratch copy of /root/reference/pkg, numba) and record the
sha256 of its scene arrays and of its frames' outputs.

    python tests/golden/make_golden_big.py [--only radial128,radial272,radial59_1536]

  radial128        10.5M tets: scene hashes + 512^2 frames in all three modes
  radial272        100.6M tets: scene hashes + 512^2 skip-adaptive, skip and
                   reference frames (the reference's Scene.build takes ~40 min
                   and ~40 GB of RAM here; frames ~20-60 s each on 8 threads)
  radial59_1536    radial59 at 1536^2 in all three modes (config 5, multi-chunk)

Output: tests/golden/reference_big.json (merged with what is already there, so
the recipes can be produced in separate runs).  The frames are the numba
kernel called as render() calls it (make_golden.ref_frame, R:169-193), checked
against render() itself for the 512^2 recipes.
"""

from __future__ import annotations

import argparse
import gc
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import make_golden as G  # noqa: E402

OUT = HERE / "reference_big.json"

RECIPES = {
    "radial128": ("radial128", 1.0, ("skip-adaptive", "skip", "reference")),
    "radial272": ("radial272", 1.0, ("skip-adaptive", "skip", "reference")),
    "radial59_1536": ("radial59", 3.0, ("skip-adaptive", "skip", "reference")),
}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="radial128,radial59_1536,radial272")
    args = ap.parse_args()
    tetray = G._import_reference()
    import cases as C

    out = json.loads(OUT.read_text()) if OUT.exists() else {
        "generator": "tests/golden/make_golden_big.py", "reference": "tetray 0.1.0 (numba)",
        "scenes": {}, "frames": {}, "timing_s": {}}
    for rid in args.only.split(","):
        scene_name, scale, modes = RECIPES[rid]
        t0 = time.perf_counter()
        sc = C.build_scene(tetray, scene_name)
        out["timing_s"][f"{scene_name}/build"] = time.perf_counter() - t0
        out["scenes"][scene_name] = G.scene_hashes(sc)
        print("scene", scene_name, out["scenes"][scene_name]["n_parts"], "partitions",
              f"{out['timing_s'][scene_name + '/build']:.1f} s", flush=True)
        cam, par = C.camera(tetray, scene_name, scale=scale), C.params(tetray, scene_name)
        for mode in modes:
            t0 = time.perf_counter()
            if scale == 1.0 and scene_name != "radial272":
                rec, _ = G.frame_record(tetray, sc, cam, mode, par, False)
            else:
                rgba, samples, visited, ppart = G.ref_frame(tetray, sc, cam, mode, par, False)
                rec = {"rgba": G.sha(rgba), "samples": G.sha(samples), "visited": G.sha(visited),
                       "total_samples": int(samples.sum()), "visited_sum": int(visited.sum()),
                       "partitions_visited_mean": float(visited.mean()),
                       "ppart": None if ppart is None else G.sha(ppart.astype("int64")),
                       "ppart_list": None, "rgba_sum": float(rgba.sum())}
            key = f"{rid}/{mode}"
            out["frames"][key] = rec
            out["timing_s"][key] = time.perf_counter() - t0
            print("frame", key, rec["total_samples"], f"{out['timing_s'][key]:.1f} s", flush=True)
            OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
        del sc
        gc.collect()
    OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
