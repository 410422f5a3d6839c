"""Trace-pass cost per 32-ray tile (TR_FLAG_TILE_TIMING): sum and max of SM
cycles per tile, i.e. how much of the trace kernel is its longest tile."""
import ctypes, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import _lib
out = np.zeros(32, np.int64)
for scene in sys.argv[1:] or ["radial59"]:
    sc = C.build_scene(B, scene)
    cam, par = C.camera(B, scene), C.params(B, scene)
    for mode in ("reference", "skip", "skip-adaptive"):
        for rep in range(2):
            _lib.lib().tr_kernel_stats(_lib.ptr(out, ctypes.c_int64), 32, 1)
            fb, st = B.render(sc, cam, mode, par, flags=0x10000)
            _lib.check(_lib.lib().tr_kernel_stats(_lib.ptr(out, ctypes.c_int64), 32, 1), "stats")
        d = dict(zip(_lib.STAT_NAMES, out.tolist()))
        tiles = (cam.width * cam.height + 31) // 32
        q_ms = (d["march_tq"] - d["march_t0"]) / 1e6 if d["march_tq"] > d["march_t0"] else float("nan")
        m_ms = (d["march_t1"] - d["march_t0"]) / 1e6
        print(scene, mode, "tiles", tiles, "avg cycles", d["tile_cycles"] / tiles, "max", d["tile_max_cycles"],
              "| march", round(m_ms, 3), "ms, queue empty after", round(q_ms, 3), "ms",
              "| device ms", round(st.device_ms, 3), flush=True)
