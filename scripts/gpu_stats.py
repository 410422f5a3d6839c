"""Kernel event statistics for the benchmark scene in each mode (debug aid)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import _lib

scene = sys.argv[1] if len(sys.argv) > 1 else "radial59"
sc = C.build_scene(B, scene)
cam, par = C.camera(B, scene), C.params(B, scene)
out = np.zeros(32, np.int64)
for mode in ("reference", "skip", "skip-adaptive"):
    for flags in (0x0,):
        _lib.lib().tr_kernel_stats(_lib.ptr(out, __import__("ctypes").c_int64), 32, 1)
        fb, st = B.render(sc, cam, mode, par, flags=flags | _lib.TR_FLAG_STATS)
        _lib.check(_lib.lib().tr_kernel_stats(_lib.ptr(out, __import__("ctypes").c_int64), 32, 1), "stats")
        d = dict(zip(_lib.STAT_NAMES, out.tolist()))
        print(scene, mode, hex(flags), "samples", st.total_samples, d, flush=True)
