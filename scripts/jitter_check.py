"""Unstructured-mesh check (GPU box): jitterN = radialN with interior vertices
moved up to 0.2 cell.  Bit-exact against the oracle in all modes, plus the
device time and point-location statistics next to the structured radialN."""
import ctypes, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import _lib
from oracle.oracle import OracleScene

out = np.zeros(32, np.int64)
for name in sys.argv[1:] or ["jitter16", "jitter59", "radial59"]:
    sc = C.build_scene(B, name)
    cam, par = C.camera(B, name), C.params(B, name)
    orc = OracleScene(sc)
    for mode in ("reference", "skip", "skip-adaptive"):
        ref = orc.render(cam, mode, par)
        fb, st = B.render(sc, cam, mode, par)
        exact = (np.array_equal(fb.rgba, ref[0]) and np.array_equal(fb.samples, ref[1]) and
                 st.partitions_visited_mean == float(ref[2].mean()) and
                 (ref[3] is None or np.array_equal(st.per_partition_samples, ref[3])))
        ms, ms_nc = [], []
        for _ in range(3):
            fb, st = B.render(sc, cam, mode, par)
            ms.append(st.device_ms)
            fb2, st2 = B.render(sc, cam, mode, par, flags=0x20000)   # cell lists off
            ms_nc.append(st2.device_ms)
            exact = exact and np.array_equal(fb2.rgba, ref[0]) and np.array_equal(fb2.samples, ref[1])
        _lib.lib().tr_kernel_stats(_lib.ptr(out, ctypes.c_int64), 32, 1)
        B.render(sc, cam, mode, par, flags=_lib.TR_FLAG_STATS)
        _lib.check(_lib.lib().tr_kernel_stats(_lib.ptr(out, ctypes.c_int64), 32, 1), "stats")
        d = dict(zip(_lib.STAT_NAMES, out.tolist()))
        print(f"{name:9s} {mode:14s} exact={exact} samples={st.total_samples} device_ms={min(ms):.3f} "
              f"no_cells_ms={min(ms_nc):.3f} "
              f"grid_hits={d['grid_hits']} descents={d['descents']}", flush=True)
