import sys, ctypes
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
import numpy as np
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import _lib
out = np.zeros(32, np.int64)
for scene in sys.argv[1:]:
    sc = C.build_scene(B, scene)
    cam, par = C.camera(B, scene), C.params(B, scene)
    for mode in ("reference", "skip", "skip-adaptive"):
        _lib.lib().tr_kernel_stats(_lib.ptr(out, ctypes.c_int64), 32, 1)
        fb, st = B.render(sc, cam, mode, par, flags=_lib.TR_FLAG_STATS)
        _lib.check(_lib.lib().tr_kernel_stats(_lib.ptr(out, ctypes.c_int64), 32, 1), "stats")
        d = dict(zip(_lib.STAT_NAMES, out.tolist()))
        marching = int((fb.samples > 0).sum())
        print(scene, mode, "samples", st.total_samples, "marching rays", marching, "max/ray", int(fb.samples.max()), d["max_ray_samples"], flush=True)
