"""Where render()'s host time goes on the GPU box: wall time of the public
render() vs the tr_render_sync call inside it vs the device frame (events),
with the epoch re-uploaded each call (bench.py's end-to-end steps).
Usage: python scripts/e2e_phases.py [scene ...]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402

import cases as C  # noqa: E402
import paper_1908_01906_b200 as B  # noqa: E402
from paper_1908_01906_b200 import _lib  # noqa: E402
from paper_1908_01906_b200.device import device_scene_for  # noqa: E402

lib = _lib.lib()
real = lib.tr_render_sync
call_ms = []


class Timed:
    def __call__(self, *a):
        t0 = time.perf_counter()
        rc = real(*a)
        call_ms.append((time.perf_counter() - t0) * 1e3)
        return rc


lib.tr_render_sync = Timed()
for scene in (sys.argv[1:] or ["radial59"]):
    sc = C.build_scene(B, scene)
    cam, par = C.camera(B, scene), C.params(B, scene)
    dev = device_scene_for(sc)
    for stale in (True, False):
        for _ in range(30):
            dev.mark_epochs_stale()
            B.render(sc, cam, "skip-adaptive", par)
        call_ms.clear()
        wall, devm = [], []
        for _ in range(300):
            if stale:
                dev.mark_epochs_stale()
            t0 = time.perf_counter()
            fb, st = B.render(sc, cam, "skip-adaptive", par)
            wall.append((time.perf_counter() - t0) * 1e3)
            devm.append(st.device_ms)
        w, c, d = np.median(wall), np.median(call_ms), np.median(devm)
        print(f"{scene} stale={stale}: render() {w:.3f} ms, tr_render_sync {c:.3f} ms, "
              f"device {d:.3f} ms -> python {1e3 * (w - c):.0f} us, C around the frame "
              f"{1e3 * (c - d):.0f} us, e2e/device {w / d:.3f}", flush=True)
