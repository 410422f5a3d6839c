"""Host-side cost of the public render() on the GPU box: per-call wall time
vs device time, and a cProfile of 300 calls (the epoch re-uploaded each call,
as bench.py's end-to-end steps do)."""
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402

import cases as C  # noqa: E402
import paper_1908_01906_b200 as B  # noqa: E402
from paper_1908_01906_b200.device import device_scene_for  # noqa: E402

scene = sys.argv[1] if len(sys.argv) > 1 else "radial59"
sc = C.build_scene(B, scene)
cam, par = C.camera(B, scene), C.params(B, scene)
dev = device_scene_for(sc)
for _ in range(20):
    dev.mark_epochs_stale()
    B.render(sc, cam, "skip-adaptive", par)
wall, devm = [], []
for _ in range(300):
    dev.mark_epochs_stale()
    t0 = time.perf_counter()
    fb, st = B.render(sc, cam, "skip-adaptive", par)
    wall.append((time.perf_counter() - t0) * 1e3)
    devm.append(st.device_ms)
print(f"{scene}: render() median {np.median(wall):.3f} ms, device {np.median(devm):.3f} ms, "
      f"host {np.median(np.array(wall) - np.array(devm)) * 1e3:.0f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    dev.mark_epochs_stale()
    B.render(sc, cam, "skip-adaptive", par)
pr.disable()
buf = io.StringIO()
pstats.Stats(pr, stream=buf).sort_stats("tottime").print_stats(25)
print(buf.getvalue())
