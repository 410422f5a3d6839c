"""Bit-exact GPU vs oracle on a multi-chunk frame (radial59 at 1024^2 and 1536^2,
all modes; a 1536^2 frame exceeds one 1M-ray chunk)."""
import hashlib, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import cases as C
import paper_1908_01906_b200 as B
from oracle.oracle import OracleScene

sc = C.build_scene(B, "radial59")
orc = OracleScene(sc)
par = C.params(B, "radial59")
for scale in (2, 3):
    cam = C.camera(B, "radial59", scale=scale)
    for mode in ("reference", "skip", "skip-adaptive"):
        t0 = time.time(); ref = orc.render(cam, mode, par); tc = time.time() - t0
        fb, st = B.render(sc, cam, mode, par)
        ok = (np.array_equal(fb.rgba, ref[0]) and np.array_equal(fb.samples, ref[1])
              and st.total_samples == int(ref[1].sum())
              and st.partitions_visited_mean == float(ref[2].mean())
              and (ref[3] is None or np.array_equal(st.per_partition_samples, ref[3])))
        print(f"{cam.width}x{cam.height} {mode:14s} exact={ok} samples={st.total_samples} "
              f"gpu_wall={st.wall_ms:.2f}ms device={st.device_ms:.3f}ms cpu={tc:.2f}s", flush=True)
