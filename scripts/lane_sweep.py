"""Lanes per ray (G) vs frame time per scene: mean / max samples per marching
ray and the device frame ms for auto, 4, 8 and 16 lanes (skip-adaptive 512^2)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402

import cases as C  # noqa: E402
import paper_1908_01906_b200 as B  # noqa: E402

for scene in sys.argv[1:] or ["radial59", "grid128", "grid272"]:
    sc = C.build_scene(B, scene)
    cam, par = C.camera(B, scene), C.params(B, scene)
    for mode in ("skip-adaptive", "reference"):
        fb, st = B.render(sc, cam, mode, par)
        s = fb.samples[fb.samples > 0]
        line = [scene, mode, f"rays {len(s)}", f"mean {s.mean():.0f}", f"max {s.max()}"]
        for name, flags in (("auto", 0), ("G4", 0x200), ("G8", 0x300), ("G16", 0x400)):
            ms = []
            for _ in range(8):
                fb, st = B.render(sc, cam, mode, par, flags=flags)
                ms.append(st.device_ms)
            line.append(f"{name} {min(ms):.3f}")
        print("  ".join(line), flush=True)
    del sc
