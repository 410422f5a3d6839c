"""Per-step distribution of the public render() time and of its phases
(GPU box; finds where the e2e outliers come from)."""
import gc, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import torch
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import device as DV

sc = C.build_scene(B, "radial59")
cam, par = C.camera(B, "radial59"), C.params(B, "radial59")
dev = DV.device_scene_for(sc)
for _ in range(5):
    dev._epochs.clear(); B.render(sc, cam, "skip-adaptive", par)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
gc_off = len(sys.argv) > 2 and sys.argv[2] == "nogc"
FLAGS = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0
if gc_off:
    gc.disable()
tot, dms = [], []
for _ in range(N):
    t = time.perf_counter()
    dev._epochs.clear()
    fb, st = B.render(sc, cam, "skip-adaptive", par, flags=FLAGS)
    tot.append((time.perf_counter() - t) * 1e3)
    dms.append(st.device_ms)
tot, dms = np.array(tot), np.array(dms)
def q(a):
    return " ".join(f"{x:6.3f}" for x in np.percentile(a, [0, 10, 50, 90, 99, 100])) + f"  mean {a.mean():6.3f}"
print("gc", "off" if gc_off else "on", "flags", hex(FLAGS), "  percentiles 0/10/50/90/99/100")
print("render() ms ", q(tot))
print("device ms   ", q(dms))
print("host ms     ", q(tot - dms))
big = np.argsort(tot)[-8:]
print("slowest steps:", [(int(i), round(float(tot[i]), 3), round(float(dms[i]), 3)) for i in sorted(big)])
