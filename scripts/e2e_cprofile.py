"""cProfile of the public render() loop (host-side overhead; GPU box)."""
import cProfile, pstats, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import device as DV
sc = C.build_scene(B, "radial59")
cam, par = C.camera(B, "radial59"), C.params(B, "radial59")
dev = DV.device_scene_for(sc)
fb = None
for _ in range(5):
    dev._epochs.clear(); fb, st = B.render(sc, cam, "skip-adaptive", par)
def loop():
    fb = None
    for _ in range(300):
        dev._epochs.clear()
        fb, st = B.render(sc, cam, "skip-adaptive", par)
pr = cProfile.Profile()
pr.enable(); loop(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
