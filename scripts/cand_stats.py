"""Candidate-raster statistics of one frame (GPU box): slabs per ray."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200.device import device_scene_for
for name in sys.argv[1:] or ["radial59"]:
    sc = C.build_scene(B, name)
    cam, par = C.camera(B, name), C.params(B, name)
    for mode in ("skip", "skip-adaptive"):
        fb, st = B.render(sc, cam, mode, par)
        dev = device_scene_for(sc)
        f = dev._frames[(cam.width, cam.height, 0)]
        n = -(-cam.width * cam.height // 32) * 32
        off = 1024 + n * (64 * 16 + 8 + 4 + 4)  # ccount after rec|tail|cnt|order
        cc = f.scratch[off:off + 4 * n].cpu().numpy().view(np.uint32)
        iv = f.scratch[1024 + n * (64 * 16 + 8):1024 + n * (64 * 16 + 12)].cpu().numpy().view(np.uint32) & 0xffff
        hit = cc[cc > 0]
        print(name, mode, "rays", n, "with cands", len(hit), "mean", hit.mean(), "p99", np.percentile(hit, 99),
              "max", cc.max(), "over48", int((cc > 48).sum()), "intervals mean", iv[iv > 0].mean(), "max", iv.max(),
              "total cands", int(cc.sum()))
