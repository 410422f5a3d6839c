"""Where the end-to-end render() time goes (GPU box; debug aid)."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import torch
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200.device import device_scene_for

sc = C.build_scene(B, "radial59")
cam, par = C.camera(B, "radial59"), C.params(B, "radial59")
dev = device_scene_for(sc)
for _ in range(3):
    B.render(sc, cam, "skip-adaptive", par)
N = 20
tt = {}
def tick(k, t0):
    tt[k] = tt.get(k, 0.0) + time.perf_counter() - t0
for _ in range(N):
    t0 = time.perf_counter(); dev._epochs.clear(); ep = dev.epoch(sc.meta_state(), par); torch.cuda.synchronize(); tick("epoch(h2d)", t0)
    t0 = time.perf_counter(); fd = dev.frame_desc(sc, cam, 2, par, False, True); tick("frame_desc", t0)
    fb = dev.frame_buffers(512, 512)
    s = torch.cuda.current_stream()
    t0 = time.perf_counter(); dev.launch(fd, ep, fb, s); tick("launch(async)", t0)
    t0 = time.perf_counter(); s.synchronize(); tick("gpu wait", t0)
    t0 = time.perf_counter()
    r = torch.empty((512, 512, 4), dtype=torch.float64, pin_memory=True); r.view(-1, 4).copy_(fb.rgba, non_blocking=True)
    sm = torch.empty((512, 512), dtype=torch.int64, pin_memory=True); sm.view(-1).copy_(fb.samples, non_blocking=True)
    s.synchronize(); tick("d2h 10MB", t0)
    t0 = time.perf_counter(); B.render(sc, cam, "skip-adaptive", par); tick("render() total (cached epoch)", t0)
    t0 = time.perf_counter(); dev._epochs.clear(); B.render(sc, cam, "skip-adaptive", par); tick("render() total (new epoch)", t0)
for k, v in tt.items():
    print(f"{k:32s} {v / N * 1e3:8.3f} ms")

# epoch pieces
import ctypes as Cc
import numpy as np
from paper_1908_01906_b200 import _lib, device as DV
active, sigma, tf = sc.meta_state()
sig = np.ascontiguousarray(sigma, dtype=np.float64)
out = np.empty_like(sig); rat = np.empty(2 * len(sig))
def clock(f, n=200):
    f(); t = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t) / n * 1e3
print(f"{'host tr_epoch_steps':32s} {clock(lambda: _lib.lib().tr_epoch_steps(len(sig), _lib.ptr(sig, Cc.c_double), par.s1, par.s2, par.p, out.ctypes.data, rat.ctypes.data)):8.3f} ms")
print(f"{'domain precheck':32s} {clock(lambda: DV._steps_on_device(sig, float(par.p))):8.3f} ms")
print(f"{'Epoch() async':32s} {clock(lambda: DV.Epoch(dev, sc.meta_state(), par)):8.3f} ms")
def ep_sync():
    DV.Epoch(dev, sc.meta_state(), par); torch.cuda.synchronize()
print(f"{'Epoch() + sync':32s} {clock(ep_sync):8.3f} ms")
print(f"{'pinned 8 MB alloc (cached)':32s} {clock(lambda: torch.empty((512, 512, 4), dtype=torch.float64, pin_memory=True)):8.3f} ms")
