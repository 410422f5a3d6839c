"""Host-side phases of DeviceScene.render (a copy of its body with timers; GPU box)."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np
import torch
import cases as C
import paper_1908_01906_b200 as B
from paper_1908_01906_b200 import device as DV
from paper_1908_01906_b200.render import Framebuffer, RenderStats

SCENE = sys.argv[1] if len(sys.argv) > 1 else "radial59"
sc = C.build_scene(B, SCENE)
cam, par = C.camera(B, SCENE), C.params(B, SCENE)
dev = DV.device_scene_for(sc)
T = {}
def render():
    t = [time.perf_counter()]
    def tick(k):
        now = time.perf_counter(); T.setdefault(k, []).append(now - t[0]); t[0] = now
    w, h = cam.width, cam.height
    dev.mark_epochs_stale(); tick("stale")
    with dev.lock, torch.cuda.device(dev.device):
        stream = torch.cuda.current_stream(dev.device)
        meta = sc.meta_state(); tick("stream+meta")
        ep = dev.epoch(meta, par); tick("epoch")
        frame = dev.frame_desc(sc, cam, 2, par, False, True, 0); tick("frame_desc")
        fb = dev.frame_buffers(w, h)
        rgba_h = torch.empty((h, w, 4), dtype=torch.float64, pin_memory=True)
        samp_h = torch.empty((h, w), dtype=torch.int64, pin_memory=True)
        cnt_h = torch.empty(3 + dev.n_parts, dtype=torch.int64, pin_memory=True); tick("pinned allocs")
        out = fb.outputs()
        out.rgba = DV.host_device_pointer(rgba_h)
        out.samples = DV.host_device_pointer(samp_h); tick("outputs")
        DV._lib.check(DV._lib.lib().tr_memset_async(fb.counters.data_ptr(), 0, 8 * fb.counters.numel(),
                                                   stream.cuda_stream), "tr_memset_async"); tick("counters reset")
        fb.start.record(stream); tick("event record")
        DV._lib.check(DV._lib.lib().tr_render_frame(DV.C.byref(dev.desc), DV.C.byref(ep.desc),
                                                  DV.C.byref(frame), DV.C.byref(out),
                                                  DV.C.c_void_p(stream.cuda_stream)), "tr_render_frame"); tick("tr_render_frame")
        fb.end.record(stream); tick("event record 2")
        DV._lib.check(DV._lib.lib().tr_copy_async(cnt_h.data_ptr(), fb.counters.data_ptr(),
                                                 8 * fb.counters.numel(), stream.cuda_stream), "tr_copy_async"); tick("counters copy")
        stream.synchronize(); tick("sync")
        dev_ms = fb.start.elapsed_time(fb.end); tick("elapsed")
    cnt = cnt_h.numpy()
    fbuf = Framebuffer(width=w, height=h, rgba=rgba_h.numpy(), samples=samp_h.numpy(),
                       background=np.asarray(sc.background, dtype=np.float64).copy())
    stats = RenderStats(total_samples=int(cnt[0]), wall_ms=0.0,
                        partitions_visited_mean=float(np.float64(cnt[1]) / np.float64(w * h)),
                        per_partition_samples=cnt[3:].copy(), samples=fbuf.samples,
                        device_ms=float(dev_ms), gpu_launches=1); tick("results")
    return fbuf, stats
fb = None
for _ in range(10):
    fb = render()
T.clear()
for _ in range(300):
    fb = render()
for k, v in T.items():
    print(f"{k:16s} median {np.median(v) * 1e6:8.1f} us  mean {np.mean(v) * 1e6:8.1f} us")
# Epoch pieces
import ctypes
ep_t = {}
act, sig, tf = sc.meta_state()
def clock(name, f, n=300):
    f(); t0 = time.perf_counter()
    for _ in range(n): f()
    print(f"{name:28s} {(time.perf_counter() - t0) / n * 1e6:8.1f} us")
clock("activity (cached)", lambda: dev.activity(np.ascontiguousarray(act, dtype=np.uint8)))
clock("pinned empty 100KB", lambda: torch.empty(100352, dtype=torch.uint8, pin_memory=True))
clock("device empty 100KB", lambda: torch.empty(100352, dtype=torch.uint8, device="cuda"))
x = torch.empty(100352, dtype=torch.uint8, pin_memory=True); y = torch.empty(100352, dtype=torch.uint8, device="cuda")
clock("h2d copy_ async", lambda: y.copy_(x, non_blocking=True))
clock("torch.zeros(1) cuda", lambda: torch.zeros(1, dtype=torch.int32, device="cuda"))
clock("current_stream", lambda: torch.cuda.current_stream(dev.device))
clock("Epoch()", lambda: DV.Epoch(dev, sc.meta_state(), par))

import cProfile, pstats, io
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    DV.Epoch(dev, sc.meta_state(), par)
pr.disable()
buf = io.StringIO()
pstats.Stats(pr, stream=buf).sort_stats("tottime").print_stats(12)
print(buf.getvalue())
