"""Device epilogue of a frame: the viewer / CLI / sweep
post-processing of tetray's imgio.py and metrics.py, run on the frame while
it is still in HBM (csrc/epilogue.cu).

  render_rgb8(scene, camera, mode, params, heatmap=True)
      the frame as imgio.framebuffer_rgb(fb) (imgio.py:76-78) and, optionally,
      imgio.heatmap_rgb(fb.samples) (imgio.py:81-87) -- bit-identical -- with
      only 3 + 3 bytes per pixel crossing PCIe instead of 32 + 8;
  ssim_rgb8(a, b)
      metrics.ssim (metrics.py:48-80) of two u8 RGB images on the GPU
      (floating-point sums in another order than scipy's: relative 1e-12).

The heatmap LUT is the reference's: 11 viridis anchor colours linearly
expanded to 256 entries (np.interp) and quantised (imgio.py:12-42).
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib

# imgio.py:12-24: viridis-like anchors of the heatmap colormap
_HEATMAP_ANCHORS = np.array([
    [0.267004, 0.004874, 0.329415], [0.282623, 0.140926, 0.457517],
    [0.253935, 0.265254, 0.529983], [0.206756, 0.371758, 0.553117],
    [0.163625, 0.471133, 0.558148], [0.127568, 0.566949, 0.550556],
    [0.134692, 0.658636, 0.517649], [0.266941, 0.748751, 0.440573],
    [0.477504, 0.821444, 0.318195], [0.741388, 0.873449, 0.149561],
    [0.993248, 0.906157, 0.143936],
])
REC709 = np.array([0.2126, 0.7152, 0.0722])   # metrics.py:21


def quantize(img: np.ndarray) -> np.ndarray:
    """imgio.py:36-39 on the host (used for the LUT and by the tests)."""
    c = np.clip(np.asarray(img, dtype=np.float64), 0.0, 1.0)
    return np.floor(c * 255.0 + 0.5).astype(np.uint8)


def _expand_colormap(anchors: np.ndarray, size: int = 256) -> np.ndarray:
    x = np.linspace(0.0, 1.0, len(anchors))
    u = np.linspace(0.0, 1.0, size)
    return np.stack([np.interp(u, x, anchors[:, c]) for c in range(3)], axis=1)


HEATMAP_LUT = quantize(_expand_colormap(_HEATMAP_ANCHORS))


def gaussian_window(size: int, sigma: float) -> np.ndarray:
    """metrics.py:44-50."""
    half = (size - 1) / 2.0
    x = np.arange(size) - half
    g1 = np.exp(-(x ** 2) / (2.0 * sigma ** 2))
    w = np.outer(g1, g1)
    return w / w.sum()


def _torch():
    import torch
    return torch


def render_rgb8(scene, camera, mode: str, params, *, heatmap: bool = True, jitter: bool = False,
                track_per_partition: bool = True, device=None, flags: int = 0):
    """Render on the GPU and return (rgb u8 (H,W,3), heatmap u8 (H,W,3) or
    None, RenderStats) -- framebuffer_rgb / heatmap_rgb computed on device."""
    from .device import device_scene_for
    from .render import _MODE_IDS, MODES, RenderStats
    if mode not in _MODE_IDS:
        raise ValueError(f"unknown mode {mode!r}; choose from {MODES}")
    torch = _torch()
    dev = device_scene_for(scene, device)
    w, h = int(camera.width), int(camera.height)
    track = track_per_partition and mode != "reference"
    with dev.lock, torch.cuda.device(dev.device):
        t0 = time.perf_counter()
        stream = torch.cuda.current_stream(dev.device)
        ep = dev.epoch(scene.meta_state(), params)
        frame = dev.frame_desc(scene, camera, _MODE_IDS[mode], params, jitter, track, flags)
        fb = dev.frame_buffers(w, h)
        dev.launch(frame, ep, fb, stream)
        n = w * h
        rgb_d = torch.empty((n, 3), dtype=torch.uint8, device=dev.device)
        _lib.check(_lib.lib().tr_quantize_rgb(C.c_void_p(fb.rgba.data_ptr()), n,
                                              C.c_void_p(rgb_d.data_ptr()),
                                              C.c_void_p(stream.cuda_stream)), "tr_quantize_rgb")
        heat_d = None
        if heatmap:
            lut = getattr(dev, "_heat_lut", None)
            if lut is None:
                lut = dev._heat_lut = torch.from_numpy(HEATMAP_LUT.reshape(-1)).to(dev.device)
            heat_d = torch.empty((n, 3), dtype=torch.uint8, device=dev.device)
            peak = torch.empty(1, dtype=torch.int64, device=dev.device)
            _lib.check(_lib.lib().tr_heatmap_rgb(C.c_void_p(fb.samples.data_ptr()), n,
                                                 C.c_void_p(lut.data_ptr()),
                                                 C.c_void_p(heat_d.data_ptr()),
                                                 C.c_void_p(peak.data_ptr()),
                                                 C.c_void_p(stream.cuda_stream)), "tr_heatmap_rgb")
        rgb = rgb_d.view(h, w, 3).cpu().numpy()
        heat = heat_d.view(h, w, 3).cpu().numpy() if heatmap else None
        cnt = fb.counters.cpu().numpy()
        wall_ms = (time.perf_counter() - t0) * 1000.0
    stats = RenderStats(total_samples=int(cnt[0]), wall_ms=wall_ms,
                        partitions_visited_mean=float(np.float64(cnt[1]) / np.float64(n)),
                        per_partition_samples=cnt[3:].copy() if track else None,
                        device_ms=float(fb.start.elapsed_time(fb.end)), gpu_launches=1)
    return rgb, heat, stats


def ssim_rgb8(a: np.ndarray, b: np.ndarray, window: int = 11, sigma: float = 1.5,
              k1: float = 0.01, k2: float = 0.03, dynamic_range: float = 255.0,
              device=None) -> float:
    """metrics.ssim of two (H,W,3) u8 images, on the GPU."""
    from .device import resolve_device
    torch = _torch()
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    if a.shape != b.shape:
        raise ValueError(f"image dimensions differ: {a.shape} vs {b.shape}")
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError("ssim_rgb8 expects (H, W, 3) uint8 images")
    h, w = a.shape[:2]
    if h < window or w < window:
        raise ValueError("images smaller than the SSIM window")
    device = resolve_device(device)
    with torch.cuda.device(device):
        ad = torch.from_numpy(a).to(device)
        bd = torch.from_numpy(b).to(device)
        wd = torch.from_numpy(gaussian_window(window, sigma)).to(device)
        rd = torch.from_numpy(REC709.copy()).to(device)
        sd = torch.empty(1, dtype=torch.float64, device=device)
        stream = torch.cuda.current_stream(device)
        c1 = (k1 * dynamic_range) ** 2
        c2 = (k2 * dynamic_range) ** 2
        _lib.check(_lib.lib().tr_ssim_rgb(C.c_void_p(ad.data_ptr()), C.c_void_p(bd.data_ptr()), h, w,
                                          window, C.c_void_p(wd.data_ptr()), C.c_void_p(rd.data_ptr()),
                                          c1, c2, C.c_void_p(sd.data_ptr()),
                                          C.c_void_p(stream.cuda_stream)), "tr_ssim_rgb")
        total = float(sd.cpu().numpy()[0])
    half = window // 2
    return total / float((h - 2 * half) * (w - 2 * half))


def quantize_rgb8(rgba: np.ndarray, device=None) -> np.ndarray:
    """tr_quantize_rgb on a host (H,W,4) float64 image (tests / tools)."""
    from .device import resolve_device
    torch = _torch()
    device = resolve_device(device)
    x = np.ascontiguousarray(rgba, dtype=np.float64)
    h, w = x.shape[:2]
    with torch.cuda.device(device):
        xd = torch.from_numpy(x.reshape(-1, 4)).to(device)
        od = torch.empty((h * w, 3), dtype=torch.uint8, device=device)
        stream = torch.cuda.current_stream(device)
        _lib.check(_lib.lib().tr_quantize_rgb(C.c_void_p(xd.data_ptr()), h * w,
                                              C.c_void_p(od.data_ptr()),
                                              C.c_void_p(stream.cuda_stream)), "tr_quantize_rgb")
        return od.view(h, w, 3).cpu().numpy()


def heatmap_rgb8(counts: np.ndarray, device=None) -> np.ndarray:
    """tr_heatmap_rgb on host (H,W) int64 counts (tests / tools)."""
    from .device import resolve_device
    torch = _torch()
    device = resolve_device(device)
    c = np.ascontiguousarray(counts, dtype=np.int64)
    h, w = c.shape
    with torch.cuda.device(device):
        cd = torch.from_numpy(c.reshape(-1)).to(device)
        lut = torch.from_numpy(HEATMAP_LUT.reshape(-1)).to(device)
        od = torch.empty((h * w, 3), dtype=torch.uint8, device=device)
        peak = torch.empty(1, dtype=torch.int64, device=device)
        stream = torch.cuda.current_stream(device)
        _lib.check(_lib.lib().tr_heatmap_rgb(C.c_void_p(cd.data_ptr()), h * w, C.c_void_p(lut.data_ptr()),
                                             C.c_void_p(od.data_ptr()), C.c_void_p(peak.data_ptr()),
                                             C.c_void_p(stream.cuda_stream)), "tr_heatmap_rgb")
        return od.view(h, w, 3).cpu().numpy()
