#!/usr/bin/env python3
"""Fixtures for the device epilogue, produced by the REFERENCE's
own imgio.py / metrics.py (run in the build container, where /root/reference
exists; the GPU box only reads the committed JSON):

    python tests/golden/make_epilogue_golden.py

Records imgio.HEATMAP_LUT (imgio.py:12-42), quantize / heatmap_rgb outputs
(imgio.py:36-39, 81-87) for seeded inputs, and metrics.ssim (metrics.py:48-80)
for seeded image pairs."""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import _import_reference  # noqa: E402


def images(seed, h, w):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    noise = rng.integers(-20, 21, (h, w, 3))
    b = np.clip(a.astype(np.int64) + noise, 0, 255).astype(np.uint8)
    return a, b


def main():
    _import_reference()
    from tetray import imgio, metrics
    out = {"heatmap_lut": imgio.HEATMAP_LUT.tolist(), "ssim": [], "quantize": [], "heatmap": []}
    for seed, h, w in ((1, 16, 16), (2, 37, 53), (3, 64, 48)):
        a, b = images(seed, h, w)
        out["ssim"].append({"seed": seed, "h": h, "w": w, "ssim": metrics.ssim(a, b),
                            "ssim_self": metrics.ssim(a, a)})
    for seed, h, w in ((4, 13, 17), (5, 40, 30)):
        rng = np.random.default_rng(seed)
        img = rng.uniform(-0.2, 1.2, (h, w, 4))
        img[0, :4, 0] = [0.5 / 255.0, 1.5 / 255.0, 254.5 / 255.0, 1.0]
        q = imgio.quantize(img[..., :3])
        out["quantize"].append({"seed": seed, "h": h, "w": w,
                                "sha256": hashlib.sha256(q.tobytes()).hexdigest()})
        counts = rng.integers(0, 500, (h, w))
        hm = imgio.heatmap_rgb(counts)
        out["heatmap"].append({"seed": seed, "h": h, "w": w,
                               "sha256": hashlib.sha256(hm.tobytes()).hexdigest(),
                               "zeros_sha256": hashlib.sha256(
                                   imgio.heatmap_rgb(np.zeros((h, w), np.int64)).tobytes()).hexdigest()})
    (HERE / "reference_epilogue.json").write_text(json.dumps(out, indent=1))
    print("wrote", HERE / "reference_epilogue.json")


if __name__ == "__main__":
    main()
