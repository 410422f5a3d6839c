"""Device epilogue (csrc/epilogue.cu, epilogue.py) against the
reference's own imgio / metrics outputs (tests/golden/reference_epilogue.json,
written by tests/golden/make_epilogue_golden.py from /root/reference)."""

import hashlib
import json

import numpy as np
import pytest

import cases
from paper_1908_01906_b200 import epilogue as EP

FIX = json.loads((cases.GOLDEN / "reference_epilogue.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _quant_input(seed, h, w):
    rng = np.random.default_rng(seed)
    img = rng.uniform(-0.2, 1.2, (h, w, 4))
    img[0, :4, 0] = [0.5 / 255.0, 1.5 / 255.0, 254.5 / 255.0, 1.0]
    return img, rng.integers(0, 500, (h, w))


def _images(seed, h, w):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    noise = rng.integers(-20, 21, (h, w, 3))
    return a, np.clip(a.astype(np.int64) + noise, 0, 255).astype(np.uint8)


def _heatmap_host(counts):   # imgio.py:81-87 restated (the oracle for the device map)
    counts = np.asarray(counts, dtype=np.float64)
    peak = counts.max()
    t = counts / peak if peak > 0 else np.zeros_like(counts)
    return EP.HEATMAP_LUT[np.floor(t * 255.0 + 0.5).astype(np.int64)]


def test_heatmap_lut_is_the_reference_lut():
    assert np.array_equal(EP.HEATMAP_LUT, np.array(FIX["heatmap_lut"], dtype=np.uint8))


def test_host_restatements_match_reference_fixtures():
    for rec, hrec in zip(FIX["quantize"], FIX["heatmap"]):
        img, counts = _quant_input(rec["seed"], rec["h"], rec["w"])
        assert sha(EP.quantize(img[..., :3])) == rec["sha256"]
        assert sha(_heatmap_host(counts)) == hrec["sha256"]
        assert sha(_heatmap_host(np.zeros_like(counts))) == hrec["zeros_sha256"]


@pytest.mark.gpu
def test_device_quantize_and_heatmap_match_reference():
    for rec, hrec in zip(FIX["quantize"], FIX["heatmap"]):
        img, counts = _quant_input(rec["seed"], rec["h"], rec["w"])
        assert sha(EP.quantize_rgb8(img)) == rec["sha256"]
        assert sha(EP.heatmap_rgb8(counts)) == hrec["sha256"]
        assert sha(EP.heatmap_rgb8(np.zeros_like(counts))) == hrec["zeros_sha256"]


@pytest.mark.gpu
def test_device_ssim_matches_reference():
    for rec in FIX["ssim"]:
        a, b = _images(rec["seed"], rec["h"], rec["w"])
        assert EP.ssim_rgb8(a, b) == pytest.approx(rec["ssim"], rel=1e-12, abs=0)
        assert EP.ssim_rgb8(a, a) == pytest.approx(rec["ssim_self"], rel=1e-12, abs=0)
    with pytest.raises(ValueError):
        EP.ssim_rgb8(np.zeros((8, 8, 3), np.uint8), np.zeros((8, 8, 3), np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("recipe", ["golden_radial4", "radial16", "a6fog"])
def test_render_rgb8_equals_host_postprocessing(B, recipe):
    sc = cases.build_scene(B, recipe)
    cam, par = cases.camera(B, recipe), cases.params(B, recipe)
    for mode in ("reference", "skip-adaptive"):
        fb, st = B.render(sc, cam, mode, par)
        rgb, heat, st8 = EP.render_rgb8(sc, cam, mode, par, heatmap=True)
        assert np.array_equal(rgb, EP.quantize(fb.rgba[..., :3]))
        assert np.array_equal(heat, _heatmap_host(fb.samples))
        assert st8.total_samples == st.total_samples
        assert st8.partitions_visited_mean == st.partitions_visited_mean

