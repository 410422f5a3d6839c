"""Pin the C oracle (oracle/oracle.c) against vectors produced by running the
reference itself (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
import math

import numpy as np
import pytest

import cases as C

GOLD = C.GOLDEN


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    return oracle


@pytest.fixture(scope="module")
def misc():
    return json.loads((GOLD / "reference_misc.json").read_text())


_SC = {}


def oscene(B, recipe):
    from oracle.oracle import OracleScene
    if recipe not in _SC:
        _SC[recipe] = OracleScene(C.build_scene(B, recipe))
    return _SC[recipe]


@pytest.mark.parametrize("cid,recipe,modes,jitter", C.FRAME_CASES, ids=[c[0] for c in C.FRAME_CASES])
def test_oracle_frames_bit_exact(B, golden, cid, recipe, modes, jitter):
    o = oscene(B, recipe)
    cam, par = C.camera(B, recipe), C.params(B, recipe)
    for mode in modes:
        rgba, samples, visited, ppart = o.render(cam, mode, par, jitter=jitter)
        g = golden["frames"][f"{cid}/{mode}"]
        assert sha(rgba) == g["rgba"], mode
        assert sha(samples) == g["samples"], mode
        assert sha(visited) == g["visited"], mode
        assert int(samples.sum()) == g["total_samples"]
        assert float(visited.mean()) == g["partitions_visited_mean"]
        if g["ppart"] is None:
            assert ppart is None
        else:
            assert sha(ppart) == g["ppart"]


def test_oracle_full_arrays_small_cases(B):
    fx = np.load(GOLD / "reference_small.npz")
    o = oscene(B, "golden_radial4")
    cam, par = C.camera(B, "golden_radial4"), C.params(B, "golden_radial4")
    rgba, samples, visited, ppart = o.render(cam, "skip-adaptive", par)
    assert np.array_equal(rgba, fx["golden_radial4/skip-adaptive/rgba"])
    assert np.array_equal(samples, fx["golden_radial4/skip-adaptive/samples"])
    assert np.array_equal(ppart, fx["golden_radial4/skip-adaptive/ppart"])


@pytest.mark.slow
@pytest.mark.parametrize("mode", ["skip-adaptive", "skip", "reference"])
def test_oracle_radial59(B, golden, mode):
    o = oscene(B, "radial59")
    cam, par = C.camera(B, "radial59"), C.params(B, "radial59")
    rgba, samples, visited, ppart = o.render(cam, mode, par)
    g = golden["frames"][f"radial59/{mode}"]
    assert sha(rgba) == g["rgba"]
    assert sha(samples) == g["samples"]
    assert int(samples.sum()) == g["total_samples"]


def test_oracle_point_location(B):
    fx = np.load(GOLD / "reference_points.npz")
    for recipe in ("golden_radial4", "radial16", "voidcell", "sinus"):
        o = oscene(B, recipe)
        found, vals, tet = o.field_at_many(fx[f"{recipe}/pts"])
        assert np.array_equal(tet, fx[f"{recipe}/tet"]), recipe
        assert np.array_equal(found, fx[f"{recipe}/found"]), recipe
        assert np.array_equal(vals, fx[f"{recipe}/vals"]), recipe


def test_oracle_traversal(B, misc):
    import ctypes as Ct
    from oracle.oracle import lib, _p
    o = oscene(B, "radial16")
    active = np.ascontiguousarray(o.scene.meta_state()[0], dtype=np.uint8)
    eps = o.scene.traversal_config.epsilon
    for ray in misc["trace_radial16"]:
        org = np.array(ray["o"])
        d = np.array(ray["d"])
        ids = np.zeros(600, np.int64)
        en = np.zeros(600)
        ex = np.zeros(600)
        k = lib().orc_trace_intervals(_p(org, Ct.c_double), _p(d, Ct.c_double), 0.0, math.inf,
                                      eps, *o.part_args(active), 600, _p(ids, Ct.c_int64),
                                      _p(en, Ct.c_double), _p(ex, Ct.c_double))
        assert ids[:k].tolist() == ray["ids"]
        assert en[:k].tolist() == ray["enter"]
        assert ex[:k].tolist() == ray["exit"]


def test_oracle_formulas_and_hash(orc, misc):
    for s1, s2, p, sig, want in misc["step_size"]:
        assert orc.step_size(s1, s2, p, sig) == want
    for a, s, s1, want in misc["opacity_correction"]:
        assert orc.opacity_correction(a, s, s1) == want
    for x, y, want in misc["hash01"]:
        assert orc.hash01(x, y) == want


def test_cli_golden_image_from_oracle(B):
    """The reference CLI's golden PPM (pkg/scripts/make_golden.py) equals the
    oracle frame quantized with imgio's round-half-up rule (imgio.py:36-39)."""
    o = oscene(B, "golden_radial4")
    cam, par = C.camera(B, "golden_radial4"), C.params(B, "golden_radial4")
    rgba, samples, _, _ = o.render(cam, "skip-adaptive", par)
    rgb8 = np.floor(np.clip(rgba[..., :3], 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    raw = (GOLD / "radial4_skip_adaptive.ppm").read_bytes()
    assert raw == b"P6\n64 64\n255\n" + rgb8.tobytes()
