"""The oracle's own scene build (oracle/build.c + oracle/scene.py) against the
REFERENCE: scene-array hashes recorded by running the reference's
Scene.build (tests/golden/make_golden.py, make_golden_big.py), the BVH arrays
of the reference's bvh.py:41-98 itself (when the stock package is importable
here), and whole frames rendered by the oracle on its own scene against the
reference's frame hashes.  This is what lets the oracle check BASELINE
config 3 (1e7-1e8 tets) without the product library."""

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

import cases as C

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def OS(built_oracle):
    import oracle.scene as OS
    return OS


@pytest.fixture(scope="module")
def big():
    return json.loads((GOLDEN / "reference_big.json").read_text())


def oracle_scene(OS, n):
    return OS.GridScene(n, OS.TF.from_json(C.radial16_tf_doc(n)), max_leaf=48 if n == 16 else None)


def oracle_hashes(sc):
    ps = sc.parts
    active, sigma, tf = sc.meta_state()
    return {"n_tets": sc.mesh.n_tets, "n_parts": len(ps), "part_offsets": sha(ps.offsets),
            "part_ids": sha(ps.ids), "part_lo": sha(ps.lo), "part_hi": sha(ps.hi),
            "part_vrange": sha(ps.vrange), "active": sha(active), "sigma": sha(sigma),
            "tet_orig": sha(sc.sampler.tet_orig), "tet_inv": sha(sc.sampler.tet_inv),
            "field": sha(sc.mesh.field), "tf_table": sha(tf.table),
            "epsilon": sc.traversal_config.epsilon, "n_active": int(active.sum()),
            "n_sigma_lt1": int((sigma < 1).sum())}


@pytest.mark.parametrize("n", [16, 59, 128])
def test_oracle_scene_build_matches_reference(OS, golden, big, n):
    want = golden["scenes"].get(f"radial{n}") or big["scenes"][f"radial{n}"]
    got = oracle_hashes(oracle_scene(OS, n))
    for k, v in want.items():
        assert got[k] == v, f"radial{n}: {k}"


def test_fast_bvh_equals_sequential_restatement(OS):
    from oracle.oracle import FlatBVH
    rng = np.random.default_rng(5)
    for n, leaf in ((1, 8), (9, 8), (1000, 1), (5000, 8), (20000, 4)):
        lo = rng.integers(0, 50, (n, 3)).astype(np.float64) * 0.5   # many ties
        hi = lo + rng.integers(0, 4, (n, 3)) * 0.25
        a, b = FlatBVH(lo, hi, leaf, fast=True), FlatBVH(lo, hi, leaf, fast=False)
        for k in ("node_lo", "node_hi", "left", "right", "start", "count", "prim"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (n, leaf, k)


def _stock_tetray():
    ref = ROOT / "baseline" / "_ref"
    if (ref / "tetray").exists():
        sys.path.insert(0, str(ref))
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tetray_test_numba")
        import tetray
        return tetray
    pytest.skip("the stock reference package (baseline/_ref) is not installed")


def test_fast_bvh_equals_reference_bvh_py(OS):
    """orc_build_bvh_fast reproduces the reference's own builder (node ids,
    boxes, prim order) over padded tet boxes and over partition boxes."""
    tetray = _stock_tetray()
    from tetray import bvh as RB

    from oracle.oracle import FlatBVH
    for n in (4, 16):
        sc = oracle_scene(OS, n)
        pad = 1e-7 * sc.mesh.bounds.diagonal()
        lo, hi = sc.mesh.tet_aabbs(pad)
        for leaf in (8, 3):
            a, r = FlatBVH(lo, hi, leaf), RB.build_bvh(lo, hi, leaf)
            for k in ("node_lo", "node_hi", "left", "right", "start", "count", "prim"):
                assert np.array_equal(getattr(a, k), getattr(r, k)), (n, leaf, k)
        a, r = FlatBVH(sc.parts.lo, sc.parts.hi, 4), RB.build_bvh(sc.parts.lo, sc.parts.hi, 4)
        assert np.array_equal(a.prim, r.prim) and np.array_equal(a.node_lo, r.node_lo)


def test_stock_scene_assembly_matches_reference_build(OS, golden):
    """oracle/stock_scene.py (the reference arm's scene) equals the stock
    Scene.build: scene hashes, and the tet BVH arrays of the stock sampler."""
    tetray = _stock_tetray()
    from oracle.stock_scene import build_stock_scene, stock_bvh_equal
    sys.path.insert(0, str(GOLDEN))
    import make_golden as G
    sc = build_stock_scene(tetray, 16, C.radial16_tf_doc(16))
    ref = tetray.Scene.build(tetray.generate_synthetic(16, "radial", tetray.Centering.VERTEX),
                             tetray.TransferFunction.from_json(C.radial16_tf_doc(16)))
    assert stock_bvh_equal(sc.sampler.bvh, ref.sampler.bvh)
    assert stock_bvh_equal(sc.bvh.tree, ref.bvh.tree)
    h, want = G.scene_hashes(sc), G.scene_hashes(ref)
    assert h == want
    # radial59 with the default KD config: the recorded reference hashes
    h59 = G.scene_hashes(build_stock_scene(tetray, 59, C.radial16_tf_doc(59)))
    for k, v in golden["scenes"]["radial59"].items():
        assert h59[k] == v, k


@pytest.mark.parametrize("n,mode", [(59, "skip-adaptive"), (59, "reference"),
                                    (128, "skip-adaptive")])
def test_oracle_frames_on_own_build_match_reference(OS, golden, big, n, mode):
    from oracle.oracle import OracleScene
    sc = oracle_scene(OS, n)
    cam, par = C.camera(OS, f"radial{n}"), C.params(OS, f"radial{n}")
    rgba, samples, visited, ppart = OracleScene(sc).render(cam, mode, par)
    want = (golden["frames"].get(f"radial{n}/{mode}") or big["frames"][f"radial{n}/{mode}"])
    assert sha(samples) == want["samples"] and sha(visited) == want["visited"]
    assert sha(rgba) == want["rgba"]
    assert (ppart is None) == (want["ppart"] is None)
    if ppart is not None:
        assert sha(ppart) == want["ppart"]
