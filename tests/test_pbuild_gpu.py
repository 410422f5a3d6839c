"""Device-built point location (csrc/pbuild.cu) against the
reference: the Morton LBVH, exclusive boxes, leaf grid and cell lists built in
HBM for an ARBITRARY mesh must render every frame bit-identical to the
reference's fixtures / the oracle, exactly as the host-built structures do
(results do not depend on the structure, SURVEY §8c -- but only if the
structure is conservative: these tests are what proves it).

Also checked structurally on small meshes (numpy over the downloaded arrays):
leaf ids are a permutation, ascending inside each leaf; node child boxes and
min ids bound their subtrees; no other leaf's box meets an exclusive box's
interior; cell lists hold every record whose padded box meets the cell, in
ascending tet id.
"""

import gc

import numpy as np
import pytest

import cases as C
from test_parity_gpu import _compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B


_SCENES = {}


def device_built(B, recipe, mode="device"):
    """(scene with point_build = mode, oracle scene)."""
    if (recipe, mode) not in _SCENES:
        from oracle.oracle import OracleScene
        sc = C.build_scene(B, recipe)
        sc.point_build = mode
        _SCENES[(recipe, mode)] = (sc, OracleScene(sc))
    return _SCENES[(recipe, mode)]


def dev_of(sc):
    from paper_1908_01906_b200.device import device_scene_for
    return device_scene_for(sc)


FRAME_CASES = [c for c in C.FRAME_CASES if c[1] not in ("single",)]


@pytest.mark.parametrize("cid,recipe,modes,jitter", FRAME_CASES, ids=[c[0] for c in FRAME_CASES])
def test_device_built_frames_match_reference(B, golden, cid, recipe, modes, jitter):
    """The device build without walk tables (the default, with device walk
    tables, runs every other GPU test)."""
    sc, orc = device_built(B, recipe, "device-nowalk")
    if sc.mesh.n_tets <= 8:
        pytest.skip("one-leaf mesh: host build")
    dev = dev_of(sc)
    assert dev.t_grid_pred is None, "expected the device build (no walk predictors)"
    cam, par = C.camera(B, recipe), C.params(B, recipe)
    for mode in modes:
        ref = orc.render(cam, mode, par, jitter=jitter)
        for flags in (0, 2, 0x80, 0x800008):
            fb, st = B.render(sc, cam, mode, par, jitter=jitter, flags=flags)
            _compare(fb, st, ref, mode, golden["frames"][f"{cid}/{mode}"])


@pytest.mark.parametrize("mode", ["reference", "skip", "skip-adaptive"])
def test_device_built_radial59(B, golden, mode):
    """BASELINE config 2 through the device build: the reference's frame."""
    from test_parity_gpu import _check_radial59
    sc, orc = device_built(B, "radial59", "device-nowalk")
    cam, par = C.camera(B, "radial59"), C.params(B, "radial59")
    g = golden["frames"][f"radial59/{mode}"]
    for flags in (0, 0x80):
        fb, st = B.render(sc, cam, mode, par, flags=flags)
        _check_radial59(fb, st, g, orc, cam, mode, par)


@pytest.mark.parametrize("recipe", ["radial16", "radial59"])
def test_device_walk_frames(B, golden, recipe):
    """point_build = "device-hostwalk": the device build plus the host's walk
    tables and predictors on its leaves -- the reference's frames, and the
    walk really is used (predictors present)."""
    sc, orc = device_built(B, recipe, "device-hostwalk")
    dev = dev_of(sc)
    assert dev.t_grid_pred is not None
    _, leaves, _ = _download(dev)
    assert (leaves["walk"][:, 4] >> 31).any(), "no valid walk table attached"
    cam, par = C.camera(B, recipe), C.params(B, recipe)
    for mode in ("reference", "skip", "skip-adaptive"):
        ref = orc.render(cam, mode, par)
        g = golden["frames"][f"{recipe}/{mode}"]
        for flags in (0, 0x2000000):
            fb, st = B.render(sc, cam, mode, par, flags=flags)
            _compare(fb, st, ref, mode, g if recipe != "radial59" else None)


@pytest.mark.parametrize("recipe", ["jitter8", "jitter16", "jitter32"])
def test_device_built_unstructured(B, recipe):
    """Unstructured meshes: low grid coverage -> the device builds the cell
    candidate lists; every mode bit-identical to the oracle."""
    sc, orc = device_built(B, recipe, "device-nowalk")
    dev = dev_of(sc)
    assert dev.cells is not None, "unstructured mesh should get cell lists"
    cam, par = C.camera(B, recipe), C.params(B, recipe)
    if cam.width > 256:
        cam = B.Camera(position=cam.position, look_at=cam.look_at, up=cam.up,
                       fov_y_deg=cam.fov_y_deg, width=192, height=160)
    for mode in ("reference", "skip", "skip-adaptive"):
        ref = orc.render(cam, mode, par)
        for flags in (0, 2):
            fb, st = B.render(sc, cam, mode, par, flags=flags)
            _compare(fb, st, ref, mode)


def test_device_built_field_at_many(B, monkeypatch):
    """tr_field_at_many over device-built structures: the reference's own
    point-location vectors (lowest-index rule on faces, edges, vertices)."""
    from paper_1908_01906_b200 import device as DV
    monkeypatch.setenv(DV.POINT_BUILD_ENV, "device")
    fx = np.load(C.GOLDEN / "reference_points.npz")
    for recipe in ("golden_radial4", "radial16", "voidcell", "sinus"):
        sc = C.build_scene(B, recipe)
        pts = fx[f"{recipe}/pts"]
        tet, vals = sc.sampler.locate_many(pts)
        dev = next(iter(sc.sampler._device.values()))
        assert hasattr(dev, "build_phases") and dev.t_grid_pred is not None   # device walk tables
        assert np.array_equal(tet, fx[f"{recipe}/tet"]), recipe
        assert np.array_equal(vals, fx[f"{recipe}/vals"]), recipe


def _download(dev):
    from paper_1908_01906_b200 import _lib
    nodes = dev.t_pnodes.cpu().numpy().view(_lib.PNODE_DTYPE)
    leaves = dev.t_pleaves.cpu().numpy().view(_lib.PLEAF_DTYPE)
    ids = dev.t_pids.cpu().numpy().view(np.uint32)
    return nodes, leaves, ids


@pytest.mark.parametrize("recipe", ["radial16", "jitter16"])
def test_device_built_structure_invariants(B, recipe):
    from paper_1908_01906_b200 import device as DV
    sc, _ = device_built(B, recipe, "device-nowalk")
    dev = dev_of(sc)
    nodes, leaves, ids = _download(dev)
    T = sc.mesh.n_tets
    assert np.array_equal(np.sort(ids), np.arange(T, dtype=np.uint32))
    lo, hi = DV._padded_boxes(sc)
    lb = np.zeros((len(leaves), 6))
    for L, lf in enumerate(leaves):
        s, n = int(lf["start"]), int(lf["count"])
        seg = ids[s:s + n]
        assert 1 <= n <= 64 and np.all(np.diff(seg.astype(np.int64)) > 0)
        assert not np.any(lf["walk"])
        lb[L, :3], lb[L, 3:] = lo[seg].min(0), hi[seg].max(0)
    # child boxes (f32, outward) and min ids bound their subtrees
    sub_lo, sub_hi, sub_min = {}, {}, {}

    def visit(c):
        if c < 0:
            L = ~c
            s, n = int(leaves[L]["start"]), int(leaves[L]["count"])
            return lb[L, :3], lb[L, 3:], int(ids[s:s + n].min())
        nd = nodes[c]
        out = []
        for k, (clo, chi) in enumerate((("lo0", "hi0"), ("lo1", "hi1"))):
            a, b, m = visit(int(nd["child"][k]))
            assert np.all(nd[clo].astype(np.float64) <= a) and np.all(nd[chi].astype(np.float64) >= b)
            assert int(nd["minid"][k]) == m
            out.append((a, b, m))
        return (np.minimum(out[0][0], out[1][0]), np.maximum(out[0][1], out[1][1]),
                min(out[0][2], out[1][2]))

    import sys
    sys.setrecursionlimit(10000)
    visit(0)
    # exclusive boxes: no other leaf box meets the open interior
    for L, lf in enumerate(leaves):
        e0, e1 = lf["ex_lo"].astype(np.float64), lf["ex_hi"].astype(np.float64)
        if not np.all(e0 < e1):
            continue
        meet = np.all(lb[:, :3] < e1, axis=1) & np.all(lb[:, 3:] > e0, axis=1)
        meet[L] = False
        assert not meet.any(), f"leaf {L}: exclusive box meets leaf {np.flatnonzero(meet)[:4]}"
    if dev.cells is not None:
        cl = dev.cells
        off = dev.t_coff.cpu().numpy().view(np.uint32)
        recs = dev.t_crecs.cpu().numpy().view(np.uint32)
        d = cl.dims
        rng = np.random.default_rng(3)
        for c in rng.integers(0, int(np.prod(d)), 300):
            o0, o1 = int(off[c]), int(off[c + 1]) & 0x7fffffff
            if o0 & 0x80000000:
                continue
            x, y, z = c // (d[1] * d[2]), (c // d[2]) % d[1], c % d[2]
            cmin = cl.org + np.array([x, y, z]) / cl.scale
            cmax = cl.org + np.array([x + 1, y + 1, z + 1]) / cl.scale
            got = ids[recs[o0:o1]]
            assert np.all(np.diff(got.astype(np.int64)) > 0)
            # every tet whose box is well inside-overlapping the cell is listed
            inner = np.all(lo < cmax - 1e-9, axis=1) & np.all(hi > cmin + 1e-9, axis=1)
            assert set(np.flatnonzero(inner)) <= set(got.tolist())


@pytest.mark.parametrize("recipe", ["radial128", "radial272"])
def test_device_built_config3_matches_reference(B, recipe):
    """BASELINE config 3 through the device build without walk tables (the
    default device build, with them, runs test_parity_big_gpu): the
    reference's own radial128 / radial272 frames, all modes."""
    from test_parity_big_gpu import MODES, check_frame, scene
    sc = scene(B, recipe)
    from paper_1908_01906_b200.device import _CACHE_ATTR
    for k in list(getattr(sc, _CACHE_ATTR, {}) or {}):
        del getattr(sc, _CACHE_ATTR)[k]
    gc.collect()
    import torch
    torch.cuda.empty_cache()
    sc.point_build = "device-nowalk"
    try:
        dev = dev_of(sc)
        assert dev.t_grid_pred is None
        for mode in MODES:
            check_frame(B, sc, recipe, recipe, mode)
    finally:
        sc.point_build = None
        for k in list(getattr(sc, _CACHE_ATTR, {}) or {}):
            del getattr(sc, _CACHE_ATTR)[k]


@pytest.mark.parametrize("recipe", ["radial16", "jitter16", "radial59"])
def test_host_point_build_still_matches(B, golden, recipe):
    """point_build = "host" (host_build.cpp; the default is the device
    build): the same frames."""
    sc, orc = device_built(B, recipe, "host")
    dev = dev_of(sc)
    assert not hasattr(dev, "build_phases"), "expected the host build"
    cam, par = C.camera(B, recipe), C.params(B, recipe)
    if cam.width > 256:
        cam = B.Camera(position=cam.position, look_at=cam.look_at, up=cam.up,
                       fov_y_deg=cam.fov_y_deg, width=192, height=160)
    for mode in ("reference", "skip", "skip-adaptive"):
        ref = orc.render(cam, mode, par)
        fb, st = B.render(sc, cam, mode, par)
        _compare(fb, st, ref, mode)


@pytest.mark.parametrize("recipe", ["radial16", "jitter16", "radial59", "jitter32"])
def test_device_walk_tables_vs_host(B, recipe):
    """tr_dpb_walk against tr_leaf_walk on the same device-built leaves:
    identical face neighbours and walk start, and every device certificate
    is a host (long-double) certificate; on the generator's meshes the two
    sets are equal.  Predictors agree to f32 rounding."""
    import ctypes
    from paper_1908_01906_b200 import _lib
    sc, _ = device_built(B, recipe, "device")
    dev = dev_of(sc)
    _, leaves, ids = _download(dev)
    host = leaves.copy()
    pred = np.zeros((len(host), 12), np.float32)
    verts = np.ascontiguousarray(sc.mesh.vertices, dtype=np.float64)
    tets = np.ascontiguousarray(sc.mesh.tets, dtype=np.int64)
    ids = np.ascontiguousarray(ids)
    _lib.check(_lib.lib().tr_leaf_walk(len(host), _lib.vptr(host), _lib.vptr(ids), _lib.vptr(verts),
                                       _lib.vptr(tets), _lib.vptr(pred)), "tr_leaf_walk")
    dw, hw = leaves["walk"].astype(np.uint32), host["walk"].astype(np.uint32)
    assert np.array_equal(dw[:, 4], hw[:, 4]), "walk start / validity differ"
    ent = lambda w: np.stack([(w[:, i >> 1] >> (16 * (i & 1))) & 0xffff for i in range(8)], 1)
    de, he = ent(dw), ent(hw)
    assert np.array_equal(de & 0xfff, he & 0xfff), "face neighbours differ"
    dc, hc = (de >> 12) & 1, (he >> 12) & 1
    assert not np.any(dc & ~hc), "a device certificate the host does not give"
    n_dev, n_host = int(dc.sum()), int(hc.sum())
    print(recipe, "certificates device / host:", n_dev, n_host)
    if recipe.startswith("radial"):
        assert n_dev == n_host
    assert n_dev >= 0.9 * n_host
