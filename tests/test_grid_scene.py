"""Device-generated cube-grid scenes (grid_scene.py, csrc/synth.cu).

CPU: the closed-form KD partitions equal the general KD build (which matches
the reference bit for bit, test_scene_build.py) and the grid scene's metadata
epoch equals the host-built scene's.  GPU: the records generated in HBM equal
the host-packed ones, and frames / point queries of gridN equal radialN's
bit for bit."""

import ctypes as C

import numpy as np
import pytest

import cases
from paper_1908_01906_b200 import partitions as PT
from paper_1908_01906_b200.grid_scene import build_grid_kd

KD_FIELDS = ("offsets", "ids", "leaf_lo", "leaf_hi", "lo", "hi", "vrange")


@pytest.mark.parametrize("field", ["radial", "ramp"])
def test_grid_kd_equals_general_kd(B, field):
    for n in (1, 2, 3, 5, 8, 11, 16):
        mesh = B.generate_synthetic(n, field, B.Centering.VERTEX)
        for leaf in (1, 5, 13, 64, max(64, mesh.n_tets // 4096)):
            for depth in (1, 4, 24):
                cfg = PT.KdBuildConfig(max_leaf_elements=leaf, max_depth=depth)
                a = PT.build_kd_arrays(mesh, cfg)
                b = build_grid_kd(n, field, cfg, with_ids=True)
                for k in KD_FIELDS:
                    assert np.array_equal(getattr(a, k), getattr(b, k)), (n, leaf, depth, k)


def test_grid_kd_default_config_large(B):
    # odd and even resolutions at the benchmark's default KD config
    for n in (24, 33):
        mesh = B.generate_synthetic(n, "radial", B.Centering.VERTEX)
        cfg = PT.default_config(mesh.n_tets)
        a = PT.build_kd_arrays(mesh, cfg)
        b = build_grid_kd(n, "radial", cfg, with_ids=True)
        for k in KD_FIELDS:
            assert np.array_equal(getattr(a, k), getattr(b, k)), (n, k)


def test_grid_scene_epoch_equals_host_scene(B):
    for n in (16, 24):
        g = cases.build_scene(B, f"grid{n}")
        r = B.Scene.build(B.generate_synthetic(n, "radial", B.Centering.VERTEX), g.tf)
        assert g.n_partitions == r.n_partitions
        assert np.array_equal(g.bvh.box_lo, r.bvh.box_lo)
        assert np.array_equal(g.bvh.box_hi, r.bvh.box_hi)
        ga, gs, _ = g.meta_state()
        ra, rs, _ = r.meta_state()
        assert np.array_equal(ga, ra) and np.array_equal(gs, rs)
        assert g.traversal_config.epsilon == r.traversal_config.epsilon
        assert [p.n_elements for p in g.partitions] == [len(p.element_ids) for p in r.partitions]


def test_grid_inverse_matrices_equal_sampler(B):
    n = 5
    g = cases.build_scene(B, f"grid{n}")
    mesh = B.generate_synthetic(n, "radial", B.Centering.VERTEX)
    s = B.MeshSampler(mesh)
    cube = np.arange(mesh.n_tets) // 5
    i, j, k = cube // (n * n), (cube // n) % n, cube % n
    key = ((i + j + k) % 2) * 5 + np.arange(mesh.n_tets) % 5
    assert np.array_equal(g.sampler.inv10[key], s.tet_inv)
    assert g.sampler.pad == s.pad


def test_grid_scene_limits(B):
    with pytest.raises(ValueError):
        B.GridMesh(0)
    with pytest.raises(ValueError):
        B.GridMesh(4, "sinusoidal")
    sz = np.zeros(3, np.int64)
    from paper_1908_01906_b200 import _lib
    assert _lib.lib().tr_grid_scene_sizes(585, _lib.ptr(sz[0:1], C.c_int64), _lib.ptr(sz[1:2], C.c_int64),
                                          _lib.ptr(sz[2:3], C.c_int64)) == 0
    assert sz.tolist() == [5 * 585 ** 3, 585 ** 3, 585 ** 3 - 1]
    assert _lib.lib().tr_grid_scene_sizes(2000, _lib.ptr(sz[0:1], C.c_int64), _lib.ptr(sz[1:2], C.c_int64),
                                          _lib.ptr(sz[2:3], C.c_int64)) != 0


@pytest.mark.gpu
def test_grid_records_equal_host_packing(B):
    import torch
    from paper_1908_01906_b200.device import device_scene_for, pack_tet_records
    for n in (1, 3, 8, 11):
        mesh = B.generate_synthetic(n, "radial", B.Centering.VERTEX)
        want = np.frombuffer(pack_tet_records(mesh, B.MeshSampler(mesh)).tobytes(),
                             np.uint8).reshape(-1, 128)
        for id_order in (True, False):
            g = cases.build_scene(B, f"grid{n}")
            g.grid_id_order = id_order
            dev = device_scene_for(g)
            got = dev.t_tets.cpu().numpy().reshape(-1, 128)
            if id_order:
                assert dev.t_pids is None
                assert np.array_equal(got, want), n
            else:   # brick order: record k is tet ids[k], every tet exactly once
                ids = dev.t_pids.cpu().numpy()
                assert np.array_equal(np.sort(ids), np.arange(mesh.n_tets))
                assert np.array_equal(got, want[ids]), n
                from paper_1908_01906_b200 import _lib
                lv = dev.t_pleaves.cpu().numpy().view(_lib.PLEAF_DTYPE)
                # leaf c (cube c) starts at its cube's 5 records, ascending ids
                assert np.array_equal(ids[lv["start"]], 5 * np.arange(n ** 3))
        torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [4, 16, 59])
def test_grid_frames_equal_host_scene(B, n):
    g = cases.build_scene(B, f"grid{n}")
    r = B.Scene.build(B.generate_synthetic(n, "radial", B.Centering.VERTEX), g.tf)
    cam, par = cases.camera(B, f"radial{max(n, 5)}"), cases.params(B, "radial16")
    if n == 4:
        cam = cases.camera(B, "golden_radial4")
    g2 = cases.build_scene(B, f"grid{n}")
    g2.grid_id_order = True
    for mode in ("reference", "skip", "skip-adaptive"):
        # default (analytic cube leaves), no grid, 4 CTAs/SM, headers instead
        # of the analytic layout (0x8000000), id-order records (g2)
        for gs, flags in ((g, 0), (g, 2), (g, 0x1000), (g, 0x8000000), (g, 0x4000000), (g2, 0)):
            fg, sg = B.render(gs, cam, mode, par, flags=flags)
            fr, sr = B.render(r, cam, mode, par)
            assert np.array_equal(fg.rgba, fr.rgba), (n, mode, flags)
            assert np.array_equal(fg.samples, fr.samples)
            assert sg.total_samples == sr.total_samples
            assert sg.partitions_visited_mean == sr.partitions_visited_mean
            if sr.per_partition_samples is not None:
                assert np.array_equal(sg.per_partition_samples, sr.per_partition_samples)


@pytest.mark.gpu
def test_grid_point_queries_equal_host_scene(B):
    from paper_1908_01906_b200.device import device_scene_for
    import torch
    n = 7
    g = cases.build_scene(B, f"grid{n}")
    mesh = B.generate_synthetic(n, "radial", B.Centering.VERTEX)
    rng = np.random.default_rng(7)
    pts = np.concatenate([rng.uniform(-0.5, n + 0.5, (20000, 3)),
                          rng.integers(0, n + 1, (3000, 3)).astype(np.float64),   # vertices
                          np.round(rng.uniform(0, n, (3000, 3)) * 2) / 2])        # faces/edges
    want_tet, want_val = B.MeshSampler(mesh).locate_many(pts)
    dev = device_scene_for(g)
    p_d = torch.from_numpy(pts).cuda()
    found = torch.empty(len(pts), dtype=torch.uint8, device="cuda")
    vals = torch.empty(len(pts), dtype=torch.float64, device="cuda")
    tet = torch.empty(len(pts), dtype=torch.int64, device="cuda")
    from paper_1908_01906_b200 import _lib
    _lib.check(_lib.lib().tr_field_at_many(C.byref(dev.desc), len(pts), C.c_void_p(p_d.data_ptr()),
                                           C.c_void_p(found.data_ptr()), C.c_void_p(vals.data_ptr()),
                                           C.c_void_p(tet.data_ptr()), None), "tr_field_at_many")
    assert np.array_equal(tet.cpu().numpy(), want_tet)
    assert np.array_equal(vals.cpu().numpy(), want_val)
