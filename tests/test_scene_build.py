"""The native scene build (KD partitions, TF metadata, sampler arrays) against
hashes of the reference's own scene objects (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

import cases as C


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B


def scene_hashes(scene):
    offs = np.cumsum([0] + [len(p.element_ids) for p in scene.partitions])
    ids = np.concatenate([p.element_ids for p in scene.partitions])
    lo = np.stack([p.bounds.lo for p in scene.partitions])
    hi = np.stack([p.bounds.hi for p in scene.partitions])
    vr = np.array([p.value_range for p in scene.partitions])
    active, sigma, tf = scene.meta_state()
    return {"n_tets": int(scene.mesh.n_tets), "n_parts": len(scene.partitions),
            "part_offsets": sha(offs.astype(np.int64)), "part_ids": sha(ids.astype(np.int64)),
            "part_lo": sha(lo), "part_hi": sha(hi), "part_vrange": sha(vr),
            "active": sha(active.astype(np.uint8)), "sigma": sha(sigma),
            "tet_orig": sha(scene.sampler.tet_orig), "tet_inv": sha(scene.sampler.tet_inv),
            "field": sha(scene.mesh.field), "tf_table": sha(tf.table),
            "epsilon": float(scene.traversal_config.epsilon),
            "n_active": int(active.sum()), "n_sigma_lt1": int((sigma < 1).sum())}


RECIPES = sorted({r for _, r, _, _ in C.FRAME_CASES})


@pytest.mark.parametrize("recipe", RECIPES + ["radial59"])
def test_scene_arrays_match_reference(B, golden, recipe):
    got = scene_hashes(C.build_scene(B, recipe))
    want = golden["scenes"][recipe]
    for k, v in want.items():
        assert got[k] == v, f"{recipe}: {k}"


def test_tf_meta_matches_numpy_restatement(B):
    """tr_tf_meta reproduces transfer.py:95-141 evaluated with numpy
    (mean over rows, per-row squared distance, pairwise mean)."""
    rng = np.random.default_rng(7)
    for n_tf in (2, 5, 64, 257):
        table = rng.random((n_tf, 4))
        table[rng.random(n_tf) < 0.3, 3] = 0.0
        tf = B.TransferFunction((-1.0, 2.5), table)
        lo_v = rng.uniform(-1.5, 3.0, 300)
        vr = np.stack([lo_v, lo_v + rng.exponential(0.7, 300)], axis=1)
        got = B.transfer.partition_meta_arrays(tf, vr)
        raw = []
        for rmin, rmax in vr:
            n = tf.size
            u0 = (rmin - tf.domain[0]) / (tf.domain[1] - tf.domain[0]) * (n - 1)
            u1 = (rmax - tf.domain[0]) / (tf.domain[1] - tf.domain[0]) * (n - 1)
            j0 = max(int(np.floor(u0)) + 1, 0)
            j1 = min(int(np.ceil(u1)) - 1, n - 1)
            rows = [B.tf_lookup(tf, rmin)] + (list(tf.table[j0:j1 + 1]) if j1 >= j0 else []) \
                + [B.tf_lookup(tf, rmax)]
            rows = np.stack(rows)
            w = rows[:, :3] * rows[:, 3][:, None]
            raw.append(float(((w - w.mean(axis=0)) ** 2).sum(axis=1).mean()))
            assert got["max_opacity"][len(raw) - 1] == rows[:, 3].max()
        assert np.array_equal(got["raw_variance"], np.array(raw))


def test_kd_respects_config_and_covers_every_tet(B):
    m = B.generate_synthetic(6, "sinusoidal", B.Centering.VERTEX)
    parts = B.build_partitions(m, B.KdBuildConfig(max_leaf_elements=30, max_depth=6))
    ids = np.concatenate([p.element_ids for p in parts])
    assert set(ids.tolist()) == set(range(m.n_tets))
    assert len(parts) <= 2 ** 6
    for p in parts:
        assert np.all(np.diff(p.element_ids) > 0)
        assert (p.bounds.lo >= p.leaf_bounds.lo).all() and (p.bounds.hi <= p.leaf_bounds.hi).all()


def test_tet1_roundtrip(B, tmp_path):
    m = B.generate_synthetic(3, "radial", B.Centering.CELL)
    B.save_mesh(m, tmp_path / "m.tet")
    assert B.load_mesh(tmp_path / "m.tet") == m
    with pytest.raises(B.MeshFormatError):
        (tmp_path / "bad.tet").write_bytes(b"TET2" + bytes(40))
        B.load_mesh(tmp_path / "bad.tet")
