"""KD-brick sharding host logic on CPU (bricks.py):
convex bricks tiling the KD root box, halo sufficiency of the per-brick tet
subsets, and the exactness of the per-round SUM exchange (gloo, world 3)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cases as C
from paper_1908_01906_b200 import bricks as BR


@pytest.mark.parametrize("recipe", ["golden_radial4", "radial16", "a6fog", "jitter8"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_bricks_tile_the_kd_root(B, recipe, n):
    sc = C.build_scene(B, recipe)
    br = BR.scene_bricks(sc, n)
    parts = sc.partitions
    llo = np.stack([p.leaf_bounds.lo for p in parts])
    lhi = np.stack([p.leaf_bounds.hi for p in parts])
    assert br.n == n and br.start[0] == 0 and br.start[-1] == len(parts)
    vol = 0.0
    for b in range(n):
        a, e = br.start[b], br.start[b + 1]
        assert e > a
        assert np.all(br.owner[a:e] == b)
        assert np.array_equal(br.lo[b], llo[a:e].min(axis=0))
        assert np.array_equal(br.hi[b], lhi[a:e].max(axis=0))
        bv = np.prod(br.hi[b] - br.lo[b])
        assert bv == pytest.approx(np.prod(lhi[a:e] - llo[a:e], axis=1).sum(), rel=1e-9)   # convex
        vol += bv
        for c in range(b):   # disjoint interiors
            assert np.any((br.hi[b] <= br.lo[c]) | (br.hi[c] <= br.lo[b]))
    root = np.prod(lhi.max(axis=0) - llo.min(axis=0))
    assert vol == pytest.approx(root, rel=1e-9)


def _containing(sc, pts):
    """All tets containing each point (K:121-128 barycentric test, -1e-9 slack)."""
    inv = np.asarray(sc.sampler.tet_inv).reshape(-1, 3, 3)
    orig = np.asarray(sc.sampler.tet_orig)
    d = pts[:, None, :] - orig[None, :, :]
    l123 = np.einsum("tij,ptj->pti", inv, d)
    l0 = 1.0 - l123[..., 0] - l123[..., 1] - l123[..., 2]
    return (l123.min(axis=2) >= -1e-9) & (l0 >= -1e-9)


@pytest.mark.parametrize("recipe", ["golden_radial4", "radial16", "jitter8"])
def test_halo_subsets_hold_every_containing_tet(B, recipe):
    """Points of a brick's partitions grown by one step (where its samples
    can fall, K:278-281) are contained only by tets of its subset."""
    sc = C.build_scene(B, recipe)
    par = C.params(B, recipe)
    step = max(par.s1, par.s2)
    br = BR.scene_bricks(sc, 4)
    subs = BR.brick_tets(sc, br, step * (1.0 + 1e-6))
    rng = np.random.default_rng(3)
    for b in range(br.n):
        inside = np.zeros(sc.mesh.n_tets, bool)
        inside[subs[b]] = True
        pids = np.arange(br.start[b], br.start[b + 1])
        for pid in rng.choice(pids, min(len(pids), 6), replace=False):
            p = sc.partitions[pid]
            lo, hi = np.asarray(p.bounds.lo) - step, np.asarray(p.bounds.hi) + step
            pts = rng.uniform(lo, hi, (48, 3))
            pts[:8] = np.stack([lo, hi, [lo[0], hi[1], lo[2]], [hi[0], lo[1], hi[2]],
                                (lo + hi) / 2, lo + 1e-12, hi - 1e-12, [lo[0], lo[1], hi[2]]])
            hit = _containing(sc, pts)
            assert not np.any(hit[:, ~inside]), (b, pid)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)            # same on every rank
        n = 4096
        state = rng.integers(-2**63, 2**63 - 1, (n, 8), dtype=np.int64)
        f = state[:, :4].view(np.float64)         # acc: specials too
        f[0] = [-0.0, 0.0, np.nan, np.inf]
        f[1] = [5e-324, -5e-324, 1.0, 0.9999]
        owner = rng.integers(0, world, n)         # the brick that advanced each ray
        mine = state.copy()
        mine[owner != rank] = 0                   # B_zero_foreign
        t = torch.from_numpy(mine)
        dist.all_reduce(t)                        # int64 SUM
        q.put((rank, np.array_equal(t.numpy(), state)))
    finally:
        dist.destroy_process_group()


def test_state_exchange_is_exact():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_exchange_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res.values())
