"""Record-sharded (KD-brick) frames (bricks.py, tr_brick_trace / tr_brick_round;
SURVEY §8f row f4) equal the one-GPU frame bit for bit: every brick holds
only its tets + halo, rays hand their state from brick to brick in rounds.
Here all bricks run on one device (the emulation); the per-round state
exchange of the multi-rank path is covered by test_bricks_dist_gpu below
(two processes sharing the GPU over gloo) and test_bricks.py (CPU)."""

import numpy as np
import pytest

import cases
from paper_1908_01906_b200 import bricks as BR

pytestmark = pytest.mark.gpu


def _same(one, many, track):
    fb1, st1 = one
    fb2, st2 = many
    assert np.array_equal(fb1.rgba, fb2.rgba)
    assert np.array_equal(fb1.samples, fb2.samples)
    assert st1.total_samples == st2.total_samples
    assert st1.partitions_visited_mean == st2.partitions_visited_mean
    if track:
        assert np.array_equal(st1.per_partition_samples, st2.per_partition_samples)


@pytest.mark.parametrize("recipe,n_bricks", [
    ("golden_radial4", 2), ("golden_radial4", 8), ("conftest48", 3), ("inside", 4),
    ("axis", 5), ("a6fog", 4), ("sinus", 6), ("radial16", 2), ("radial16", 7),
    ("jitter16", 4)])
def test_bricks_equal_single_device(B, recipe, n_bricks):
    sc = cases.build_scene(B, recipe)
    cam, par = cases.camera(B, recipe), cases.params(B, recipe)
    if recipe == "conftest48":   # ragged frame
        cam = B.Camera(position=cam.position, look_at=cam.look_at, up=cam.up,
                       fov_y_deg=cam.fov_y_deg, width=45, height=38)
    br = BR.BrickRenderer(sc, n_bricks, max(par.s1, par.s2))
    assert br.bricks.n == n_bricks
    assert max(br.tets_per_brick) < sc.mesh.n_tets or n_bricks == 1 or recipe == "golden_radial4"
    for mode in ("reference", "skip", "skip-adaptive"):
        for jitter in (False, True):
            one = B.render(sc, cam, mode, par, jitter=jitter)
            many = br.render(cam, mode, par, jitter=jitter)
            _same(one, many, mode != "reference")
        assert br.rounds >= 1


@pytest.mark.parametrize("recipe,n_bricks", [("radial16", 4), ("a6fog", 3), ("sinus", 5)])
def test_bricks_unsynchronized_rounds_equal_single_device(B, recipe, n_bricks):
    """n_bricks rounds with no host read in between (the multi-rank default),
    then the synchronized check round: the same frame."""
    sc = cases.build_scene(B, recipe)
    cam, par = cases.camera(B, recipe), cases.params(B, recipe)
    br = BR.BrickRenderer(sc, n_bricks, max(par.s1, par.s2), sync_rounds=False)
    for mode in ("reference", "skip", "skip-adaptive"):
        _same(B.render(sc, cam, mode, par), br.render(cam, mode, par), mode != "reference")
        assert br.rounds == n_bricks   # the check round found no active ray


def test_bricks_radial59(B):
    """BASELINE config 2 scene split into 8 bricks; each brick holds a
    fraction of the tets."""
    sc = cases.build_scene(B, "radial59")
    cam, par = cases.camera(B, "radial59"), cases.params(B, "radial59")
    br = BR.BrickRenderer(sc, 8, par.s2)
    assert max(br.tets_per_brick) < 0.25 * sc.mesh.n_tets
    for mode in ("reference", "skip", "skip-adaptive"):
        _same(B.render(sc, cam, mode, par), br.render(cam, mode, par), mode != "reference")


def test_bricks_refuse_steps_beyond_the_halo(B):
    sc = cases.build_scene(B, "radial16")
    cam, par = cases.camera(B, "radial16", scale=0.125), cases.params(B, "radial16")
    br = BR.BrickRenderer(sc, 2, par.s1)
    br.render(cam, "skip", par)
    with pytest.raises(ValueError):
        br.render(cam, "skip-adaptive", par)


def _dist_worker(rank, world, port, q, exchange="sum"):
    import os
    import sys
    sys.path[:0] = [str(cases.ROOT), str(cases.ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_1908_01906_b200 as B
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = cases.build_scene(B, "radial16")
        cam, par = cases.camera(B, "radial16", scale=0.25), cases.params(B, "radial16")
        br = BR.BrickRenderer(sc, world, par.s2, dist=dist, exchange=exchange)
        out = {}
        for rep in range(2):   # the second frame reuses the inboxes (frame-tagged states)
            for mode in ("reference", "skip-adaptive"):
                fb, st = br.render(cam, mode, par)
                out[mode] = (fb.rgba, fb.samples, st.total_samples, st.partitions_visited_mean,
                             st.per_partition_samples, br.rounds)
        br.close()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange,world", [("sum", 2), ("peer", 2), ("peer", 3)])
def test_bricks_dist_gpu(B, exchange, world):
    """Two or three ranks (processes sharing the GPU) each hold one brick; all
    assemble the one-device frame.  sum: gloo all-reduces of the CUDA state
    array; peer: the march stores each suspended ray's state into the inbox
    of the rank owning its next run through a CUDA IPC mapping (the NVLink
    path), gloo barriers; two frames reuse the inboxes."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sc = cases.build_scene(B, "radial16")
    cam, par = cases.camera(B, "radial16", scale=0.25), cases.params(B, "radial16")
    for mode in ("reference", "skip-adaptive"):
        fb, st = B.render(sc, cam, mode, par)
        for r in range(world):
            rgba, samples, tot, vis, ppart, rounds = res[r][mode]
            assert np.array_equal(rgba, fb.rgba)
            assert np.array_equal(samples, fb.samples)
            assert tot == st.total_samples and vis == st.partitions_visited_mean
            if mode != "reference":
                assert np.array_equal(ppart, st.per_partition_samples)
