"""Multi-process sharded frames through the public render(distributed=True):
N processes (sharing the one GPU of this run, gloo transport: NCCL refuses two
ranks on one device) each render their interleaved 8x4 pixel tiles straight
into the node-shared page-locked frame (distributed.SharedBlocks), the
counters are all-reduced and rank 0 returns the frame; the cross-node
variant (compact tiles gathered to rank 0, render_sharded_gather) too.  It must be
bit-identical to the one-process frame -- rows are independent
(pkg/src/tetray/_kernels.py:323-328), integer sums are order-free."""

import socket

import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu

RECIPES = (("radial16", 0.25), ("golden_radial4", 1.0), ("axis", 1.0), ("radial59", 0.5))


@pytest.fixture(scope="module")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B


def _worker(rank, world, port, q, path):
    import os
    import sys
    sys.path[:0] = [str(cases.ROOT), str(cases.ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # "gather": as if every rank were on its own node (render_sharded_gather)
    os.environ["LOCAL_WORLD_SIZE"] = "1" if path == "gather" else str(world)
    import torch
    import torch.distributed as dist

    import paper_1908_01906_b200 as B
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for recipe, scale in RECIPES:
            sc = cases.build_scene(B, recipe)
            cam, par = cases.camera(B, recipe, scale=scale), cases.params(B, recipe)
            for mode in ("reference", "skip-adaptive"):
                fb, st = B.render(sc, cam, mode, par, distributed=True)
                if rank == 0:
                    out[(recipe, mode)] = (fb.rgba, fb.samples, st.total_samples,
                                           st.partitions_visited_mean, st.per_partition_samples)
                else:
                    assert fb is None and st is None
        q.put((rank, out))
    finally:
        from paper_1908_01906_b200.distributed import release_shared_frames
        release_shared_frames()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,path", [(2, "shared"), (3, "shared"), (2, "gather")])
def test_distributed_render_equals_one_gpu_frame(B, world, path):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, path)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for recipe, scale in RECIPES:
        sc = cases.build_scene(B, recipe)
        cam, par = cases.camera(B, recipe, scale=scale), cases.params(B, recipe)
        for mode in ("reference", "skip-adaptive"):
            fb, st = B.render(sc, cam, mode, par)
            rgba, samples, tot, vis, ppart = res[0][(recipe, mode)]
            assert np.array_equal(rgba, fb.rgba), (recipe, mode)
            assert np.array_equal(samples, fb.samples), (recipe, mode)
            assert tot == st.total_samples and vis == st.partitions_visited_mean
            if mode == "reference":
                assert ppart is None
            else:
                assert np.array_equal(ppart, st.per_partition_samples)
