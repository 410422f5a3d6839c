"""Multi-GPU frame merge, host logic on CPU with gloo (world_size 2).

Each rank owns the interleaved 8x4 pixel tiles t % world == rank and writes
them into compact slot-major buffers (what tr_render_frame does with
TrFrame.compact); the frame is reassembled by all-gather + tile scatter and
the counters by an int64 all-reduce (paper_1908_01906_b200/distributed.py).
Here the per-rank tiles are cut from the oracle's full frame, so the merged
result must equal it bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cases as C


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _compact_slots(full, width, height, rank, world):
    """Slot-major compact buffer of `rank`'s tiles (zeros outside the image)."""
    from paper_1908_01906_b200 import distributed as D
    slots = D.slots_per_rank(width, height, world)
    flat = full.reshape(height * width, *full.shape[2:])
    out = np.zeros((slots * D.TILE_PIXELS, *full.shape[2:]), dtype=full.dtype)
    for s in range(slots):
        t = rank + world * s
        if t >= D.num_tiles(width, height):
            continue
        ix, iy = D.tile_pixels(t, width)
        ok = (ix < width) & (iy < height)
        out[s * D.TILE_PIXELS + np.flatnonzero(ok)] = flat[iy[ok] * width + ix[ok]]
    return out


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1908_01906_b200 as B
        from oracle.oracle import OracleScene
        from paper_1908_01906_b200 import distributed as D
        sc = C.build_scene(B, "conftest48")
        cam = B.Camera(position=[10.0, 6.0, 8.0], look_at=[2.0, 2.0, 2.0], up=[0, 1, 0],
                       fov_y_deg=40.0, width=45, height=38)  # ragged: partial tiles
        par = C.params(B, "conftest48")
        rgba, samples, visited, ppart = OracleScene(sc).render(cam, "skip", par)
        w, h = cam.width, cam.height
        # this rank's share of the counters: its own pixels' totals, its partition counts
        mine = np.zeros((h, w), bool)
        for s in range(D.slots_per_rank(w, h, world)):
            t = rank + world * s
            if t < D.num_tiles(w, h):
                ix, iy = D.tile_pixels(t, w)
                ok = (ix < w) & (iy < h)
                mine[iy[ok], ix[ok]] = True
        counters = np.array([samples[mine].sum(), visited[mine].sum()], dtype=np.int64)

        def all_gather(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return torch.cat(out).numpy()

        def all_reduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            return t.numpy()

        m_rgba, m_samples, m_visited, m_cnt = D.merge_partials(
            _compact_slots(rgba, w, h, rank, world), _compact_slots(samples, w, h, rank, world),
            _compact_slots(visited, w, h, rank, world), counters, world, w, h,
            all_gather, all_reduce, D.scatter_tiles_host)
        results[rank] = (np.array_equal(m_rgba, rgba), np.array_equal(m_samples, samples),
                         np.array_equal(m_visited, visited),
                         m_cnt.tolist() == [int(samples.sum()), int(visited.sum())],
                         int(mine.sum()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_frame_merge_is_bit_exact(built_lib, world):
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    assert len(results) == world
    for r in range(world):
        ok_rgba, ok_s, ok_v, ok_c, _ = results[r]
        assert ok_rgba and ok_s and ok_v and ok_c, (r, results[r])
    assert sum(results[r][4] for r in range(world)) == 45 * 38  # every pixel owned once


def test_tile_ownership_partitions_the_frame():
    from paper_1908_01906_b200 import distributed as D
    for w, h, world in [(512, 512, 8), (45, 38, 3), (9, 7, 4), (1, 1, 2)]:
        seen = np.zeros((h, w), np.int32)
        for r in range(world):
            for s in range(D.slots_per_rank(w, h, world)):
                t = r + world * s
                if t >= D.num_tiles(w, h):
                    continue
                assert D.tile_owner(t, world) == (r, s)
                ix, iy = D.tile_pixels(t, w)
                ok = (ix < w) & (iy < h)
                seen[iy[ok], ix[ok]] += 1
        assert (seen == 1).all()
