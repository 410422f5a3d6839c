"""Multi-GPU frame rendering: one process per GPU, the scene
replicated in every GPU's HBM, the frame's 8x4 pixel tiles interleaved over
the ranks (tile t -> rank t % world, slot t // world), so long and short rays
spread evenly.  The merge is exactly the frame's data dependencies, and only
rank 0 (the caller that returns the image) receives it:

  * disjoint pixel tiles   -> NCCL gather of each rank's compact slots to
                              rank 0, then tr_scatter_tiles into image layout
  * mergeable aggregates   -> NCCL reduce (int64 sum) to rank 0 of
                              [total samples, visited sum, per-partition samples]

With the gloo backend (CPU-side debugging, the 2-process one-GPU test) the
same collectives run on host copies of the device tensors.

Integer sums are order independent and tiles are disjoint, so an N-GPU frame
is bit-identical to the 1-GPU frame (tests/test_distributed.py checks the
host-side logic with gloo on CPU; tests/test_parity_gpu.py the kernels).
"""

from __future__ import annotations

import atexit
import ctypes as C
import mmap
import os
import secrets
import sys
import time

import numpy as np

from . import _lib
from .device import last_launches

TILE_W, TILE_H = 8, 4
TILE_PIXELS = TILE_W * TILE_H


def num_tiles(width: int, height: int) -> int:
    return ((width + TILE_W - 1) // TILE_W) * ((height + TILE_H - 1) // TILE_H)


def slots_per_rank(width: int, height: int, world: int) -> int:
    return (num_tiles(width, height) + world - 1) // world


def tile_owner(tile: int, world: int) -> tuple[int, int]:
    """(rank, slot) of a tile under the interleaved assignment."""
    return tile % world, tile // world


def tile_pixels(tile: int, width: int):
    """(ix, iy) of the 32 lanes of a tile (lane = 8*row + col)."""
    tiles_x = (width + TILE_W - 1) // TILE_W
    lane = np.arange(TILE_PIXELS)
    ix = (tile % tiles_x) * TILE_W + lane % TILE_W
    iy = (tile // tiles_x) * TILE_H + lane // TILE_W
    return ix, iy


def scatter_tiles_host(width, height, world, slots, rgba_all, samples_all, visited_all):
    """numpy statement of tr_scatter_tiles (used by the CPU/gloo tests to
    check the merge plumbing; the product calls the CUDA kernel)."""
    rgba = np.zeros((height * width, 4))
    samples = np.zeros(height * width, np.int64)
    visited = np.zeros(height * width, np.int32)
    n = num_tiles(width, height)
    for r in range(world):
        for s in range(slots):
            t = r + world * s
            if t >= n:
                continue
            ix, iy = tile_pixels(t, width)
            ok = (ix < width) & (iy < height)
            src = (r * slots + s) * TILE_PIXELS + np.arange(TILE_PIXELS)
            dst = iy * width + ix
            rgba[dst[ok]] = rgba_all[src[ok]]
            samples[dst[ok]] = samples_all[src[ok]]
            visited[dst[ok]] = visited_all[src[ok]]
    return rgba.reshape(height, width, 4), samples.reshape(height, width), \
        visited.reshape(height, width)


def merge_partials(rank_rgba, rank_samples, rank_visited, rank_counters, world, width, height,
                   all_gather, all_reduce, scatter):
    """The collective part of a sharded frame, with the transport injected
    (torch.distributed NCCL on GPU, gloo in the CPU tests).  Returns the
    image-layout rgba/samples/visited and the summed counters."""
    g_rgba = all_gather(rank_rgba)
    g_samples = all_gather(rank_samples)
    g_visited = all_gather(rank_visited)
    counters = all_reduce(rank_counters)
    slots = slots_per_rank(width, height, world)
    return (*scatter(width, height, world, slots, g_rgba, g_samples, g_visited), counters)


def _gloo() -> bool:
    import torch.distributed as dist
    return dist.get_backend() == "gloo"


def _gather0(src, dst, rank: int, world: int) -> None:
    """dst (rank 0: world equal chunks) <- every rank's src."""
    import torch
    import torch.distributed as dist
    if _gloo():
        h = src.cpu()
        lst = [torch.empty_like(h) for _ in range(world)] if rank == 0 else None
        dist.gather(h, lst, dst=0)
        if rank == 0:
            dst.copy_(torch.cat(lst))
        return
    dist.gather(src, list(dst.chunk(world)) if rank == 0 else None, dst=0)


def _reduce0(t) -> None:
    import torch.distributed as dist
    if _gloo():
        h = t.cpu()
        dist.reduce(h, dst=0)
        t.copy_(h)
        return
    dist.reduce(t, dst=0)


class ShardedFrame:
    """One frame's launch plan on one rank: epoch, frame descriptor, buffers
    and (world > 1) the NCCL merge.  world == 1 renders straight into the
    image layout with no collective."""

    def __init__(self, dscene, scene, camera, mode_id: int, params, *, track: bool, rank: int = 0,
                 world: int = 1, flags: int = 0, jitter: bool = False, compact=None):
        import torch
        self.torch = torch
        self.dscene = dscene
        self.scene, self.camera, self.params = scene, camera, params
        self.world, self.rank = world, rank
        self.w, self.h = int(camera.width), int(camera.height)
        # compact tile slots + the gather / reduce (default: world > 1)
        self.compact = (world > 1) if compact is None else bool(compact)
        self.slots = slots_per_rank(self.w, self.h, world) if self.compact else 0
        self.epoch = dscene.epoch(scene.meta_state(), params)
        self.frame = dscene.frame_desc(scene, camera, mode_id, params, jitter, track, flags,
                                       shard_rank=rank, shard_count=world, compact=self.compact)
        self.fb = dscene.frame_buffers(self.w, self.h, compact_slots=self.slots)
        dev = dscene.device
        if self.compact:
            n = world * self.slots * TILE_PIXELS
            self.g_rgba = torch.empty((n, 4), dtype=torch.float64, device=dev)
            self.g_samples = torch.empty(n, dtype=torch.int64, device=dev)
            self.g_visited = torch.empty(n, dtype=torch.int32, device=dev)
            self.rgba = torch.empty((self.h * self.w, 4), dtype=torch.float64, device=dev)
            self.samples = torch.empty(self.h * self.w, dtype=torch.int64, device=dev)
            self.visited = torch.empty(self.h * self.w, dtype=torch.int32, device=dev)
            self.local = torch.empty(2, dtype=torch.int64, device=dev)
        else:
            self.rgba, self.samples, self.visited = self.fb.rgba, self.fb.samples, self.fb.visited
            self.local = None

    def launches_per_step(self) -> int:
        """Our kernels per frame as the library counted them in the last
        tr_render_frame (trace + order + march launches per ray chunk; the
        auto lane width launches two march kernels, one returns at once),
        plus the tile scatter when sharded."""
        import ctypes as C
        import numpy as np
        out = np.zeros(3, np.int64)
        _lib.check(_lib.lib().tr_last_launch(_lib.ptr(out, C.c_int64)), "tr_last_launch")
        return int(out[0]) + (1 if self.compact else 0)

    def run(self, stream, kernel_events=None, march_events=None):
        """One frame.  kernel_events brackets the whole render call (trace +
        order + march kernels); march_events the march kernel alone."""
        fb = self.fb
        fb.counters.zero_()
        out = fb.outputs()
        if march_events is not None:
            for ev in march_events:  # torch creates its CUDA event lazily on first record
                if not ev.cuda_event:
                    ev.record(stream)
            out.ev_march_begin = march_events[0].cuda_event
            out.ev_march_end = march_events[1].cuda_event
        if kernel_events is not None:
            kernel_events[0].record(stream)
        _lib.check(_lib.lib().tr_render_frame(C.byref(self.dscene.desc), C.byref(self.epoch.desc),
                                              C.byref(self.frame), C.byref(out),
                                              C.c_void_p(stream.cuda_stream)), "tr_render_frame")
        if kernel_events is not None:
            kernel_events[1].record(stream)
        if self.compact:
            self.local.copy_(fb.counters[:2])
            _gather0(fb.rgba, self.g_rgba, self.rank, self.world)
            _gather0(fb.samples, self.g_samples, self.rank, self.world)
            _gather0(fb.visited, self.g_visited, self.rank, self.world)
            _reduce0(fb.counters)
            if self.rank != 0:
                return
            _lib.check(_lib.lib().tr_scatter_tiles(
                self.w, self.h, self.world, C.c_void_p(self.g_rgba.data_ptr()),
                C.c_void_p(self.g_samples.data_ptr()), C.c_void_p(self.g_visited.data_ptr()),
                self.slots, C.c_void_p(self.rgba.data_ptr()), C.c_void_p(self.samples.data_ptr()),
                C.c_void_p(self.visited.data_ptr()), C.c_void_p(stream.cuda_stream)),
                "tr_scatter_tiles")

    def total_samples(self) -> int:
        return int(self.fb.counters[0].item())

    def local_samples(self) -> int:
        if self.compact:
            return int(self.local[0].item())
        return int(self.fb.counters[0].item())

    def local_pixels(self) -> int:
        if not self.compact:
            return self.w * self.h
        n = num_tiles(self.w, self.h)
        mine = len(range(self.rank, n, self.world))
        return min(mine * TILE_PIXELS, self.w * self.h)

    def host_outputs(self):
        """(rgba (H,W,4), samples (H,W), counters) on the host."""
        return (self.rgba.view(self.h, self.w, 4).cpu().numpy(),
                self.samples.view(self.h, self.w).cpu().numpy(),
                self.fb.counters.cpu().numpy())


_FRAMES: dict = {}


def _all_reduce(t) -> None:
    import torch.distributed as dist
    if _gloo():
        h = t.cpu()
        dist.all_reduce(h)
        t.copy_(h)
        return
    dist.all_reduce(t)


class SharedBlocks:
    """Frame result blocks (rgba f64 | samples i64, image layout) in
    page-locked host memory shared by the ranks of one node: /dev/shm files
    that every rank maps and registers with CUDA (tr_host_register).  Each
    rank's kernels store its own pixel tiles straight into the block over its
    own PCIe link, so rank 0 returns the frame with no gather and no
    device->host copy of the image.

    A block is handed out again only once no array rank 0 returned views it
    (the views' base is the block's array: its reference count says so).
    Rank 0 picks the NEXT frame's block while a frame runs and every rank
    learns it from that frame's counter all-reduce, so no extra collective
    is needed; a new block is created by rank 0 before it is announced."""

    MAX_BLOCKS = 64

    def __init__(self, token: str, nbytes: int, rank: int):
        self.token, self.nbytes, self.rank = token, nbytes, rank
        self.blocks = []   # [base uint8 array over the mapping, device address]
        self.cur = 0
        if rank == 0:
            self._create(0)

    def _path(self, i: int) -> str:
        return f"/dev/shm/tetray_b200_{self.token}_{self.nbytes}_{i}"

    def _create(self, i: int) -> None:
        fd = os.open(self._path(i), os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
        try:
            os.ftruncate(fd, self.nbytes)
        finally:
            os.close(fd)

    def block(self, i: int):
        """(base array, device address) of block i, mapped on first use."""
        while len(self.blocks) <= i:
            k = len(self.blocks)
            fd = os.open(self._path(k), os.O_RDWR)
            try:
                mm = mmap.mmap(fd, self.nbytes)
            finally:
                os.close(fd)
            base = np.frombuffer(mm, dtype=np.uint8)
            dptr = C.c_void_p()
            _lib.check(_lib.lib().tr_host_register(C.c_void_p(base.ctypes.data), self.nbytes,
                                                   C.byref(dptr)), "tr_host_register")
            self.blocks.append([base, int(dptr.value)])
        return self.blocks[i][0], self.blocks[i][1]

    def pick_next(self) -> int:
        """Rank 0: a block no returned frame views, other than the current one."""
        for i, b in enumerate(self.blocks):
            if i != self.cur and sys.getrefcount(b[0]) == 2:   # the list entry + the argument
                return i
        k = len(self.blocks)
        if k >= self.MAX_BLOCKS:
            raise RuntimeError(f"render(distributed=True): {k} frames still referenced")
        self._create(k)
        self.block(k)
        return k

    def close(self) -> None:
        for base, _ in self.blocks:
            _lib.lib().tr_host_unregister(C.c_void_p(base.ctypes.data))
        if self.rank == 0:
            for i in range(len(self.blocks)):
                try:
                    os.unlink(self._path(i))
                except OSError:
                    pass
        self.blocks = []


_SHARED: dict = {}
_TOKEN: list = []


def _shared_blocks(nbytes: int, rank: int, device):
    """The node-shared block pool of one frame size (collective on first
    use), or None when any rank could not create / map / page-lock it (the
    frame then takes the gather path; every rank agrees)."""
    import torch
    import torch.distributed as dist
    if nbytes in _SHARED:
        return _SHARED[nbytes]
    if not _TOKEN:   # one name prefix per process group, from rank 0
        obj = [f"{os.getpid()}_{secrets.token_hex(4)}" if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        _TOKEN.append(obj[0])
        atexit.register(release_shared_frames)
    pool, ok = None, 1
    try:
        pool = SharedBlocks(_TOKEN[0], nbytes, rank)
    except OSError:
        ok = 0
    dist.barrier()   # block 0 exists before the other ranks map it
    if pool is not None:
        try:
            pool.block(0)
        except (OSError, RuntimeError):
            ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device="cpu" if _gloo() else device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 0 and pool is not None:
        pool.close()
        pool = None
    _SHARED[nbytes] = pool
    return pool


def release_shared_frames() -> None:
    """Unmap the node-shared result blocks (rank 0 also removes their
    /dev/shm files; arrays rank 0 returned stay valid).  Runs at exit; call it
    where processes end without atexit (multiprocessing workers)."""
    for pool in _SHARED.values():
        if pool is not None:
            pool.close()
    _SHARED.clear()


def _node_local(world: int) -> bool:
    """Every rank on this host (torchrun exports LOCAL_WORLD_SIZE)."""
    return int(os.environ.get("LOCAL_WORLD_SIZE", world)) == world


def render_sharded(scene, camera, mode: str, params, *, jitter: bool = False,
                   track_per_partition: bool = True, device=None, flags: int = 0):
    """render() over the ranks of the initialised torch.distributed group:
    every rank calls it with the same arguments; rank 0 returns the
    (Framebuffer, RenderStats) of the whole frame, bit-identical to the
    one-GPU render(); the other ranks return (None, None).

    Ranks of one node write their tiles into a node-shared page-locked
    frame (SharedBlocks) and all-reduce the counters; across nodes the
    tiles are gathered to rank 0 over NCCL (render_sharded_gather)."""
    import torch
    import torch.distributed as dist

    from .device import device_scene_for
    from .render import _MODE_IDS, Framebuffer, RenderStats
    rank, world = dist.get_rank(), dist.get_world_size()
    if not _node_local(world):
        return render_sharded_gather(scene, camera, mode, params, jitter=jitter,
                                     track_per_partition=track_per_partition, device=device,
                                     flags=flags)
    dscene = device_scene_for(scene, device)
    track = track_per_partition and mode != "reference"
    w, h = int(camera.width), int(camera.height)
    npx = w * h
    P = dscene.n_parts
    pool = _shared_blocks(40 * npx, rank, dscene.device)
    if pool is None:
        return render_sharded_gather(scene, camera, mode, params, jitter=jitter,
                                     track_per_partition=track_per_partition, device=device,
                                     flags=flags)
    frame = dscene.frame_desc(scene, camera, _MODE_IDS[mode], params, jitter, track, flags,
                              shard_rank=rank, shard_count=world, compact=False)
    t0 = time.perf_counter()
    with dscene.lock, torch.cuda.device(dscene.device):
        stream = torch.cuda.current_stream(dscene.device)
        ep = dscene.epoch(scene.meta_state(), params, stream)
        fb = dscene.frame_buffers(w, h)
        base, dptr = pool.block(pool.cur)
        nxt = pool.pick_next() if rank == 0 else 0
        out = fb.outputs()
        out.rgba, out.samples = dptr, dptr + 32 * npx   # this rank's tiles, in place
        fb.counters.zero_()
        _lib.check(_lib.lib().tr_render_frame(C.byref(dscene.desc), C.byref(ep.desc),
                                              C.byref(frame), C.byref(out),
                                              C.c_void_p(stream.cuda_stream)), "tr_render_frame")
        # [totals | work | per-partition samples | next block]: one all-reduce;
        # it runs after every rank's frame, so rank 0 then sees every tile
        red = torch.empty(4 + P, dtype=torch.int64, device=dscene.device)
        red[:3 + P].copy_(fb.counters)
        red[3 + P:].fill_(nxt)
        _all_reduce(red)
        cnt_h = torch.empty(4 + P, dtype=torch.int64, pin_memory=True)
        cnt_h.copy_(red, non_blocking=True)
        stream.synchronize()
    cnt = cnt_h.numpy()
    pool.cur = int(cnt[3 + P])
    if rank != 0:
        return None, None
    rgba = base[:32 * npx].view(np.float64).reshape(h, w, 4)
    samples = base[32 * npx:40 * npx].view(np.int64).reshape(h, w)
    fbuf = Framebuffer(width=w, height=h, rgba=rgba, samples=samples,
                       background=np.asarray(scene.background, dtype=np.float64).copy())
    st = RenderStats(total_samples=int(cnt[0]), wall_ms=(time.perf_counter() - t0) * 1e3,
                     partitions_visited_mean=float(np.float64(cnt[1]) / np.float64(w * h)),
                     per_partition_samples=cnt[3:3 + P].copy() if track else None,
                     samples=samples, device_ms=0.0, gpu_launches=last_launches())
    return fbuf, st


def render_sharded_gather(scene, camera, mode: str, params, *, jitter: bool = False,
                          track_per_partition: bool = True, device=None, flags: int = 0):
    """render_sharded across nodes: each rank's compact tiles gathered to
    rank 0 over NCCL, counters reduced there, rank 0 reads the frame back."""
    import torch
    import torch.distributed as dist

    from .device import device_scene_for
    from .render import _MODE_IDS, Framebuffer, RenderStats
    rank, world = dist.get_rank(), dist.get_world_size()
    dscene = device_scene_for(scene, device)
    track = track_per_partition and mode != "reference"
    w, h = int(camera.width), int(camera.height)
    key = (id(dscene), w, h, world, rank, _MODE_IDS[mode], track, bool(jitter), flags)
    runner = _FRAMES.get(key)
    if runner is None or runner.scene is not scene:
        runner = ShardedFrame(dscene, scene, camera, _MODE_IDS[mode], params, track=track,
                              rank=rank, world=world, flags=flags, jitter=jitter, compact=True)
        _FRAMES.clear()
        _FRAMES[key] = runner
    runner.camera, runner.params = camera, params
    runner.frame = dscene.frame_desc(scene, camera, _MODE_IDS[mode], params, jitter, track,
                                     flags, shard_rank=rank, shard_count=world, compact=True)
    t0 = time.perf_counter()
    with dscene.lock, torch.cuda.device(dscene.device):
        stream = torch.cuda.current_stream(dscene.device)
        runner.epoch = dscene.epoch(scene.meta_state(), params, stream)
        runner.run(stream)
        if rank != 0:
            stream.synchronize()
            return None, None
        rgba_h = torch.empty((h, w, 4), dtype=torch.float64, pin_memory=True)
        samp_h = torch.empty((h, w), dtype=torch.int64, pin_memory=True)
        cnt_h = torch.empty(runner.fb.counters.numel(), dtype=torch.int64, pin_memory=True)
        rgba_h.view(-1, 4).copy_(runner.rgba, non_blocking=True)
        samp_h.view(-1).copy_(runner.samples, non_blocking=True)
        cnt_h.copy_(runner.fb.counters, non_blocking=True)
        stream.synchronize()
    cnt = cnt_h.numpy()
    samples = samp_h.numpy()
    fb = Framebuffer(width=w, height=h, rgba=rgba_h.numpy(), samples=samples,
                     background=np.asarray(scene.background, dtype=np.float64).copy())
    st = RenderStats(total_samples=int(cnt[0]), wall_ms=(time.perf_counter() - t0) * 1e3,
                     partitions_visited_mean=float(np.float64(cnt[1]) / np.float64(w * h)),
                     per_partition_samples=cnt[3:].copy() if track else None, samples=samples,
                     device_ms=0.0, gpu_launches=runner.launches_per_step())
    return fb, st


def bench_e2e_sharded(scene, camera, mode: str, params, steps: int, device) -> dict:
    """End-to-end sharded frames through render_sharded: the epoch is
    re-uploaded (H2D) every step on every rank and the image reaches host
    memory every step (one node: each rank's tiles stored into the shared
    page-locked frame; across nodes: gathered to rank 0 and read back);
    wall clock, max over ranks."""
    import torch
    import torch.distributed as dist

    from .device import device_scene_for
    dscene = device_scene_for(scene, device)
    for _ in range(3):
        render_sharded(scene, camera, mode, params, device=device)
    dist.barrier()
    t0 = time.perf_counter()
    fb = st = None
    for _ in range(steps):
        dscene.mark_epochs_stale()   # every step copies the metadata epoch again
        fb, st = render_sharded(scene, camera, mode, params, device=device)
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dscene.device)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    ep = next(iter(dscene._epochs.values()))
    if dist.get_rank() != 0:
        return None
    d2h = fb.rgba.nbytes + fb.samples.nbytes + 8 * (3 + dscene.n_parts)
    return {"value": st.total_samples * steps / float(dt[0]), "unit": "samples/s",
            "h2d_bytes_per_step": int(ep.h2d_bytes), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": float(dt[0]) * 1000.0 / steps, "steps": steps}
