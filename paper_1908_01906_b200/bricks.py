"""Exact record-sharded (KD-brick) rendering -- SURVEY §8f row f4.

For meshes larger than one GPU's HBM the tets are split by KD subtree: the
partitions (KD leaves, partitions.py:73-128, left-first DFS ids) are grouped
into convex bricks, and brick b's device scene holds only the tets whose
padded boxes meet brick b's box grown by a halo of the largest step.  The
partition structures (BVH, BSP, boxes, activity) are small and replicated.

A frame (csrc/render.cu, tr_brick_trace / tr_brick_round):

1. every rank traces the full front-to-back interval list of each ray
   (K:360-391), exactly as the one-GPU frame does; in mode 0 the mesh-box
   interval is cut at the brick boxes;
2. rounds: each active ray's next *run* -- the consecutive samples whose
   intervals belong to one brick -- is marched by that brick's rank, starting
   from the ray state the previous run left (acc rgba, samples taken,
   position in the interval list).  A run ends at the brick's last interval or
   at early termination (K:285-295, K:388-389), where the pixel is written;
3. between rounds the ranks exchange the states: either (SUM) each active
   ray was advanced by exactly one rank, so an int64 SUM all-reduce of the
   state array with every other entry zeroed reproduces it bit for bit, or
   (PEER, one node) the march stores a suspended ray's state straight into
   the inbox of the rank owning its next run (CUDA IPC over NVLink) and the
   ranks only meet at a barrier.

Compositing order, sample positions (entry + (k + phase) * step with the
ray's own k), per-partition counts and `visited` are the one-GPU frame's, so
the result is bit-identical (tests/test_bricks_gpu.py).  Why a halo suffices:
every sample of a partition's interval lies on the ray inside the
partition's box, except the forced k = 0 sample, which can pass the exit by
< one step (K:278-281); a point's lowest-index containing tet has a padded
box holding the point, so it is in the subset of any brick whose grown box
holds the point.  Global tet ids are kept (leaf id lists and subtree minima),
so "lowest index" is unchanged.

`BrickRenderer` runs all bricks on one device (the single-GPU emulation the
tests use) or, with `dist`, one brick per rank of a torch.distributed group
(NCCL on GPUs; the exchange is one all_reduce per round).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .device import DeviceScene, FrameBuffers, _padded_boxes, resolve_device


@dataclass
class Bricks:
    """Convex bricks over the partitions: brick b = partitions [start[b], start[b+1])."""
    start: np.ndarray       # (n+1,) DFS partition ranges
    lo: np.ndarray          # (n, 3) brick boxes
    hi: np.ndarray
    owner: np.ndarray       # (P,) int16 brick of each partition

    @property
    def n(self) -> int:
        return len(self.lo)


def _union_ok(lo, hi, vol, a, b):
    """Box of leaves [a, b) and whether it is their exact union (convex)."""
    blo, bhi = lo[a:b].min(axis=0), hi[a:b].max(axis=0)
    bv = float(np.prod(bhi - blo))
    return blo, bhi, abs(bv - float(vol[a:b].sum())) <= 1e-9 * max(bv, 1e-300)


def kd_bricks(leaf_lo: np.ndarray, leaf_hi: np.ndarray, weight: np.ndarray, n_bricks: int) -> Bricks:
    """Split the DFS-ordered KD leaves into n_bricks contiguous ranges whose
    unions are boxes (every KD subtree is one), balancing `weight` (tets)."""
    leaf_lo = np.asarray(leaf_lo, np.float64)
    leaf_hi = np.asarray(leaf_hi, np.float64)
    w = np.asarray(weight, np.float64)
    P = len(leaf_lo)
    if not 1 <= n_bricks <= min(P, 64):
        raise ValueError(f"n_bricks must lie in [1, min(partitions, 64)], got {n_bricks}")
    vol = np.prod(leaf_hi - leaf_lo, axis=1)
    ranges = [(0, P)]
    while len(ranges) < n_bricks:
        best = None
        for idx in np.argsort([-w[a:b].sum() for a, b in ranges]):
            a, b = ranges[idx]
            if b - a < 2:
                continue
            total = w[a:b].sum()
            cw = np.cumsum(w[a:b])
            # candidate cuts by closeness to half the weight
            for m in a + 1 + np.argsort(np.abs(cw[:-1] - total / 2.0)):
                plo, phi, pok = _union_ok(leaf_lo, leaf_hi, vol, a, m)
                slo, shi, sok = _union_ok(leaf_lo, leaf_hi, vol, m, b)
                if not (pok and sok):
                    continue
                if np.any((phi <= slo) | (shi <= plo)):   # interiors disjoint on some axis
                    best = (idx, m)
                    break
            if best is not None:
                break
        if best is None:
            raise ValueError(f"cannot split the partitions into {n_bricks} convex bricks")
        idx, m = best
        a, b = ranges.pop(idx)
        ranges[idx:idx] = [(a, m), (m, b)]
    start = np.array([r[0] for r in ranges] + [P], np.int64)
    lo = np.stack([leaf_lo[a:b].min(axis=0) for a, b in ranges])
    hi = np.stack([leaf_hi[a:b].max(axis=0) for a, b in ranges])
    owner = np.empty(P, np.int16)
    for k, (a, b) in enumerate(ranges):
        owner[a:b] = k
    return Bricks(start, lo, hi, owner)


def scene_bricks(scene, n_bricks: int) -> Bricks:
    """Bricks of a Scene from its partitions' KD leaf boxes, weighted by tets."""
    parts = scene.partitions
    lo = np.stack([np.asarray(p.leaf_bounds.lo) for p in parts])
    hi = np.stack([np.asarray(p.leaf_bounds.hi) for p in parts])
    w = np.array([len(p.element_ids) for p in parts], np.float64)
    return kd_bricks(lo, hi, w, n_bricks)


def brick_tets(scene, bricks: Bricks, halo: float) -> list[np.ndarray]:
    """Ascending global tet ids per brick: padded tet boxes meeting the brick
    box grown by `halo`."""
    lo, hi = _padded_boxes(scene)
    out = []
    for b in range(bricks.n):
        glo, ghi = bricks.lo[b] - halo, bricks.hi[b] + halo
        m = np.all(hi >= glo, axis=1) & np.all(lo <= ghi, axis=1)
        out.append(np.nonzero(m)[0].astype(np.int64))
    return out


class BrickRenderer:
    """Record-sharded frames of one scene over n bricks (see the module doc).

    max_step: the largest step any frame will use (s2 in skip-adaptive, else
    s1): it sets the halo, so frames with larger steps are refused."""

    def __init__(self, scene, n_bricks: int, max_step: float, device=None, dist=None,
                 sync_rounds: Optional[bool] = None, exchange: str = "sum"):
        """sync_rounds: read the active-ray count back after every round
        (default for the one-device emulation) or run n_bricks rounds with no
        host read first (default with `dist`: a ray's runs cross each convex
        brick at most once, so n rounds finish every ray; one synchronized
        round then confirms it -- and keeps going if ever needed).

        exchange (with `dist`): "sum" -- an int64 SUM all-reduce of the whole
        state array per round; "peer" -- when a run suspends, the march
        stores the ray's state into the inbox of the one rank owning its next
        run through CUDA IPC mappings (NVLink on one node), so each suspended
        ray moves once and a round needs just a barrier (the ranks must share
        a node)."""
        import torch
        if exchange not in ("sum", "peer"):
            raise ValueError(f"exchange must be 'sum' or 'peer', not {exchange!r}")
        self.exchange = exchange if dist is not None else "sum"
        self._frame_no = 0
        self._ipc = []   # (own inbox pointer, opened peer pointers)
        self.scene = scene
        self.device = resolve_device(device)
        self.dist = dist
        self.bricks = scene_bricks(scene, n_bricks)
        self.max_step = float(max_step)
        pad = 1e-9 * max(scene.mesh.bounds.diagonal(), 1e-30)
        self.halo = self.max_step * (1.0 + 1e-6) + pad
        subsets = brick_tets(scene, self.bricks, self.halo)
        self.tets_per_brick = [len(s) for s in subsets]
        if dist is None:
            mine = list(range(self.bricks.n))
        else:
            if dist.get_world_size() != self.bricks.n:
                raise ValueError("one brick per rank: world size must equal n_bricks")
            mine = [dist.get_rank()]
        self.mine = mine
        self.sync_rounds = (dist is None) if sync_rounds is None else bool(sync_rounds)
        self.devs = {b: DeviceScene(scene, self.device, tet_subset=subsets[b]) for b in mine}
        d = self.device
        self.t_owner = torch.from_numpy(self.bricks.owner.copy()).to(d)
        self.t_lo = torch.from_numpy(np.ascontiguousarray(self.bricks.lo)).to(d)
        self.t_hi = torch.from_numpy(np.ascontiguousarray(self.bricks.hi)).to(d)
        self.counters = torch.zeros(4, dtype=torch.int32, device=d)
        self._bufs = {}

    def resident_bytes(self) -> dict:
        return {b: dev.resident_bytes for b, dev in self.devs.items()}

    def _buffers(self, w: int, h: int):
        import torch
        key = (w, h)
        if key not in self._bufs:
            dev0 = next(iter(self.devs.values()))
            fb = FrameBuffers(dev0, w, h)
            rays = -(-w // 8) * 8 * (-(-h // 4)) * 4   # whole 8x4 tiles: one ray chunk
            fb.scratch_bytes = int(_lib.lib().tr_scratch_bytes(rays))
            fb.scratch = torch.empty(fb.scratch_bytes, dtype=torch.uint8, device=self.device)
            state = torch.empty(rays * _lib.RAY_STATE_BYTES, dtype=torch.uint8, device=self.device)
            queue = torch.empty(rays, dtype=torch.int32, device=self.device)
            peer = self._peer_inboxes(rays) if self.exchange == "peer" else None
            self._bufs[key] = (fb, state, queue, peer)
        return self._bufs[key]

    def _peer_inboxes(self, rays: int):
        """PEER exchange: this rank's [2][rays] inbox (CUDA IPC allocation)
        and the device table of every rank's inbox mapped here."""
        import torch
        L = _lib.lib()
        nbytes = 2 * rays * _lib.RAY_STATE_BYTES
        own, h = C.c_void_p(), (C.c_ubyte * 64)()
        with torch.cuda.device(self.device):
            _lib.check(L.tr_ipc_alloc(nbytes, C.byref(own), h), "tr_ipc_alloc")
            handles = [None] * self.dist.get_world_size()
            self.dist.all_gather_object(handles, bytes(h))
            table, opened = [], []
            for r, hr in enumerate(handles):
                if r == self.dist.get_rank():
                    table += [0, 0]
                    continue
                buf = C.create_string_buffer(hr, 64)
                p = C.c_void_p()
                _lib.check(L.tr_ipc_open(C.cast(buf, C.c_void_p), C.byref(p)), "tr_ipc_open")
                opened.append(p.value)
                table += [p.value, p.value + rays * _lib.RAY_STATE_BYTES]
            t_table = torch.tensor(table, dtype=torch.int64, device=self.device)
        self._ipc.append((own.value, opened))
        self._token = torch.zeros(1, dtype=torch.int32, device=self.device)
        return own.value, t_table

    def _round_barrier(self, stream) -> None:
        """PEER exchange: every rank's round (and its NVLink stores) is done
        before any rank plans the next one."""
        if self.dist.get_backend() == "nccl":
            self.dist.all_reduce(self._token)   # stream-ordered, no host wait
        else:
            stream.synchronize()
            self.dist.barrier()

    def close(self) -> None:
        """Release the PEER inboxes (collective: every rank calls it)."""
        if not self._ipc:
            return
        import torch
        torch.cuda.synchronize(self.device)
        self.dist.barrier()
        L = _lib.lib()
        for own, opened in self._ipc:
            for p in opened:
                L.tr_ipc_close(C.c_void_p(p))
        self.dist.barrier()
        for own, _ in self._ipc:
            L.tr_dev_free(C.c_void_p(own))
        self._ipc = []
        self._bufs.clear()

    def render(self, camera, mode: str, params, *, jitter: bool = False,
               track_per_partition: bool = True, flags: int = 0, profile: bool = False):
        """Same contract and results as render(); the frame is assembled on
        every rank (dist: after the final exchange)."""
        import torch
        from .render import _MODE_IDS, Framebuffer, RenderStats
        if mode not in _MODE_IDS:
            raise ValueError(f"unknown mode {mode!r}")
        mid = _MODE_IDS[mode]
        step = float(params.s2) if mid == 2 else float(params.s1)
        if step > self.max_step:
            raise ValueError(f"step {step} exceeds the bricks' halo step {self.max_step}")
        track = track_per_partition and mode != "reference"
        sc = self.scene
        w, h = int(camera.width), int(camera.height)
        dev0 = next(iter(self.devs.values()))
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            ep = dev0.epoch(sc.meta_state(), params)   # partition data is global
            frame = dev0._frame_desc(sc, camera, mid, params, jitter, track, flags, 0, 1, False)
            fb, state, queue, peer = self._buffers(w, h)
            self._frame_no += 1
            fb.counters.zero_()
            if self.dist is not None:
                fb.rgba.zero_(); fb.samples.zero_(); fb.visited.zero_()
            out = fb.outputs()
            B = _lib.TrBricks(rank=self.mine[0], n_bricks=self.bricks.n,
                              owner=self.t_owner.data_ptr(), brick_lo=self.t_lo.data_ptr(),
                              brick_hi=self.t_hi.data_ptr(), state=state.data_ptr(),
                              queue=queue.data_ptr(), counters=self.counters.data_ptr(),
                              zero_foreign=1 if self.exchange == "sum" and self.dist is not None else 0,
                              write_background=1 if self.mine[0] == 0 else 0)
            B.exchange_tag = 256 * self._frame_no
            if peer is not None:
                B.n_peers = self.bricks.n - 1
                B.inbox, B.peer_inbox = peer[0], peer[1].data_ptr()

            def exchange():
                if self.dist is None:
                    return
                if peer is None:   # exactly one rank advanced each active ray
                    self.dist.all_reduce(state.view(torch.int64))
                else:
                    self._round_barrier(stream)
            L = _lib.lib()
            s = C.c_void_p(stream.cuda_stream)
            ev = []   # profile: (round, brick, start event, end event)
            queued = []   # profile: (round, brick, rays that brick marched: its PEER pushes)
            def mark():
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                return e
            fb.start.record(stream)
            _lib.check(L.tr_brick_trace(C.byref(dev0.desc), C.byref(ep.desc), C.byref(frame),
                                        C.byref(B), C.byref(out), s), "tr_brick_trace")
            rounds = 0
            if profile and not self.sync_rounds:
                ev.append((-1, -1, None, mark()))   # end of the trace
            if not self.sync_rounds:
                for _ in range(self.bricks.n):   # no host reads between these rounds
                    B.exchange_tag = 256 * self._frame_no + rounds
                    for b in self.mine:
                        B.rank = b
                        e0 = mark() if profile else None
                        _lib.check(L.tr_brick_round(C.byref(self.devs[b].desc), C.byref(ep.desc),
                                                    C.byref(frame), C.byref(B), C.byref(out), s),
                                   "tr_brick_round")
                        if profile:
                            ev.append((rounds, b, e0, mark()))
                            queued.append((rounds, b, int(self.counters[0].item())))
                    rounds += 1
                    exchange()
            while True:
                active = None
                if profile:
                    ev.append((-1, -1, None, mark()))   # end of the trace / previous round
                if rounds >= 255:
                    raise RuntimeError("brick frame did not finish in 255 rounds")
                B.exchange_tag = 256 * self._frame_no + rounds
                for b in self.mine:
                    B.rank = b
                    e0 = mark() if profile else None
                    _lib.check(L.tr_brick_round(C.byref(self.devs[b].desc), C.byref(ep.desc),
                                                C.byref(frame), C.byref(B), C.byref(out), s),
                               "tr_brick_round")
                    if profile:
                        ev.append((rounds, b, e0, mark()))
                        queued.append((rounds, b, int(self.counters[0].item())))
                    if active is None:
                        ctr = self.counters.cpu().numpy()
                        if ctr[2] & 1:
                            raise RuntimeError("a ray needs more intervals than the stored list")
                        active = int(ctr[1])
                        if peer is not None and rounds > 0:   # each rank planned only its own rays
                            t = self.counters[1:2].clone()
                            self.dist.all_reduce(t)
                            active = int(t.item())
                        if active == 0:
                            break
                if active == 0:
                    break
                rounds += 1
                exchange()
            fb.end.record(stream)
            if self.dist is not None:
                # every pixel and count was written by exactly one rank
                for t in (fb.rgba.view(torch.int64), fb.samples, fb.visited, fb.counters):
                    self.dist.all_reduce(t)
            rgba = fb.rgba[: w * h].cpu().numpy().reshape(h, w, 4)
            samples = fb.samples[: w * h].cpu().numpy().reshape(h, w)
            cnt = fb.counters.cpu().numpy()
            dev_ms = fb.start.elapsed_time(fb.end)
        self.rounds = rounds
        if profile:   # per-round per-brick device ms (the emulation runs them one after another)
            self.profile = {"frame_ms": float(dev_ms),
                            "trace_ms": float(fb.start.elapsed_time(ev[0][3])),
                            "runs": [(r, b, float(e0.elapsed_time(e1))) for r, b, e0, e1 in ev
                                     if e0 is not None],
                            "queued": queued}
        fbuf = Framebuffer(width=w, height=h, rgba=rgba, samples=samples,
                           background=np.asarray(sc.background, dtype=np.float64).copy())
        stats = RenderStats(
            total_samples=int(cnt[0]), wall_ms=float(dev_ms),
            partitions_visited_mean=float(np.float64(cnt[1]) / np.float64(w * h)),
            per_partition_samples=cnt[3:].copy() if track else None,
            samples=samples, device_ms=float(dev_ms), gpu_launches=1 + 2 * len(self.mine) * (rounds + 1))
        return fbuf, stats
