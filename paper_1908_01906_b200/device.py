"""Device-resident dataset, metadata epochs and frame launches.

Layout in HBM, all owned by torch tensors:
  tets       TrTetRecord[T]     128 B/tet  (inv 72 B | orig 24 B | field x4 32 B),
                                in point-BVH leaf order
  pnodes     TrPNode[]          64 B BVH2 nodes over padded tet boxes (f32, outward)
  pleaves    TrPLeaf[]          64 B: exclusive box (f32, inward) + id range + walk table
  pleaf_ids  uint32[]           ascending per leaf
  bnodes     TrBNode[]          112 B BVH2 nodes over partition boxes (f64)
  knodes     TrKNode[]          16 B BSP nodes over partition boxes (trace pass)
  pgrid      int32[]            uniform-grid leaf candidates
  scratch    per-ray interval lists of a ray chunk (IV_CAP x 16 B + 16 B per ray)
  epoch      one buffer per (active, sigma, tf) snapshot and (s1, s2, p):
             step f64[P] | (step, step/s1) f64[P,2] | tf f64[n,4] | active u8[P] | node activity u8[M]

The scene is uploaded once per (sampler, partition BVH) pair and cached;
transfer-function edits only create a new epoch (never touch geometry),
mirroring the reference's TF decoupling (transfer.py:144-167, A7).
"""

from __future__ import annotations

import contextlib
import ctypes as C
import math
import os
import sys
import threading
import time
import weakref
from collections import OrderedDict
from typing import Optional

import numpy as np

from . import _lib
from .mesh import BOX_PAD_REL

_CACHE_ATTR = "_b200_device_cache"
_LEAF_MAX = 8


def _torch():
    import torch
    return torch


def resolve_device(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 render path has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise RuntimeError(f"device {device} is not a CUDA device (no CPU fallback)")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return device


def _upload(arr: np.ndarray, device):
    """Host array -> new device byte tensor, synchronously, through the
    library's page-locked staging (tr_upload: a pageable copy of a fresh
    numpy array runs at a fraction of PCIe speed)."""
    torch = _torch()
    raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    t = torch.empty(raw.nbytes, dtype=torch.uint8, device=device)
    if raw.nbytes:
        stream = torch.cuda.current_stream(t.device)
        _lib.check(_lib.lib().tr_upload(C.c_void_p(t.data_ptr()), _lib.vptr(raw), raw.nbytes,
                                        C.c_void_p(stream.cuda_stream)), "tr_upload")
    return t


def _padded_boxes(scene) -> tuple[np.ndarray, np.ndarray]:
    """Tet boxes padded by 1e-7 * diag (mesh.py:248-250), native + OpenMP."""
    mesh = scene.mesh
    pad = BOX_PAD_REL * max(mesh.bounds.diagonal(), 1e-30)
    verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
    tets = np.ascontiguousarray(mesh.tets, dtype=np.int64)
    lo = np.empty((len(tets), 3))
    hi = np.empty((len(tets), 3))
    _lib.check(_lib.lib().tr_tet_boxes(len(tets), _lib.ptr(verts, C.c_double),
                                       _lib.ptr(tets, C.c_int64), pad, _lib.ptr(lo, C.c_double),
                                       _lib.ptr(hi, C.c_double)), "tr_tet_boxes")
    return lo, hi


class PointGrid:
    """Uniform-grid leaf index of the point BVH (tr_pbvh_grid)."""

    def __init__(self, dims, org, scale, cells):
        self.dims, self.org, self.scale, self.cells = dims, org, scale, cells


class CellLists:
    """tr_cells_build output: the exact point-location path for meshes whose
    leaves do not line up with the grid (unstructured tets)."""

    def __init__(self, dims, org, scale, off, recs, tbox):
        self.dims, self.org, self.scale = dims, org, scale
        self.off, self.recs, self.tbox = off, recs, tbox


CELL_COVERAGE_MIN = 0.9   # below this mean grid coverage the cell lists are built
CELL_REFINE = 2           # cell-list grid: the point grid refined 2x per axis
CELL_MAX_LIST = 96        # longer lists fall back to the BVH descent

POINT_BUILD_ENV = "TETRAY_POINT_BUILD"
POINT_BUILDS = ("device", "device-nowalk", "device-hostwalk", "host")


def point_build_mode(scene) -> str:
    """Where a general mesh's point-location structures are built:
    "device" (csrc/pbuild.cu: Morton LBVH, exclusive boxes, grid, cell lists
    and the leaf walk tables, all in HBM), "device-nowalk" (the same without
    walk tables), "device-hostwalk" (the device build with the host's
    long-double walk tables, tr_leaf_walk) or "host" (host_build.cpp).  From
    scene.point_build, else $TETRAY_POINT_BUILD, else "device"."""
    m = getattr(scene, "point_build", None) or os.environ.get(POINT_BUILD_ENV) or "device"
    if m not in POINT_BUILDS:
        raise ValueError(f"point_build must be one of {POINT_BUILDS}, not {m!r}")
    return m if scene.mesh.n_tets > _LEAF_MAX else "host"


def build_point_bvh(box_lo: np.ndarray, box_hi: np.ndarray, leaf_max: int = _LEAF_MAX,
                    cells=None):
    """(nodes, leaves, ids, grid, cell lists or None).  cells=None: build the
    cell lists when the grid's exclusive-box coverage is below
    CELL_COVERAGE_MIN."""
    L = _lib.lib()
    box_lo = np.ascontiguousarray(box_lo, dtype=np.float64)
    box_hi = np.ascontiguousarray(box_hi, dtype=np.float64)
    h = C.c_void_p()
    _lib.check(L.tr_pbvh_build(len(box_lo), _lib.ptr(box_lo, C.c_double),
                               _lib.ptr(box_hi, C.c_double), leaf_max, C.byref(h)), "tr_pbvh_build")
    try:
        sz = np.zeros(4, np.int64)
        _lib.check(L.tr_pbvh_sizes(h, _lib.ptr(sz, C.c_int64)), "tr_pbvh_sizes")
        nodes = np.zeros(int(sz[0]), dtype=_lib.PNODE_DTYPE)
        leaves = np.zeros(int(sz[1]), dtype=_lib.PLEAF_DTYPE)
        ids = np.zeros(int(sz[2]), dtype=np.uint32)
        _lib.check(L.tr_pbvh_copy(h, _lib.vptr(nodes), _lib.vptr(leaves), _lib.vptr(ids)),
                   "tr_pbvh_copy")
        grid = PointGrid(np.zeros(3, np.int32), np.zeros(3), np.zeros(3),
                         np.zeros(int(sz[3]), np.int32))
        _lib.check(L.tr_pbvh_grid(h, _lib.vptr(grid.dims), _lib.ptr(grid.org, C.c_double),
                                  _lib.ptr(grid.scale, C.c_double), _lib.vptr(grid.cells)),
                   "tr_pbvh_grid")
        grid.coverage = float(L.tr_pbvh_coverage(h))
        lists = None
        if cells or (cells is None and grid.coverage < CELL_COVERAGE_MIN):
            hc = C.c_void_p()
            _lib.check(L.tr_cells_build(h, _lib.ptr(box_lo, C.c_double), _lib.ptr(box_hi, C.c_double),
                                        CELL_REFINE, CELL_MAX_LIST, C.byref(hc)), "tr_cells_build")
            try:
                cs = np.zeros(3, np.int64)
                _lib.check(L.tr_cells_sizes(hc, _lib.ptr(cs, C.c_int64)), "tr_cells_sizes")
                lists = CellLists(np.zeros(3, np.int32), np.zeros(3), np.zeros(3),
                                  np.zeros(int(cs[0]) + 1, np.uint32),
                                  np.zeros(max(int(cs[1]), 1), np.uint32),
                                  np.zeros((int(cs[2]), 8), np.float32))
                _lib.check(L.tr_cells_copy(hc, _lib.vptr(lists.dims), _lib.ptr(lists.org, C.c_double),
                                           _lib.ptr(lists.scale, C.c_double), _lib.vptr(lists.off),
                                           _lib.vptr(lists.recs), _lib.vptr(lists.tbox)), "tr_cells_copy")
            finally:
                L.tr_host_free(hc)
    finally:
        L.tr_host_free(h)
    return nodes, leaves, ids, grid, lists


def build_partition_bsp(lo: np.ndarray, hi: np.ndarray):
    """Axis-aligned BSP over partition boxes (tr_kbsp_build): nodes, leaf pids, root box."""
    L = _lib.lib()
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    hi = np.ascontiguousarray(hi, dtype=np.float64)
    h = C.c_void_p()
    _lib.check(L.tr_kbsp_build(len(lo), _lib.ptr(lo, C.c_double), _lib.ptr(hi, C.c_double),
                               C.byref(h)), "tr_kbsp_build")
    try:
        sz = np.zeros(2, np.int64)
        _lib.check(L.tr_kbsp_sizes(h, _lib.ptr(sz, C.c_int64)), "tr_kbsp_sizes")
        nodes = np.zeros(int(sz[0]), dtype=_lib.KNODE_DTYPE)
        pids = np.zeros(int(sz[1]), dtype=np.int32)
        root = np.zeros(6)
        _lib.check(L.tr_kbsp_copy(h, _lib.vptr(nodes), _lib.vptr(pids), _lib.ptr(root, C.c_double)),
                   "tr_kbsp_copy")
    finally:
        L.tr_host_free(h)
    return nodes, pids, root


def pack_tet_records(mesh, sampler, order=None) -> np.ndarray:
    """128-B records; record k holds tet order[k] (None: tet k)."""
    order = None if order is None else np.ascontiguousarray(order, dtype=np.uint32)
    n = mesh.n_tets if order is None else len(order)
    rec = np.empty(n, dtype=_lib.TET_RECORD_DTYPE)
    orig = np.ascontiguousarray(sampler.tet_orig, dtype=np.float64)
    inv = np.ascontiguousarray(sampler.tet_inv, dtype=np.float64)
    tets = np.ascontiguousarray(mesh.tets, dtype=np.int64)
    fld = np.ascontiguousarray(mesh.field, dtype=np.float64)
    _lib.check(_lib.lib().tr_pack_tets(n, _lib.ptr(tets, C.c_int64),
                                       _lib.ptr(orig, C.c_double), _lib.ptr(inv, C.c_double),
                                       _lib.ptr(fld, C.c_double), int(mesh.centering),
                                       None if order is None else _lib.vptr(order),
                                       _lib.vptr(rec)), "tr_pack_tets")
    return rec


_POW_RESTATED = None   # the library restates glibc pow (tables found at build time)


def _steps_on_device(sigma: np.ndarray, p: float) -> bool:
    """True when every |min(sigma, 1) - 1| ** p lies on glibc pow's restated
    path (csrc/glibc_pow.cuh), so the device steps equal the host's bit for
    bit: x in {0 (p > 0), 1} or x a positive normal double with 2^-65 <= |p| <
    2^63 and |p ln x| well below the 512 exp-overflow bound."""
    global _POW_RESTATED
    if _POW_RESTATED is None:
        _POW_RESTATED = bool(_lib.lib().tr_pow_glibc_available())
    if not _POW_RESTATED or not math.isfinite(p):
        return False
    ap = abs(p)
    if not (2.0 ** -65 <= ap < 2.0 ** 63):
        return False
    lo = max(math.exp(-499.0 / ap), float(np.finfo(np.float64).tiny))
    hi = math.exp(499.0 / ap)
    if p > 0.0 and lo < 2.0 ** -54:
        # every sigma < 1 gives x = 1 - sigma >= 2^-53 > lo (Sterbenz), sigma >= 1
        # gives x = 0: only the far end can leave the domain
        return bool(sigma.min() >= 1.0 - hi)   # NaN fails
    x = np.abs(np.minimum(sigma, 1.0) - 1.0)
    if p <= 0.0 and not x.all():
        return False
    nz = x[x != 0.0]   # x == 1 is inside [lo, hi]
    if nz.size == 0:
        return True
    return bool(nz.min() >= lo) and bool(nz.max() <= hi)   # NaN fails both


class Epoch:
    """One uploaded (active, step, tf) snapshot."""

    def __init__(self, dev: "DeviceScene", meta_state, params, stream=None, hold: bool = True):
        """stream: the upload stream (default: the current one).  hold=False
        when the caller synchronizes `stream` before the epoch can be
        dropped (render()): the staging buffer needs no keep-alive record."""
        torch = _torch()
        active, sigma, tf = meta_state
        self.meta_state = meta_state  # pins the tuple so its id stays unique
        P = dev.n_parts
        act = np.ascontiguousarray(active, dtype=np.uint8).reshape(-1)
        sig = np.ascontiguousarray(sigma, dtype=np.float64).reshape(-1)
        if len(act) != P or len(sig) != P:
            raise ValueError(f"metadata epoch has {len(act)} partitions, scene has {P}")
        kact, bact = dev.activity(act)
        table = np.ascontiguousarray(tf.table, dtype=np.float64)
        self.n_tf = int(table.shape[0])
        self.tf_lo, self.tf_hi = float(tf.domain[0]), float(tf.domain[1])
        s1, s2, pw = float(params.s1), float(params.s2), float(params.p)
        # one pinned staging buffer + one device buffer; sections and upload
        # in C (tr_epoch_upload; layout in tr_epoch_bytes)
        L = _lib.lib()
        nbytes = int(L.tr_epoch_bytes(P, self.n_tf, dev.n_bnodes, dev.n_knodes))
        self.host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=dev.device)
        # step sizes (K:20-22) and exponents (K:27) on the device when every
        # |min(sigma, 1) - 1| ** p is on the restated glibc pow's path
        self._step_dev = _steps_on_device(sig, pw)
        self.desc = _lib.TrEpoch()
        self._keep = (sig, act, bact, kact, table)   # the arrays `up` points at
        self.up = _lib.TrEpochUpload(
            n_parts=P, sigma=sig.ctypes.data, active=act.ctypes.data,
            bnode_active=bact.ctypes.data, knode_active=kact.ctypes.data,
            n_bnodes=dev.n_bnodes, n_knodes=dev.n_knodes, tf_table=table.ctypes.data,
            n_tf=self.n_tf, tf_lo=self.tf_lo, tf_hi=self.tf_hi, s1=s1, s2=s2, p=pw,
            steps_on_device=1 if self._step_dev else 0, host_buf=self.host.data_ptr(),
            dev_buf=self.buf.data_ptr(), buf_bytes=nbytes)
        self._dev = dev
        self._P = P
        self.stale = False
        self._uploaded = torch.cuda.Event()   # recorded after each copy out of `host`
        self._recorded = False
        self.upload(stream, hold)

    def upload(self, stream=None, hold: bool = True) -> None:
        """Pack the epoch's host arrays into the page-locked staging buffer and
        copy them to the device (tr_epoch_upload_s); device steps recomputed.
        A re-upload (a stale epoch: a caller asked for the copy again) first
        waits for the previous copy out of the staging buffer."""
        torch = _torch()
        dev = self._dev
        if stream is None:
            stream = torch.cuda.current_stream(dev.device)
        if self._recorded:
            self._uploaded.synchronize()
        h2d = C.c_int64(0)
        _lib.check(_lib.lib().tr_epoch_upload_s(C.byref(self.up), C.byref(self.desc), C.byref(h2d),
                                                stream.cuda_stream), "tr_epoch_upload_s")
        self.h2d_bytes = int(h2d.value)
        self.stale = False
        if not self.up.packed:
            # device steps: the first frame reads back the epoch's inexact word
            self.verified = not self.desc.inexact
        # the staging block now holds the sections: a re-upload (stale) only
        # moves it (one kernel over PCIe with device steps)
        self.up.packed = 1
        self._uploaded.record(stream)
        self._recorded = True
        # the copy is not torch's: keep the staging buffer alive until it has run
        if hold:
            dev.hold_until_done(self.host, stream)

    @property
    def step_host(self) -> np.ndarray:
        """The epoch's per-partition steps (read back when the device made them)."""
        return self.buf[:8 * self._P].cpu().numpy().view(np.float64)


# render() lets the kernels write rgba / samples into the page-locked result
# arrays directly (TETRAY_B200_STAGED_OUTPUTS=1: device buffers + copies)
DIRECT_HOST_OUTPUTS = os.environ.get("TETRAY_B200_STAGED_OUTPUTS", "0") != "1"


_HOST_DEV: dict = {}   # page-locked block address -> device address (blocks are reused)


def host_device_pointer(t) -> int:
    """Device address of a page-locked (pin_memory) host tensor."""
    h = t.data_ptr()
    d = _HOST_DEV.get(h)
    if d is None:
        p = C.c_void_p()
        _lib.check(_lib.lib().tr_host_device_pointer(C.c_void_p(h), C.byref(p)),
                   "tr_host_device_pointer")
        d = _HOST_DEV[h] = int(p.value)
        if len(_HOST_DEV) > 4096:
            _HOST_DEV.clear()
    return d


# rays per trace/march chunk (interval-list scratch: ~1 KB per ray)
MAX_CHUNK_RAYS = 1 << 20


class FrameBuffers:
    """Device outputs of one frame shape, reused across frames."""

    def __init__(self, dev: "DeviceScene", width: int, height: int, compact_slots: int = 0):
        torch = _torch()
        d = dev.device
        n = compact_slots * 32 if compact_slots else width * height
        self.rgba = torch.empty((n, 4), dtype=torch.float64, device=d)
        self.samples = torch.empty(n, dtype=torch.int64, device=d)
        self.visited = torch.empty(n, dtype=torch.int32, device=d)
        # [totals(2) | work(1) | ppart(P)] zeroed with one fill per frame
        self.counters = torch.empty(3 + dev.n_parts, dtype=torch.int64, device=d)
        # interval lists of one ray chunk (<= 1M rays; larger frames run in chunks)
        rays = ((n + 31) // 32) * 32
        self.scratch_bytes = int(_lib.lib().tr_scratch_bytes(min(rays, MAX_CHUNK_RAYS)))
        self.scratch = torch.empty(self.scratch_bytes, dtype=torch.uint8, device=d)
        self.start = torch.cuda.Event(enable_timing=True)
        self.end = torch.cuda.Event(enable_timing=True)

    def outputs(self) -> _lib.TrOutputs:
        c = self.counters.data_ptr()
        return _lib.TrOutputs(rgba=self.rgba.data_ptr(), samples=self.samples.data_ptr(),
                              visited=self.visited.data_ptr(), ppart=c + 24, totals=c,
                              work=c + 16, scratch=self.scratch.data_ptr(),
                              scratch_bytes=self.scratch_bytes)


class DeviceScene:
    """The scene's geometry in HBM plus its epoch and output caches."""

    def __init__(self, scene, device, tet_subset: Optional[np.ndarray] = None):
        """tet_subset: ascending global tet ids this device holds (a brick of
        a record-sharded frame, bricks.py); None = every tet."""
        torch = _torch()
        self.device = device
        self.lock = threading.Lock()
        self.tet_subset = None if tet_subset is None else np.ascontiguousarray(tet_subset, np.int64)
        mesh = scene.mesh
        with torch.cuda.device(device):
            t0 = time.perf_counter()
            part_lo = np.ascontiguousarray(scene.bvh.box_lo, dtype=np.float64)
            part_hi = np.ascontiguousarray(scene.bvh.box_hi, dtype=np.float64)
            bnodes = getattr(scene.bvh, "nodes", None)
            if not (isinstance(bnodes, np.ndarray) and bnodes.dtype == _lib.BNODE_DTYPE):
                from .traversal import build_bvh_over_boxes
                bnodes = build_bvh_over_boxes(part_lo, part_hi)
            knodes, kpids, kroot = build_partition_bsp(part_lo, part_hi)
            self.knodes_host, self.kpids_host = knodes, kpids
            self.n_knodes = int(len(knodes))
            self.bnodes_host = np.ascontiguousarray(bnodes)
            self.n_parts = int(part_lo.shape[0])
            self.n_bnodes = int(len(bnodes))
            self.n_tets = int(mesh.n_tets if self.tet_subset is None else len(self.tet_subset))
            if getattr(mesh, "device_generated", False):
                point = self._point_structures_grid(scene)
            elif point_build_mode(scene) != "host" and self.tet_subset is None:
                point = self._point_structures_device(scene, point_build_mode(scene) == "device")
                if point_build_mode(scene) == "device-hostwalk":
                    tw = time.perf_counter()
                    self._attach_walk_tables(scene)
                    self.build_phases["walk_s"] = time.perf_counter() - tw
            else:
                point = self._point_structures_host(scene)
            self.build_s = time.perf_counter() - t0
            self.t_bnodes = _upload(bnodes, device)
            self.t_plo = _upload(part_lo, device)
            self.t_phi = _upload(part_hi, device)
            self.t_knodes = _upload(knodes, device)
            self.t_kpids = _upload(kpids, device)
            torch.cuda.synchronize(device)
        grid = self.grid
        self.resident_bytes = sum(t.numel() for t in (self.t_tets, self.t_pnodes, self.t_pleaves,
                                                      self.t_pids, self.t_bnodes, self.t_plo,
                                                      self.t_phi, self.t_grid, self.t_grid_leaf,
                                                      self.t_grid_pred,
                                                      self.t_knodes, self.t_kpids)
                                  if t is not None)
        ptr = lambda t: 0 if t is None else t.data_ptr()
        self.desc = _lib.TrDeviceScene(
            tets=ptr(self.t_tets), pnodes=ptr(self.t_pnodes),
            pleaves=ptr(self.t_pleaves), pleaf_ids=ptr(self.t_pids),
            n_tets=self.n_tets, n_pnodes=point[0], n_pleaves=point[1],
            centering=int(mesh.centering), bnodes=self.t_bnodes.data_ptr(),
            part_lo=self.t_plo.data_ptr(), part_hi=self.t_phi.data_ptr(), n_parts=self.n_parts,
            n_bnodes=self.n_bnodes,
            mesh_lo=(C.c_double * 3)(*mesh.bounds.lo), mesh_hi=(C.c_double * 3)(*mesh.bounds.hi),
            pgrid=ptr(self.t_grid),
            pgrid_leaf=ptr(self.t_grid_leaf) if self.t_grid_leaf is not None else ptr(self.t_pleaves),
            gdim=(C.c_int32 * 3)(*grid.dims),
            gorg=(C.c_double * 3)(*grid.org), gscale=(C.c_double * 3)(*grid.scale),
            knodes=self.t_knodes.data_ptr(), kleaf_pids=self.t_kpids.data_ptr(),
            n_knodes=self.n_knodes, kroot=(C.c_double * 6)(*kroot))
        if self.t_grid_pred is not None:
            self.desc.pgrid_pred = self.t_grid_pred.data_ptr()
        elif getattr(self, "grid_pred_class", None) is not None:
            self.desc.pred_classes = 2
            self.desc.pred_class = (C.c_float * 24)(*self.grid_pred_class)
            # the march derives leaves and records from the cube layout
            self.desc.grid_n, self.desc.grid_pad, self.desc.grid_brick = self.grid_analytic
            self.desc.class_walk = self.t_class_walk.data_ptr()
        if self.cells is not None:
            cl = self.cells
            self.desc.cell_off = self.t_coff.data_ptr()
            self.desc.cell_recs = self.t_crecs.data_ptr()
            self.desc.tbox = self.t_tbox.data_ptr()
            self.desc.cdim = (C.c_int32 * 3)(*cl.dims)
            self.desc.corg = (C.c_double * 3)(*cl.org)
            self.desc.cscale = (C.c_double * 3)(*cl.scale)
            # the exclusive-leaf grid proves < half of the points: go to the lists first
            self.desc.cells_first = 1 if getattr(self.grid, "coverage", 1.0) < 0.5 else 0
            self.resident_bytes += sum(t.numel() for t in (self.t_coff, self.t_crecs, self.t_tbox))
        self._epochs: OrderedDict = OrderedDict()
        self._frames: dict = {}
        self._results = _ResultPool()
        self._act_key, self._act_val = None, None
        self._desc_key, self._desc_val = None, None

    def _point_structures_host(self, scene):
        """Host builders (csrc/host_build.cpp) + upload: records in point-BVH
        leaf order, BVH nodes, leaves, leaf ids and the grid with one copy of
        its candidate leaf header per cell."""
        device = self.device
        mesh, sampler = scene.mesh, scene.sampler
        lo, hi = _padded_boxes(scene)
        sub = self.tet_subset
        if sub is not None:   # ascending global ids: local order = id order
            if len(sub) == 0:
                raise ValueError("empty tet subset")
            lo, hi = lo[sub], hi[sub]
        pnodes, pleaves, pids, grid, lists = build_point_bvh(lo, hi,
                                                             cells=getattr(scene, "cell_lists", None))
        del lo, hi
        if sub is not None:
            pids = sub[pids].astype(np.uint32)   # leaf ids as global tet ids
            m = pnodes["minid"]                  # subtree minima too (descent pruning)
            ok = m < len(sub)
            m[ok] = sub[m[ok]].astype(np.uint32)
        # leaf walk tables (tr_leaf_walk): face neighbours + certificates
        verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        tets = np.ascontiguousarray(mesh.tets, dtype=np.int64)
        pred = np.zeros((len(pleaves), 12), np.float32)   # TrLeafPred per leaf
        _lib.check(_lib.lib().tr_leaf_walk(len(pleaves), _lib.vptr(pleaves), _lib.vptr(pids),
                                           _lib.vptr(verts), _lib.vptr(tets), _lib.vptr(pred)),
                   "tr_leaf_walk")
        # records in LEAF order (record k = tet pleaf_ids[k]): a leaf scan
        # reads consecutive 128-B lines with no id indirection
        rec = pack_tet_records(mesh, sampler, order=pids)
        self.pnodes_host, self.pleaves_host = pnodes, pleaves
        self.t_tets = _upload(rec, device)
        del rec
        self.t_pnodes = _upload(pnodes, device)
        self.t_pleaves = _upload(pleaves, device)
        self.t_pids = _upload(pids, device)
        self.t_grid = _upload(grid.cells, device)
        cell_leaf = np.zeros(len(grid.cells), dtype=_lib.PLEAF_DTYPE)
        cell_leaf["ex_lo"] = 1.0   # empty box: no candidate
        cell_leaf["ex_hi"] = 0.0
        has = grid.cells >= 0
        cell_leaf[has] = pleaves[grid.cells[has]]
        self.t_grid_leaf = _upload(cell_leaf, device)
        cell_pred = np.zeros((len(grid.cells), 12), np.float32)
        cell_pred[has] = pred[grid.cells[has]]
        self.t_grid_pred = _upload(cell_pred, device)
        self.grid = grid
        self.cells = lists
        if lists is not None:
            self.t_coff = _upload(lists.off, device)
            self.t_crecs = _upload(lists.recs, device)
            self.t_tbox = _upload(lists.tbox, device)
        return len(pnodes), len(pleaves)

    def _point_structures_device(self, scene, walk: bool = True):
        """The same structures built in HBM (csrc/pbuild.cu):
        mesh arrays uploaded once through page-locked staging, then Morton
        LBVH, exclusive boxes, leaf grid, cell lists and the records in leaf
        order on the device.  No walk tables (leaves scanned in id order)."""
        torch = _torch()
        device = self.device
        L = _lib.lib()
        mesh, sampler = scene.mesh, scene.sampler
        stream = torch.cuda.current_stream(device)
        sp = C.c_void_p(stream.cuda_stream)

        def up(arr, dtype):
            a = np.ascontiguousarray(arr, dtype=dtype)
            t = torch.empty(a.nbytes, dtype=torch.uint8, device=device)
            _lib.check(L.tr_upload(C.c_void_p(t.data_ptr()), _lib.vptr(a), a.nbytes, sp), "tr_upload")
            return t

        t0 = time.perf_counter()
        t_verts, t_tets = up(mesh.vertices, np.float64), up(mesh.tets, np.int64)
        t_up = time.perf_counter() - t0
        pad = BOX_PAD_REL * max(mesh.bounds.diagonal(), 1e-30)
        cells = getattr(scene, "cell_lists", None)
        below = CELL_COVERAGE_MIN if cells is None else (2.0 if cells else -1.0)
        h = C.c_void_p()
        tb = time.perf_counter()
        _lib.check(L.tr_pbvh_build_device(len(mesh.vertices), C.c_void_p(t_verts.data_ptr()), mesh.n_tets,
                                          C.c_void_p(t_tets.data_ptr()), pad, _LEAF_MAX, below,
                                          CELL_REFINE, CELL_MAX_LIST, sp, C.byref(h)),
                   "tr_pbvh_build_device")
        t_call = time.perf_counter() - tb
        try:
            if walk:   # walk tables + predictors on the device
                _lib.check(L.tr_dpb_walk(h, C.c_void_p(t_verts.data_ptr()), C.c_void_p(t_tets.data_ptr()),
                                         sp), "tr_dpb_walk")
            sz = np.zeros(6, np.int64)
            _lib.check(L.tr_dpb_sizes(h, _lib.ptr(sz, C.c_int64)), "tr_dpb_sizes")
            n_nodes, n_leaves, n_ids, n_grid, n_cc, n_cr = (int(x) for x in sz)
            grid = PointGrid(np.zeros(3, np.int32), np.zeros(3), np.zeros(3), None)
            cdim, corg, cscale, cov = np.zeros(3, np.int32), np.zeros(3), np.zeros(3), np.zeros(1)
            _lib.check(L.tr_dpb_grid(h, _lib.vptr(grid.dims), _lib.ptr(grid.org, C.c_double),
                                     _lib.ptr(grid.scale, C.c_double), _lib.ptr(cov, C.c_double),
                                     _lib.vptr(cdim), _lib.ptr(corg, C.c_double),
                                     _lib.ptr(cscale, C.c_double)), "tr_dpb_grid")
            grid.coverage = float(cov[0])
            u8 = lambda n: torch.empty(max(int(n), 1), dtype=torch.uint8, device=device)
            self.t_pnodes = u8(n_nodes * _lib.PNODE_DTYPE.itemsize)
            self.t_pleaves = u8(n_leaves * _lib.PLEAF_DTYPE.itemsize)
            self.t_pids = u8(n_ids * 4)
            self.t_grid = u8(n_grid * 4)
            self.t_grid_leaf = u8(n_grid * _lib.PLEAF_DTYPE.itemsize)
            self.t_grid_pred = u8(n_grid * 48) if walk else None   # TrLeafPred per cell
            lists = None
            if n_cc:
                lists = CellLists(cdim, corg, cscale, None, None, None)
                self.t_coff = u8((n_cc + 1) * 4)
                self.t_crecs = u8(n_cr * 4)
                self.t_tbox = u8(n_ids * 32)
            dp = lambda t: C.c_void_p(t.data_ptr())
            _lib.check(L.tr_dpb_copy(h, dp(self.t_pnodes), dp(self.t_pleaves), dp(self.t_pids),
                                     dp(self.t_grid), dp(self.t_grid_leaf),
                                     dp(self.t_grid_pred) if walk else None,
                                     dp(self.t_coff) if lists else None,
                                     dp(self.t_crecs) if lists else None,
                                     dp(self.t_tbox) if lists else None, sp), "tr_dpb_copy")
        finally:
            tf = time.perf_counter()
            L.tr_dpb_free(h)
            t_free = time.perf_counter() - tf
        t_build = time.perf_counter() - tb
        del t_verts
        # records in leaf order, packed on the device
        t1, t_up0 = time.perf_counter(), t_up
        t_orig = up(sampler.tet_orig, np.float64)
        t_inv = up(sampler.tet_inv, np.float64)
        t_field = up(mesh.field, np.float64)
        t_up += time.perf_counter() - t1
        self.t_tets = u8(n_ids * _lib.TET_RECORD_DTYPE.itemsize)
        _lib.check(L.tr_pack_tets_device(n_ids, dp(t_tets), dp(t_orig), dp(t_inv), dp(t_field),
                                         int(mesh.centering), dp(self.t_pids), dp(self.t_tets), sp),
                   "tr_pack_tets_device")
        stream.synchronize()
        self.build_phases = {"upload_s": t_up, "lbvh_s": t_build, "lbvh_call_s": t_call,
                             "lbvh_free_s": t_free,
                             "pack_s": time.perf_counter() - t1 - (t_up - t_up0)}
        del t_tets, t_orig, t_inv, t_field
        self.pnodes_host = self.pleaves_host = None
        self.grid = grid
        self.cells = lists
        self.upload_s = t_up
        return n_nodes, n_leaves

    def _attach_walk_tables(self, scene):
        """tr_leaf_walk (host, long-double certificates) over the device-built
        leaves: walk tables into the leaf headers and the per-cell copies,
        walk-start predictors per grid cell (as _point_structures_host)."""
        mesh = scene.mesh
        pleaves = self.t_pleaves.cpu().numpy().view(_lib.PLEAF_DTYPE).copy()
        pids = np.ascontiguousarray(self.t_pids.cpu().numpy().view(np.uint32))
        verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        tets = np.ascontiguousarray(mesh.tets, dtype=np.int64)
        pred = np.zeros((len(pleaves), 12), np.float32)
        _lib.check(_lib.lib().tr_leaf_walk(len(pleaves), _lib.vptr(pleaves), _lib.vptr(pids),
                                           _lib.vptr(verts), _lib.vptr(tets), _lib.vptr(pred)),
                   "tr_leaf_walk")
        cells = self.t_grid.cpu().numpy().view(np.int32)
        has = cells >= 0
        cell_leaf = np.zeros(len(cells), dtype=_lib.PLEAF_DTYPE)
        cell_leaf["ex_lo"] = 1.0
        cell_leaf["ex_hi"] = 0.0
        cell_leaf[has] = pleaves[cells[has]]
        cell_pred = np.zeros((len(cells), 12), np.float32)
        cell_pred[has] = pred[cells[has]]
        self.t_pleaves = _upload(pleaves, self.device)
        self.t_grid_leaf = _upload(cell_leaf, self.device)
        self.t_grid_pred = _upload(cell_pred, self.device)

    def _point_structures_grid(self, scene):
        """Synthetic cube-grid scene generated in HBM (tr_grid_scene_build,
        csrc/synth.cu): records in id order, one leaf per cube, the cube grid
        as the point grid (its leaf array doubles as the cell headers)."""
        torch = _torch()
        mesh, sampler = scene.mesh, scene.sampler
        n = int(mesh.n)
        sz = np.zeros(3, np.int64)
        L = _lib.lib()
        _lib.check(L.tr_grid_scene_sizes(n, _lib.ptr(sz[0:1], C.c_int64), _lib.ptr(sz[1:2], C.c_int64),
                                         _lib.ptr(sz[2:3], C.c_int64)), "tr_grid_scene_sizes")
        n_tets, n_leaves, n_nodes = (int(v) for v in sz)
        self.t_tets = torch.empty(n_tets * 128, dtype=torch.uint8, device=self.device)
        self.t_pleaves = torch.empty(n_leaves * _lib.PLEAF_DTYPE.itemsize, dtype=torch.uint8,
                                     device=self.device)
        self.t_pnodes = torch.empty(n_nodes * 64, dtype=torch.uint8, device=self.device)
        inv10 = np.ascontiguousarray(sampler.inv10, dtype=np.float64).reshape(90)
        stream = torch.cuda.current_stream(self.device)
        # brick-ordered records (+ their tet ids) unless GRID_ID_ORDER is asked for
        brick = not getattr(scene, "grid_id_order", False)
        self.t_pids = (torch.empty(n_tets, dtype=torch.int32, device=self.device)
                       if brick else None)
        _lib.check(L.tr_grid_scene_build(n, int(mesh.field_id), float(sampler.pad),
                                         _lib.ptr(inv10, C.c_double), self.t_tets.data_ptr(),
                                         self.t_pleaves.data_ptr(), self.t_pnodes.data_ptr(),
                                         None if self.t_pids is None else self.t_pids.data_ptr(),
                                         C.c_void_p(stream.cuda_stream)), "tr_grid_scene_build")
        torch.cuda.synchronize(self.device)
        self.t_grid = None
        self.t_grid_leaf = None
        self.t_grid_pred = None
        self.grid_pred_class = np.zeros(24, np.float32)   # TrLeafPred of an even / odd cube
        walk16 = np.zeros(16, np.uint32)                   # their TrPLeaf.walk tables
        _lib.check(L.tr_grid_walk_pred(float(sampler.pad), _lib.vptr(self.grid_pred_class),
                                       _lib.vptr(walk16)), "tr_grid_walk_pred")
        self.t_class_walk = _upload(walk16, self.device)
        self.grid_analytic = (n, float(sampler.pad), 1 if brick else 0)
        self.cells = None
        self.pnodes_host = self.pleaves_host = None
        self.grid = PointGrid(np.full(3, n, np.int32), np.zeros(3), np.ones(3), None)
        return n_nodes, n_leaves

    # ---------------------------------------------------------------- epochs
    def activity(self, act: np.ndarray):
        """Subtree-activity bits of both partition trees for an active mask
        (reused while the mask is unchanged, e.g. across colour-only TF edits)."""
        key = act.tobytes()
        if self._act_key == key:
            return self._act_val
        kact = np.empty(self.n_knodes, dtype=np.uint8)
        _lib.check(_lib.lib().tr_knodes_activity(self.n_knodes, _lib.vptr(self.knodes_host),
                                                 _lib.vptr(self.kpids_host), _lib.ptr(act, C.c_uint8),
                                                 _lib.ptr(kact, C.c_uint8)), "tr_knodes_activity")
        bact = np.empty(self.n_bnodes, dtype=np.uint8)
        _lib.check(_lib.lib().tr_bnodes_activity(self.n_bnodes, _lib.vptr(self.bnodes_host),
                                                 _lib.ptr(act, C.c_uint8), _lib.ptr(bact, C.c_uint8)),
                   "tr_bnodes_activity")
        self._act_key, self._act_val = key, (kact, bact)
        return kact, bact

    def epoch(self, meta_state, params, stream=None, hold: bool = True,
              defer_stale: bool = False) -> Epoch:
        """The cached epoch of meta_state (uploaded on first use).  A stale
        cached epoch is copied again here, or -- defer_stale -- left stale for
        the caller to re-upload inside its frame call (render())."""
        key = (id(meta_state), float(params.s1), float(params.s2), float(params.p))
        ep = self._epochs.get(key)
        if ep is None or ep.meta_state is not meta_state:
            ep = Epoch(self, meta_state, params, stream, hold)
            self._epochs[key] = ep
            while len(self._epochs) > 8:
                self._epochs.popitem(last=False)
        else:
            if ep.stale and not defer_stale:
                ep.upload(stream, hold)
            self._epochs.move_to_end(key)
        return ep

    def mark_epochs_stale(self) -> None:
        """The next frame of each cached epoch copies it to the device again
        (bench.py's end-to-end steps: every step's inputs cross PCIe)."""
        for ep in self._epochs.values():
            ep.stale = True

    def hold_until_done(self, obj, stream) -> None:
        """Keep `obj` (e.g. a pinned staging buffer read by an async copy
        torch does not track) referenced until `stream` passes this point."""
        torch = _torch()
        q = self.__dict__.setdefault("_inflight", [])
        while q and q[0][0].query():
            q.pop(0)
        ev = torch.cuda.Event()
        ev.record(stream)
        q.append((ev, obj))

    def frame_buffers(self, width: int, height: int, compact_slots: int = 0) -> FrameBuffers:
        key = (width, height, compact_slots)
        fb = self._frames.get(key)
        if fb is None:
            fb = self._frames[key] = FrameBuffers(self, width, height, compact_slots)
        return fb

    # ---------------------------------------------------------------- frames
    def frame_desc(self, scene, camera, mode: int, params, jitter: bool, track: bool,
                   flags: int = 0, shard_rank: int = 0, shard_count: int = 1,
                   compact: bool = False) -> _lib.TrFrame:
        key = (camera.position.tobytes(), camera.look_at.tobytes(), camera.up.tobytes(),
               float(camera.fov_y_deg), int(camera.width), int(camera.height), mode,
               float(params.s1), float(params.termination_opacity),
               float(scene.traversal_config.epsilon), np.asarray(scene.background).tobytes(),
               bool(jitter), bool(track), flags, shard_rank, shard_count, bool(compact))
        if key == self._desc_key:
            return self._desc_val
        desc = self._frame_desc(scene, camera, mode, params, jitter, track, flags, shard_rank,
                                shard_count, compact)
        self._desc_key, self._desc_val = key, desc
        return desc

    def _frame_desc(self, scene, camera, mode, params, jitter, track, flags, shard_rank,
                    shard_count, compact) -> _lib.TrFrame:
        right, up, fwd = camera.basis()
        w, h = int(camera.width), int(camera.height)
        bg = np.asarray(scene.background, dtype=np.float64).reshape(4)
        D3 = C.c_double * 3
        return _lib.TrFrame(
            cam_pos=D3(*camera.position), cam_right=D3(*right), cam_up=D3(*up), cam_fwd=D3(*fwd),
            tan_half=math.tan(math.radians(camera.fov_y_deg) / 2.0), aspect=w / h,
            width=w, height=h, jitter=1 if jitter else 0, mode=mode, s1=float(params.s1),
            term=float(params.termination_opacity),
            eps=float(scene.traversal_config.epsilon), bg=(C.c_double * 4)(*bg),
            track_ppart=1 if track else 0, shard_rank=shard_rank, shard_count=shard_count,
            compact=1 if compact else 0, flags=flags)

    def launch(self, frame: _lib.TrFrame, epoch: Epoch, fb: FrameBuffers, stream,
               out: Optional[_lib.TrOutputs] = None) -> None:
        _lib.check(_lib.lib().tr_memset_async(fb.counters.data_ptr(), 0, 8 * fb.counters.numel(),
                                              stream.cuda_stream), "tr_memset_async")
        if out is None:
            out = fb.outputs()
        fb.start.record(stream)
        _lib.check(_lib.lib().tr_render_frame(C.byref(self.desc), C.byref(epoch.desc),
                                              C.byref(frame), C.byref(out),
                                              C.c_void_p(stream.cuda_stream)), "tr_render_frame")
        fb.end.record(stream)

    def render(self, scene, camera, mode: int, params, *, jitter: bool, track: bool,
               flags: int = 0):
        from .render import Framebuffer, RenderStats
        torch = _torch()
        w, h = int(camera.width), int(camera.height)
        idx = self.device.index
        ctx = (contextlib.nullcontext() if torch.cuda.current_device() == idx
               else torch.cuda.device(self.device))
        with self.lock, ctx:
            t0 = time.perf_counter()
            raw_stream = torch._C._cuda_getCurrentRawStream(idx)
            ep = self.epoch(scene.meta_state(), params, None, hold=False, defer_stale=True)
            frame = self.frame_desc(scene, camera, mode, params, jitter, track, flags)
            fb = self.frame_buffers(w, h)
            # one page-locked block: rgba | samples | counters (+ inexact word)
            npx = h * w
            base, dptr = self._results.take(8 * (5 * npx + 4 + self.n_parts))
            rgba_h = base[:32 * npx].view(np.float64).reshape(h, w, 4)
            samp_h = base[32 * npx:40 * npx].view(np.int64).reshape(h, w)
            cnt_h = base[40 * npx:].view(np.int64)
            if ep._recorded:
                ep._uploaded.synchronize()   # a staging-buffer copy of its own upload()
                ep._recorded = False
            out = fb.outputs()
            if DIRECT_HOST_OUTPUTS:
                # the kernels store each finished pixel straight into the
                # page-locked result arrays, overlapping the device->host
                # transfer with the march (tr_host_device_pointer)
                out.rgba = dptr
                out.samples = dptr + 32 * npx
            inexact = None
            if not ep.verified:
                cnt_h[-1] = 0
                inexact = cnt_h.ctypes.data + 8 * (3 + self.n_parts)
            dms = C.c_float(0.0)
            reup = C.byref(ep.up) if ep.stale else None
            # (stale epoch re-upload,) counters reset, the frame, counters (+ inexact
            # word) D2H, sync: one call
            _lib.check(_lib.lib().tr_render_sync(C.byref(self.desc), C.byref(ep.desc),
                                                 C.byref(frame), C.byref(out),
                                                 3 + self.n_parts, cnt_h.ctypes.data, inexact,
                                                 raw_stream, C.byref(dms), reup),
                       "tr_render_sync")
            ep.stale = False
            if not DIRECT_HOST_OUTPUTS:
                torch.from_numpy(rgba_h).view(-1, 4).copy_(fb.rgba)
                torch.from_numpy(samp_h).view(-1).copy_(fb.samples)
            if not ep.verified:
                if int(cnt_h[-1]) != 0:
                    raise RuntimeError("device step sizes of this epoch are inexact (sigma outside "
                                       "the restated glibc pow domain); frame discarded")
                ep.verified = True
            wall_ms = (time.perf_counter() - t0) * 1000.0
        fbuf = Framebuffer(width=w, height=h, rgba=rgba_h, samples=samp_h,
                           background=np.asarray(scene.background, dtype=np.float64).copy())
        stats = RenderStats(
            total_samples=int(cnt_h[0]), wall_ms=wall_ms,
            partitions_visited_mean=float(np.float64(cnt_h[1]) / np.float64(w * h)),
            per_partition_samples=cnt_h[3:3 + self.n_parts].copy() if track else None,
            samples=samp_h, device_ms=float(dms.value), gpu_launches=last_launches())
        return fbuf, stats


class _ResultPool:
    """Page-locked result blocks for render(): a block is handed out again
    once no array returned from it is alive (the returned arrays are numpy
    views of the block's base array, so its reference count says when)."""

    KEEP = 4

    def __init__(self):
        self.blocks = []   # [nbytes, tensor, base ndarray, device address]

    def take(self, nbytes: int):
        for b in self.blocks:
            if b[0] == nbytes and sys.getrefcount(b[2]) == 2:   # the list + the argument
                return b[2], b[3]
        torch = _torch()
        t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        blk = [nbytes, t, t.numpy(), host_device_pointer(t)]
        self.blocks.append(blk)
        if len(self.blocks) > self.KEEP:   # a busy block leaves with its last view
            for k, b in enumerate(self.blocks):
                if b is not blk and sys.getrefcount(b[2]) > 2:
                    del self.blocks[k]
                    break
            else:
                del self.blocks[0]
        return blk[2], blk[3]

_LAST_LAUNCH = (C.c_int64 * 3)()


def last_launches() -> int:
    """Kernels of ours the last tr_render_frame launched (tr_last_launch)."""
    _lib.check(_lib.lib().tr_last_launch(_LAST_LAUNCH), "tr_last_launch")
    return int(_LAST_LAUNCH[0])


def device_scene_for(scene, device=None) -> DeviceScene:
    """Cached DeviceScene of `scene` (rebuilt if its sampler or BVH changed)."""
    if device is None:   # the common case, without building a torch.device
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 render path has no CPU fallback")
        idx = torch.cuda.current_device()
    else:
        idx = resolve_device(device).index
    cache = getattr(scene, _CACHE_ATTR, None)
    if cache is None:
        cache = {}
        try:
            object.__setattr__(scene, _CACHE_ATTR, cache)
        except AttributeError:
            cache = _GLOBAL_CACHE.setdefault(id(scene), {})
    key = (idx, id(scene.sampler), id(scene.bvh))
    ent = cache.get(key)
    if ent is None or ent[0]() is not scene.sampler or ent[1]() is not scene.bvh:
        for k in [k for k in cache if k[0] == idx]:
            del cache[k]
        dev = DeviceScene(scene, _torch().device("cuda", idx))
        cache[key] = (weakref.ref(scene.sampler), weakref.ref(scene.bvh), dev)
        return dev
    return ent[2]


_GLOBAL_CACHE: dict = {}


class _SamplerScene:
    """Adapter so a bare MeshSampler can be made device-resident for point
    queries (no partitions needed: a single dummy partition)."""

    def __init__(self, sampler):
        from .traversal import PartitionBVH, build_bvh_over_boxes
        self.sampler = sampler
        self.mesh = sampler.mesh
        lo = sampler.mesh.bounds.lo.reshape(1, 3).copy()
        hi = sampler.mesh.bounds.hi.reshape(1, 3).copy()
        self.bvh = PartitionBVH(box_lo=lo, box_hi=hi, nodes=build_bvh_over_boxes(lo, hi))


def sample_points(sampler, points, device=None):
    """Batched point query on the GPU: (found u8->bool, value f64, tet id i64)."""
    torch = _torch()
    device = resolve_device(device)
    holder = sampler._device if hasattr(sampler, "_device") else {}
    dev = holder.get(str(device))
    if dev is None:
        dev = DeviceScene(_SamplerScene(sampler), device)
        if hasattr(sampler, "_device"):
            sampler._device[str(device)] = dev
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    n = len(pts)
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream(device)
        p_d = torch.from_numpy(pts).to(device, non_blocking=False)
        found = torch.empty(n, dtype=torch.uint8, device=device)
        vals = torch.empty(n, dtype=torch.float64, device=device)
        tet = torch.empty(n, dtype=torch.int64, device=device)
        _lib.check(_lib.lib().tr_field_at_many(C.byref(dev.desc), n, C.c_void_p(p_d.data_ptr()),
                                               C.c_void_p(found.data_ptr()),
                                               C.c_void_p(vals.data_ptr()),
                                               C.c_void_p(tet.data_ptr()),
                                               C.c_void_p(stream.cuda_stream)), "tr_field_at_many")
        out = (found.cpu().numpy().astype(bool), vals.cpu().numpy(), tet.cpu().numpy())
    return out
