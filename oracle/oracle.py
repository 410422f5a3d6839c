"""ctypes front end of the C parity oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product
package.  It renders a Scene (this repo's or tetray's, duck-typed) exactly the
way the reference's numba kernel does (pkg/src/tetray/_kernels.py:312-398),
from the reference-layout arrays: a median-split flat BVH over the padded tet
boxes (leaf 8, mesh.py:248-250) and one over the partition boxes (leaf 4,
traversal.py:89), both built by the C restatement of bvh.py:41-98.

Pinned against fixtures produced by running the reference itself
(tests/golden/make_golden.py -> tests/golden/*.json, tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes as C
import math
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)

_lib = None

_MODE_IDS = {"reference": 0, "skip": 1, "skip-adaptive": 2}


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            import subprocess
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        L = C.CDLL(str(LIB_PATH))
        L.orc_build_bvh.restype = C.c_int64
        L.orc_build_bvh.argtypes = [C.c_int64, f64p, f64p, C.c_int64, f64p, f64p, i64p, i64p,
                                    i64p, i64p, i64p]
        L.orc_step_size.restype = C.c_double
        L.orc_step_size.argtypes = [C.c_double] * 4
        L.orc_opacity_correction.restype = C.c_double
        L.orc_opacity_correction.argtypes = [C.c_double] * 3
        L.orc_tf_sample.restype = None
        L.orc_tf_sample.argtypes = [f64p, C.c_long, C.c_double, C.c_double, C.c_double, f64p]
        L.orc_build_bvh_fast.restype = C.c_int64
        L.orc_build_bvh_fast.argtypes = L.orc_build_bvh.argtypes
        L.orc_hash01.restype = C.c_double
        L.orc_hash01.argtypes = [C.c_int64, C.c_int64]
        mesh_args = [f64p, f64p, i64p, i64p, i64p, i64p, i64p, i64p, f64p, f64p, f64p, C.c_int64]
        part_args = [f64p, f64p, i64p, i64p, i64p, i64p, i64p, f64p, f64p, u8p]
        L.orc_field_at_many.restype = None
        L.orc_field_at_many.argtypes = [C.c_int64, f64p, *mesh_args, u8p, f64p, i64p, C.c_int]
        L.orc_next_interval.restype = C.c_int64
        L.orc_next_interval.argtypes = [f64p, f64p, C.c_double, C.c_double, C.c_double,
                                        C.c_int64, *part_args, f64p]
        L.orc_trace_intervals.restype = C.c_int64
        L.orc_trace_intervals.argtypes = [f64p, f64p, C.c_double, C.c_double, C.c_double,
                                          *part_args, C.c_int64, i64p, f64p, f64p]
        L.orc_march_range.restype = C.c_int64
        L.orc_march_range.argtypes = [f64p, f64p, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_double, f64p, C.c_long, C.c_double,
                                      C.c_double, *mesh_args, f64p, i32p]
        L.orc_render_frame.restype = None
        L.orc_render_frame.argtypes = [
            f64p, f64p, f64p, f64p, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int32,
            C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, f64p,
            f64p, C.c_int64, C.c_double, C.c_double, f64p, f64p, *part_args, f64p, *mesh_args,
            f64p, i64p, i32p, i64p, C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_int64,
            C.c_int]
        _lib = L
    return _lib


def _p(a, t):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(t))


class FlatBVH:
    """Reference-layout BVH (bvh.py:24-38) built by orc_build_bvh."""

    def __init__(self, lo: np.ndarray, hi: np.ndarray, leaf_size: int, fast: bool = True):
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        n = len(lo)
        m = 2 * n + 1
        self.node_lo = np.zeros((m, 3))
        self.node_hi = np.zeros((m, 3))
        self.left = np.zeros(m, np.int64)
        self.right = np.zeros(m, np.int64)
        self.start = np.zeros(m, np.int64)
        self.count = np.zeros(m, np.int64)
        self.prim = np.zeros(n, np.int64)
        build = lib().orc_build_bvh_fast if fast else lib().orc_build_bvh
        k = build(n, _p(lo, C.c_double), _p(hi, C.c_double), leaf_size,
                                _p(self.node_lo, C.c_double), _p(self.node_hi, C.c_double),
                                _p(self.left, C.c_int64), _p(self.right, C.c_int64),
                                _p(self.start, C.c_int64), _p(self.count, C.c_int64),
                                _p(self.prim, C.c_int64))
        for name in ("node_lo", "node_hi", "left", "right", "start", "count"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name)[:k]))

    def args(self):
        return [_p(self.node_lo, C.c_double), _p(self.node_hi, C.c_double),
                _p(self.left, C.c_int64), _p(self.right, C.c_int64), _p(self.start, C.c_int64),
                _p(self.count, C.c_int64), _p(self.prim, C.c_int64)]


class OracleScene:
    """Reference-layout kernel inputs of a scene (R:183-193 argument list)."""

    def __init__(self, scene):
        mesh, sampler = scene.mesh, scene.sampler
        self.scene = scene
        self.tets = np.ascontiguousarray(mesh.tets, dtype=np.int64)
        self.tet_orig = np.ascontiguousarray(sampler.tet_orig, dtype=np.float64)
        self.tet_inv = np.ascontiguousarray(sampler.tet_inv, dtype=np.float64)
        self.field = np.ascontiguousarray(mesh.field, dtype=np.float64)
        self.centering = int(mesh.centering)
        lo, hi = mesh.tet_aabbs()
        pad = 1e-7 * max(mesh.bounds.diagonal(), 1e-30)   # mesh.py:249
        self.mbvh = FlatBVH(lo - pad, hi + pad, 8)          # mesh.py:250
        self.p_lo = np.ascontiguousarray(scene.bvh.box_lo, dtype=np.float64)
        self.p_hi = np.ascontiguousarray(scene.bvh.box_hi, dtype=np.float64)
        self.pbvh = FlatBVH(self.p_lo, self.p_hi, 4)        # traversal.py:89
        self.mesh_lo = np.ascontiguousarray(mesh.bounds.lo, dtype=np.float64)
        self.mesh_hi = np.ascontiguousarray(mesh.bounds.hi, dtype=np.float64)

    def mesh_args(self):
        return [*self.mbvh.args(), _p(self.tets, C.c_int64), _p(self.tet_orig, C.c_double),
                _p(self.tet_inv, C.c_double), _p(self.field, C.c_double), self.centering]

    def part_args(self, active):
        return [*self.pbvh.args(), _p(self.p_lo, C.c_double), _p(self.p_hi, C.c_double),
                _p(active, C.c_uint8)]

    def field_at_many(self, pts, threads=None):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        n = len(pts)
        found = np.zeros(n, np.uint8)
        vals = np.zeros(n)
        tet = np.zeros(n, np.int64)
        lib().orc_field_at_many(n, _p(pts, C.c_double), *self.mesh_args(), _p(found, C.c_uint8),
                                _p(vals, C.c_double), _p(tet, C.c_int64),
                                threads or os.cpu_count() or 1)
        return found.astype(bool), vals, tet

    def render(self, camera, mode, params, *, jitter=False, track_per_partition=True,
               threads=None, rows=None, meta_state=None):
        """(rgba (H,W,4), samples (H,W), visited (H,W), ppart (P,) or None).
        `rows=(r0, r1)` renders only that row band (others stay zero)."""
        scene = self.scene
        active, sigma, tf = meta_state or scene.meta_state()
        active = np.ascontiguousarray(active, dtype=np.uint8)
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        right, up, fwd = (np.ascontiguousarray(v) for v in camera.basis())
        pos = np.ascontiguousarray(camera.position, dtype=np.float64)
        tan_half = math.tan(math.radians(camera.fov_y_deg) / 2.0)
        w, h = camera.width, camera.height
        P = len(self.p_lo)
        track = track_per_partition and mode != "reference"
        rgba = np.zeros((h, w, 4))
        samples = np.zeros((h, w), np.int64)
        visited = np.zeros((h, w), np.int32)
        ppart = np.zeros(P, np.int64)
        table = np.ascontiguousarray(tf.table, dtype=np.float64)
        bg = np.ascontiguousarray(scene.background, dtype=np.float64)
        r0, r1 = rows if rows is not None else (0, h)
        lib().orc_render_frame(
            _p(pos, C.c_double), _p(right, C.c_double), _p(up, C.c_double), _p(fwd, C.c_double),
            tan_half, w / h, w, h, 1 if jitter else 0, _MODE_IDS[mode], params.s1, params.s2,
            params.p, params.termination_opacity, scene.traversal_config.epsilon,
            _p(bg, C.c_double), _p(table, C.c_double), len(table), tf.domain[0], tf.domain[1],
            _p(self.mesh_lo, C.c_double), _p(self.mesh_hi, C.c_double), *self.part_args(active),
            _p(sigma, C.c_double), *self.mesh_args(), _p(rgba, C.c_double),
            _p(samples, C.c_int64), _p(visited, C.c_int32), _p(ppart, C.c_int64), P,
            1 if track else 0, 1, r0, r1, threads or os.cpu_count() or 1)
        return rgba, samples, visited, (ppart if track else None)


def step_size(s1, s2, p, sigma):
    return lib().orc_step_size(s1, s2, p, sigma)


def opacity_correction(alpha, s, s1):
    return lib().orc_opacity_correction(alpha, s, s1)


def tf_sample(table, lo, hi, v):
    """K:74-90 -> (r, g, b, a)."""
    table = np.ascontiguousarray(table, dtype=np.float64)
    out = np.zeros(4)
    lib().orc_tf_sample(_p(table, C.c_double), len(table), lo, hi, float(v), _p(out, C.c_double))
    return tuple(out.tolist())


def hash01(ix, iy):
    return lib().orc_hash01(ix, iy)
