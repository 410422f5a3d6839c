"""The oracle's own scene build (TEST INFRASTRUCTURE ONLY; see oracle/build.c).

Builds, without the product library and without the reference package, the
kernel inputs of a synthetic `radialN` / `rampN` scene exactly as the
reference's Scene.build makes them (pkg/src/tetray/scene.py:52-68):

  mesh       generate_synthetic(n, field, VERTEX)        mesh.py:198-231  (orc_gen_grid)
  sampler    tet_orig / tet_inv                          mesh.py:251-254
             (np.linalg.inv of the 10 distinct integer edge matrices -- every
             tet's edge matrix is one of them, translation-invariant -- then
             gathered per tet: numpy's batched inv runs LAPACK gesv per
             matrix, so the bits are those of inverting all T matrices)
  partitions build_partitions(mesh, default_config(T))  partitions.py:37-128 (orc_kd_build)
  metadata   update_transfer_function                    transfer.py:95-167 (numpy, below)
  epsilon    1e-4 x bounds diagonal                      traversal.py:55-60

The result duck-types the attributes oracle.OracleScene and the stock
reference scene assembly (oracle/stock_scene.py) read.  Pinned against the
reference's own scene hashes at radial16/59/128/272
(tests/test_oracle_build.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .oracle import _p, lib, tf_sample

_FIELDS = {"ramp": 0, "radial": 1}


def _bind():
    L = lib()
    if not getattr(L, "_build_bound", False):
        f64p, i64p, u8p = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_uint8)
        L.orc_gen_grid.restype = C.c_int
        L.orc_gen_grid.argtypes = [C.c_int64, C.c_int, f64p, i64p, f64p, u8p]
        L.orc_tet_boxes.restype = None
        L.orc_tet_boxes.argtypes = [C.c_int64, f64p, i64p, C.c_double, f64p, f64p]
        L.orc_kd_build.restype = C.c_void_p
        L.orc_kd_build.argtypes = [C.c_int64, f64p, i64p, f64p, C.c_int, C.c_int64, C.c_int64,
                                   f64p, f64p, i64p, i64p]
        L.orc_kd_take.restype = None
        L.orc_kd_take.argtypes = [C.c_void_p, i64p, i64p, f64p, f64p, f64p]
        L._build_bound = True
    return L


class Bounds:
    def __init__(self, lo, hi):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)

    def diagonal(self) -> float:   # geometry.py:53-56
        return float(np.linalg.norm(self.hi - self.lo))


class GridMesh:
    """generate_synthetic(n, field, VERTEX) (mesh.py:198-231)."""

    def __init__(self, n: int, field: str = "radial"):
        g = n + 1
        self.vertices = np.empty((g ** 3, 3))
        self.tets = np.empty((5 * n ** 3, 4), np.int64)
        self.field = np.empty(g ** 3)
        self.pattern = np.empty(5 * n ** 3, np.uint8)
        rc = _bind().orc_gen_grid(n, _FIELDS[field], _p(self.vertices, C.c_double),
                                  _p(self.tets, C.c_int64), _p(self.field, C.c_double),
                                  _p(self.pattern, C.c_uint8))
        if rc != 0:
            raise ValueError(f"orc_gen_grid({n}, {field!r}) failed")
        self.n = n
        self.centering = 0
        self.bounds = Bounds(np.zeros(3), np.full(3, float(n)))   # AABB.from_points(vertices)

    @property
    def n_tets(self) -> int:
        return len(self.tets)

    def tet_aabbs(self, pad: float = 0.0):
        lo = np.empty((self.n_tets, 3))
        hi = np.empty((self.n_tets, 3))
        _bind().orc_tet_boxes(self.n_tets, _p(self.vertices, C.c_double), _p(self.tets, C.c_int64),
                              pad, _p(lo, C.c_double), _p(hi, C.c_double))
        return lo, hi


class GridSampler:
    """tet_orig / tet_inv of MeshSampler (mesh.py:251-254)."""

    def __init__(self, mesh: GridMesh):
        pats = {}   # tets 0-4: cube (0,0,0) (even), 5-9: cube (0,0,1) (odd)
        for t in range(min(10, mesh.n_tets)):
            p = mesh.vertices[mesh.tets[t]]
            pats[int(mesh.pattern[t])] = np.stack([p[1] - p[0], p[2] - p[0], p[3] - p[0]],
                                                  axis=-1)
        keys = sorted(pats)
        inv = np.linalg.inv(np.stack([pats[k] for k in keys]))
        lut = np.zeros((10, 3, 3))
        for i, k in enumerate(keys):
            lut[k] = inv[i]
        self.tet_inv = np.ascontiguousarray(lut[mesh.pattern])
        self.tet_orig = np.ascontiguousarray(mesh.vertices[mesh.tets[:, 0]])


class TF:
    """TransferFunction (transfer.py:22-75): domain + (n, 4) table."""

    def __init__(self, domain, table):
        self.domain = (float(domain[0]), float(domain[1]))
        self.table = np.ascontiguousarray(table, dtype=np.float64).reshape(-1, 4)

    @classmethod
    def from_json(cls, doc):
        return cls(tuple(doc["domain"]), np.asarray(doc["rgba"], dtype=np.float64))

    @property
    def size(self) -> int:
        return int(self.table.shape[0])


def partition_meta(tf: TF, vrange: np.ndarray):
    """(active u8[P], sigma f64[P]): compute_partition_meta + normalize_variances
    (transfer.py:95-141) and active_sigma_arrays (traversal.py:94-99)."""
    lo, hi = tf.domain
    n = tf.size
    maxop = np.empty(len(vrange))
    raw = np.empty(len(vrange))
    for i, (rmin, rmax) in enumerate(vrange):
        rmin, rmax = float(rmin), float(rmax)
        u_min = (rmin - lo) / (hi - lo) * (n - 1)
        u_max = (rmax - lo) / (hi - lo) * (n - 1)
        j0 = max(int(np.floor(u_min)) + 1, 0)
        j1 = min(int(np.ceil(u_max)) - 1, n - 1)
        rows = [np.array(tf_sample(tf.table, lo, hi, rmin))]
        if j1 >= j0:
            rows.extend(tf.table[j0:j1 + 1])
        rows.append(np.array(tf_sample(tf.table, lo, hi, rmax)))
        rows = np.stack(rows)
        alpha = rows[:, 3]
        weighted = rows[:, :3] * alpha[:, None]
        mean = weighted.mean(axis=0)
        raw[i] = float(((weighted - mean) ** 2).sum(axis=1).mean())
        maxop[i] = float(alpha.max())
    v_min, v_max = float(raw.min()), float(raw.max())
    sigma = np.ones(len(raw)) if v_max == v_min else (raw - v_min) / (v_max - v_min)
    return (maxop > 0.0).astype(np.uint8), np.ascontiguousarray(sigma, dtype=np.float64)


class PartitionSet:
    """build_partitions output as flat arrays (partition p = ids[offsets[p]:offsets[p+1]])."""

    def __init__(self, offsets, ids, lo, hi, vrange):
        self.offsets, self.ids, self.lo, self.hi, self.vrange = offsets, ids, lo, hi, vrange

    def __len__(self):
        return len(self.lo)

    def element_ids(self, p):
        return self.ids[self.offsets[p]:self.offsets[p + 1]]


def kd_build(mesh: GridMesh, max_leaf: int, max_depth: int = 24) -> PartitionSet:
    L = _bind()
    n_parts, n_ids = C.c_int64(0), C.c_int64(0)
    lo = np.ascontiguousarray(mesh.bounds.lo)
    hi = np.ascontiguousarray(mesh.bounds.hi)
    h = L.orc_kd_build(mesh.n_tets, _p(mesh.vertices, C.c_double), _p(mesh.tets, C.c_int64),
                       _p(mesh.field, C.c_double), int(mesh.centering), max_leaf, max_depth,
                       _p(lo, C.c_double), _p(hi, C.c_double), C.byref(n_parts), C.byref(n_ids))
    P, N = n_parts.value, n_ids.value
    offsets = np.zeros(P + 1, np.int64)
    ids = np.zeros(N, np.int64)
    plo, phi, vr = np.zeros((P, 3)), np.zeros((P, 3)), np.zeros((P, 2))
    L.orc_kd_take(h, _p(offsets, C.c_int64), _p(ids, C.c_int64), _p(plo, C.c_double),
                  _p(phi, C.c_double), _p(vr, C.c_double))
    return PartitionSet(offsets, ids, plo, phi, vr)


def _normalize(v):   # geometry.py:13-17
    n = float(np.linalg.norm(v))
    if n == 0.0:
        raise ValueError("cannot normalize zero vector")
    return v / n


class Camera:
    """render.py:47-75 (same numpy calls, so the same basis bits)."""

    def __init__(self, position, look_at, up, fov_y_deg=45.0, width=256, height=256):
        self.position = np.asarray(position, dtype=np.float64).reshape(3)
        self.look_at = np.asarray(look_at, dtype=np.float64).reshape(3)
        self.up = np.asarray(up, dtype=np.float64).reshape(3)
        self.fov_y_deg, self.width, self.height = fov_y_deg, int(width), int(height)

    def basis(self):
        fwd = _normalize(self.look_at - self.position)
        right = _normalize(np.cross(fwd, self.up))
        return right, np.cross(right, fwd), fwd


class AdaptiveParams:
    """render.py:29-44."""

    def __init__(self, s1, s2, p=2.0, termination_opacity=0.99):
        self.s1, self.s2, self.p, self.termination_opacity = s1, s2, p, termination_opacity


class _BVHBoxes:
    def __init__(self, lo, hi):
        self.box_lo, self.box_hi = lo, hi


class _Traversal:
    def __init__(self, eps):
        self.epsilon = eps


class GridScene:
    """Scene.build(generate_synthetic(n, field, VERTEX), tf) (scene.py:52-68)
    with default_config(T) (partitions.py:37-40) unless `max_leaf` is given."""

    def __init__(self, n: int, tf: TF, field: str = "radial", max_leaf=None, max_depth=24,
                 background=(0.0, 0.0, 0.0, 1.0)):
        self.mesh = GridMesh(n, field)
        self.sampler = GridSampler(self.mesh)
        T = self.mesh.n_tets
        leaf = max(64, T // 4096) if max_leaf is None else int(max_leaf)
        self.parts = kd_build(self.mesh, leaf, max_depth)
        self.bvh = _BVHBoxes(self.parts.lo, self.parts.hi)
        self.traversal_config = _Traversal(1e-4 * self.mesh.bounds.diagonal())
        self.background = np.asarray(background, dtype=np.float64)
        self.set_transfer_function(tf)

    def set_transfer_function(self, tf: TF):
        self.tf = tf
        active, sigma = partition_meta(tf, self.parts.vrange)
        self._meta = (active, sigma, tf)

    def meta_state(self):
        return self._meta

    @property
    def n_partitions(self) -> int:
        return len(self.parts)


def radial_tf(doc16: dict, n: int) -> TF:
    """The radial16 TF scaled to radialN (tests/cases.py radial16_tf_doc)."""
    return TF((0.0, 14.0 * n / 16.0), doc16["rgba"])


__all__ = ["GridScene", "GridMesh", "TF", "Camera", "AdaptiveParams", "kd_build", "partition_meta", "radial_tf"]
