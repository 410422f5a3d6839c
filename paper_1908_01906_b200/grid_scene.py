"""Synthetic cube-grid scenes built without host mesh arrays.

The reference builds a scene on the host: generate_synthetic (mesh.py:147-231)
allocates the vertex, tet and field arrays, MeshSampler (mesh.py:238-254)
the padded tet boxes, BVH and inverse edge matrices, and build_partitions
(partitions.py:73-128) runs the KD split over tet centroids.  At BASELINE
config 4 (radial585: 1.0e9 tets) those arrays exceed 250 GB of host memory.
For the generator's mesh every one of these products has a closed form, so
`GridScene.build` makes the same Scene without them:

  * partitions: tr_kd_build_grid -- the KD split of partitions.py evaluated on
    cube ranges (identical partitions, bounds and value ranges; checked
    against the general builder in tests/test_grid_scene.py);
  * geometry: generated straight into HBM by tr_grid_scene_build
    (csrc/synth.cu) when the scene is first rendered -- tet records, one
    leaf per cube, the cube grid as the point grid, a BVH2 over the cubes;
  * inverse edge matrices: the 10 distinct ones (5 tets x 2 cube parities)
    inverted on the host with numpy, exactly as MeshSampler does.

Rendering, metadata epochs and TF edits then go through the unchanged
render() / Scene API.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .boxes import Box
from .mesh import BOX_PAD_REL, Centering, _inverse_edge_matrices, generate_synthetic
from .partitions import KdArrays, KdBuildConfig, Partition, default_config
from .scene import Scene
from .transfer import TransferFunction

FIELD_IDS = {"ramp": 0, "radial": 1}


class GridMesh:
    """generate_synthetic(n, field, VERTEX) described, not materialised."""

    device_generated = True

    def __init__(self, n: int, field: str = "radial"):
        if n < 1:
            raise ValueError(f"resolution must be >= 1, got {n}")
        if field not in FIELD_IDS:
            raise ValueError(f"grid scenes support fields {sorted(FIELD_IDS)}, not {field!r}")
        self.n = int(n)
        self.field = field
        self.field_id = FIELD_IDS[field]
        self.centering = Centering.VERTEX
        self.n_tets = 5 * self.n ** 3
        self.n_vertices = (self.n + 1) ** 3
        self.bounds = Box(np.zeros(3), np.full(3, float(self.n)))
        self.synthetic = (self.n, field)


class GridSampler:
    """MeshSampler's per-scene constants for a GridMesh: the box pad
    (mesh.py:249) and the 10 distinct inverse edge matrices (mesh.py:251-254)."""

    def __init__(self, mesh: GridMesh):
        self.mesh = mesh
        self.pad = BOX_PAD_REL * max(mesh.bounds.diagonal(), 1e-30)
        # cube (0,0,0) is even, cube (0,0,1) odd: their 10 tets carry every
        # edge matrix of the mesh (integer edges, translation invariant)
        small = generate_synthetic(2, "ramp", Centering.VERTEX)
        _, inv = _inverse_edge_matrices(small.vertices, small.tets[:10])
        self.inv10 = np.ascontiguousarray(inv)
        self._device = {}


def build_grid_kd(n: int, field: str, config: KdBuildConfig, with_ids: bool = False) -> KdArrays:
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.tr_kd_build_grid(int(n), FIELD_IDS[field], config.max_leaf_elements,
                                  config.max_depth, 1 if with_ids else 0, C.byref(h)),
               "tr_kd_build_grid")
    try:
        sz = np.zeros(2, dtype=np.int64)
        _lib.check(L.tr_kd_sizes(h, _lib.ptr(sz, C.c_int64)), "tr_kd_sizes")
        p, m = int(sz[0]), int(sz[1])
        out = KdArrays(np.empty(p + 1, np.int64), np.empty(max(m, 1), np.int64),
                       np.empty((p, 3)), np.empty((p, 3)), np.empty((p, 3)), np.empty((p, 3)),
                       np.empty((p, 2)))
        _lib.check(L.tr_kd_copy(h, _lib.ptr(out.offsets, C.c_int64), _lib.ptr(out.ids, C.c_int64),
                                _lib.ptr(out.leaf_lo, C.c_double), _lib.ptr(out.leaf_hi, C.c_double),
                                _lib.ptr(out.lo, C.c_double), _lib.ptr(out.hi, C.c_double),
                                _lib.ptr(out.vrange, C.c_double)), "tr_kd_copy")
        out.ids = out.ids[:m]
    finally:
        L.tr_host_free(h)
    return out


def build_grid_partitions(n: int, field: str, config: KdBuildConfig) -> list[Partition]:
    """The partitions build_partitions would produce for generate_synthetic(n,
    field), without element id lists (each holds all tets of a cube range;
    `n_elements` gives the count)."""
    kd = build_grid_kd(n, field, config)
    parts = []
    empty = np.empty(0, np.int64)
    for i in range(len(kd.offsets) - 1):
        p = Partition(id=i, bounds=Box(kd.lo[i], kd.hi[i]), element_ids=empty,
                      value_range=(float(kd.vrange[i, 0]), float(kd.vrange[i, 1])),
                      leaf_bounds=Box(kd.leaf_lo[i], kd.leaf_hi[i]))
        p.n_elements = int(kd.offsets[i + 1] - kd.offsets[i])
        parts.append(p)
    return parts


class GridScene(Scene):
    """A Scene over a device-generated synthetic cube grid."""

    @classmethod
    def build(cls, n: int, tf: TransferFunction, field: str = "radial",
              kd_config: Optional[KdBuildConfig] = None, epsilon: Optional[float] = None,
              background=None) -> "GridScene":
        mesh = GridMesh(n, field)
        kd = kd_config if kd_config is not None else default_config(mesh.n_tets)
        return cls._assemble(mesh, GridSampler(mesh), build_grid_partitions(n, field, kd), kd, tf,
                             epsilon, background)
