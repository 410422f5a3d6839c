"""Convex KD partitions of the mesh (tetray.partitions surface,
pkg/src/tetray/partitions.py:22-134).  The build itself is native
(tr_kd_build in csrc/host_build.cpp) and reproduces the reference's median,
straddle, flat-element and stopping rules exactly, so partition ids, bounds
and value ranges match bit for bit."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .boxes import Box
from .mesh import Centering, TetMesh


@dataclass
class KdBuildConfig:
    max_leaf_elements: int
    max_depth: int = 24
    split_rule: str = "median-of-centroids"

    def __post_init__(self):
        if self.max_leaf_elements < 1:
            raise ValueError("max_leaf_elements must be >= 1")
        if self.max_depth < 1:
            raise ValueError("max_depth must be >= 1")
        if self.split_rule != "median-of-centroids":
            raise ValueError(f"unknown split rule {self.split_rule!r}")


def default_config(n_tets: int) -> KdBuildConfig:
    """partitions.py:37-40: coarse partitions of max(64, T/4096) elements."""
    return KdBuildConfig(max_leaf_elements=max(64, n_tets // 4096), max_depth=24)


@dataclass
class Partition:
    id: int
    bounds: Box
    element_ids: np.ndarray
    value_range: tuple[float, float]
    meta: Optional[object] = None
    leaf_bounds: Optional[Box] = None


def element_value_ranges(mesh: TetMesh) -> np.ndarray:
    if mesh.centering == Centering.VERTEX:
        v = mesh.field[mesh.tets]
        return np.stack([v.min(axis=1), v.max(axis=1)], axis=1)
    return np.stack([mesh.field, mesh.field], axis=1)


def refine_partition_bounds(partition: Partition, mesh: TetMesh, leaf_bounds: Box) -> Partition:
    if len(partition.element_ids) == 0:
        raise ValueError("partition has no elements")
    pts = mesh.vertices[mesh.tets[partition.element_ids]].reshape(-1, 3)
    partition.bounds = Box.around(pts).clipped_to(leaf_bounds)
    return partition


@dataclass
class KdArrays:
    """Flat result of the native KD build."""
    offsets: np.ndarray   # (P+1,)
    ids: np.ndarray       # concatenated sorted element ids
    leaf_lo: np.ndarray   # (P,3) KD leaf boxes
    leaf_hi: np.ndarray
    lo: np.ndarray        # (P,3) refined bounds
    hi: np.ndarray
    vrange: np.ndarray    # (P,2)


def build_kd_arrays(mesh: TetMesh, config: KdBuildConfig) -> KdArrays:
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.tr_kd_build(mesh.n_vertices, _lib.ptr(mesh.vertices, C.c_double), mesh.n_tets,
                             _lib.ptr(mesh.tets, C.c_int64), _lib.ptr(mesh.field, C.c_double),
                             int(mesh.centering), _lib.ptr(mesh.bounds.lo, C.c_double),
                             _lib.ptr(mesh.bounds.hi, C.c_double), config.max_leaf_elements,
                             config.max_depth, C.byref(h)), "tr_kd_build")
    try:
        sz = np.zeros(2, dtype=np.int64)
        _lib.check(L.tr_kd_sizes(h, _lib.ptr(sz, C.c_int64)), "tr_kd_sizes")
        p, n = int(sz[0]), int(sz[1])
        out = KdArrays(np.empty(p + 1, np.int64), np.empty(n, np.int64),
                       np.empty((p, 3)), np.empty((p, 3)), np.empty((p, 3)), np.empty((p, 3)),
                       np.empty((p, 2)))
        _lib.check(L.tr_kd_copy(h, _lib.ptr(out.offsets, C.c_int64), _lib.ptr(out.ids, C.c_int64),
                                _lib.ptr(out.leaf_lo, C.c_double), _lib.ptr(out.leaf_hi, C.c_double),
                                _lib.ptr(out.lo, C.c_double), _lib.ptr(out.hi, C.c_double),
                                _lib.ptr(out.vrange, C.c_double)), "tr_kd_copy")
    finally:
        L.tr_host_free(h)
    return out


def build_partitions(mesh: TetMesh, config: Optional[KdBuildConfig] = None) -> list[Partition]:
    """KD-tree leaf partitions in the reference's DFS (left-first) id order."""
    config = config or default_config(mesh.n_tets)
    kd = build_kd_arrays(mesh, config)
    parts = []
    for i in range(len(kd.offsets) - 1):
        ids = kd.ids[kd.offsets[i]:kd.offsets[i + 1]]
        parts.append(Partition(id=i, bounds=Box(kd.lo[i], kd.hi[i]), element_ids=ids,
                               value_range=(float(kd.vrange[i, 0]), float(kd.vrange[i, 1])),
                               leaf_bounds=Box(kd.leaf_lo[i], kd.leaf_hi[i])))
    return parts


def partition_bounds_arrays(partitions: list[Partition]) -> tuple[np.ndarray, np.ndarray]:
    lo = np.ascontiguousarray(np.stack([p.bounds.lo for p in partitions]))
    hi = np.ascontiguousarray(np.stack([p.bounds.hi for p in partitions]))
    return lo, hi
