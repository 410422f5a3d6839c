"""Partition traversal structure (tetray.traversal surface,
pkg/src/tetray/traversal.py:25-99).  The BVH over partition boxes is built
natively (tr_bbvh_build) as a BVH2 with f64 child boxes; next_interval's
result does not depend on the tree, only on the partition
boxes, the active mask and the leaf arithmetic, which the kernel keeps."""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .partitions import Partition, partition_bounds_arrays

BUILD_COUNT = 0  # traversal.py:22: incremented on every partition BVH build


@dataclass
class Ray:
    origin: np.ndarray
    direction: np.ndarray
    t_min: float = 0.0
    t_max: float = math.inf

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float64).reshape(3)
        self.direction = np.asarray(self.direction, dtype=np.float64).reshape(3)
        n = float(np.linalg.norm(self.direction))
        if abs(n - 1.0) > 1e-9:
            raise ValueError(f"ray direction must be unit length (|d| = {n})")
        if not self.t_min <= self.t_max:
            raise ValueError(f"t_min {self.t_min} > t_max {self.t_max}")


@dataclass
class PartitionInterval:
    partition_id: int
    t_enter: float
    t_exit: float


@dataclass
class TraversalConfig:
    epsilon: float

    def __post_init__(self):
        if not self.epsilon > 0.0:
            raise ValueError("epsilon must be positive")

    @staticmethod
    def for_diagonal(diag: float) -> "TraversalConfig":
        return TraversalConfig(epsilon=1e-4 * diag)  # traversal.py:57-60


@dataclass
class PartitionBVH:
    box_lo: np.ndarray        # (P,3) refined partition bounds
    box_hi: np.ndarray
    nodes: np.ndarray         # TrBNode records (BNODE_DTYPE)
    n_partitions: int = field(init=False)

    def __post_init__(self):
        self.n_partitions = int(self.box_lo.shape[0])

    def activity(self, active: np.ndarray) -> np.ndarray:
        """Per-node bits: child subtree reaches an active partition."""
        act = np.ascontiguousarray(active, dtype=np.uint8)
        out = np.empty(len(self.nodes), dtype=np.uint8)
        _lib.check(_lib.lib().tr_bnodes_activity(len(self.nodes), _lib.vptr(self.nodes),
                                                 _lib.ptr(act, C.c_uint8), _lib.ptr(out, C.c_uint8)),
                   "tr_bnodes_activity")
        return out


def build_bvh_over_boxes(lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    L = _lib.lib()
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    hi = np.ascontiguousarray(hi, dtype=np.float64)
    h = C.c_void_p()
    _lib.check(L.tr_bbvh_build(len(lo), _lib.ptr(lo, C.c_double), _lib.ptr(hi, C.c_double),
                               C.byref(h)), "tr_bbvh_build")
    try:
        n = np.zeros(1, np.int64)
        _lib.check(L.tr_bbvh_sizes(h, _lib.ptr(n, C.c_int64)), "tr_bbvh_sizes")
        nodes = np.zeros(int(n[0]), dtype=_lib.BNODE_DTYPE)
        _lib.check(L.tr_bbvh_copy(h, _lib.vptr(nodes)), "tr_bbvh_copy")
    finally:
        L.tr_host_free(h)
    return nodes


def build_partition_bvh(partitions: list[Partition]) -> PartitionBVH:
    """Rebuilt only when partition geometry changes; TF edits never call it."""
    global BUILD_COUNT
    if not partitions:
        raise ValueError("need at least one partition")
    lo, hi = partition_bounds_arrays(partitions)
    bvh = PartitionBVH(box_lo=lo, box_hi=hi, nodes=build_bvh_over_boxes(lo, hi))
    BUILD_COUNT += 1
    return bvh


def active_sigma_arrays(partitions: list[Partition]) -> tuple[np.ndarray, np.ndarray]:
    active = np.fromiter((1 if (p.meta is not None and p.meta.active) else 0 for p in partitions),
                         dtype=np.uint8, count=len(partitions))
    sigma = np.fromiter((p.meta.normalized_variance if p.meta is not None else 1.0
                         for p in partitions), dtype=np.float64, count=len(partitions))
    return active, sigma
