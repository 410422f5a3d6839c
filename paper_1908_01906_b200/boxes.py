"""Box arithmetic the render path needs on the host.

Only three quantities reach the kernels through it, and each must carry the
reference's bits:

  * the mesh box (R:183-193 passes it as mesh_lo/mesh_hi for mode 0);
  * its diagonal, which sets epsilon = 1e-4 * diag (traversal.py:57-60) and
    the tet-box pad 1e-7 * diag (mesh.py:249) -- computed with the same
    numpy call (np.linalg.norm of hi - lo) as geometry.py:66-69;
  * refined partition bounds = box of the elements' corners clipped to the
    KD leaf box (partitions.py:58-66).

The rest of tetray.geometry (union, containment, volumes) is host-side
helper code outside the hot path and is not provided.
"""

from __future__ import annotations

import numpy as np


class Box:
    """Closed box [lo, hi] as two float64 3-vectors (lo > hi on an axis: empty)."""

    __slots__ = ("lo", "hi")

    def __init__(self, lo, hi):
        self.lo = np.asarray(lo, dtype=np.float64).reshape(3)
        self.hi = np.asarray(hi, dtype=np.float64).reshape(3)

    @classmethod
    def around(cls, points) -> "Box":
        p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        return cls(p.min(axis=0), p.max(axis=0))

    def clipped_to(self, other: "Box") -> "Box":
        return Box(np.maximum(self.lo, other.lo), np.minimum(self.hi, other.hi))

    def diagonal(self) -> float:
        if (self.lo > self.hi).any():
            return 0.0
        return float(np.linalg.norm(self.hi - self.lo))

    def __repr__(self) -> str:
        return f"Box(lo={self.lo.tolist()}, hi={self.hi.tolist()})"


# the name tetray exports for the same role (pkg/src/tetray/__init__.py:10)
AABB = Box


def unit(v: np.ndarray) -> np.ndarray:
    """v / |v| with numpy's norm (the camera basis, R:67-74)."""
    n = float(np.linalg.norm(v))
    if n == 0.0:
        raise ValueError("cannot normalize zero vector")
    return v / n
