"""Tetrahedral meshes: data model, TET1 IO, the synthetic `radialN` family,
and the host arrays the device point locator is built from.

Mirrors the public surface of tetray.mesh (pkg/src/tetray/mesh.py:37-284) so
callers can switch packages; the arrays it produces (tet_orig, tet_inv,
padded tet boxes, field values) are bit-identical to the reference's, which
tests/test_scene_build.py pins against fixtures made by the reference.
"""

from __future__ import annotations

import enum
import struct
from pathlib import Path
from typing import Optional

import numpy as np

from .boxes import Box

MAGIC = b"TET1"
_HEADER = struct.Struct("<4sBQQ")          # mesh.py:4-8 / 24-25
DEGENERACY_REL_TOL = 1e-12                 # mesh.py:28
VOID_LO, VOID_HI = 0.3, 0.7                # mesh.py:31-34
VOIDBLOCK_BASE, VOIDBLOCK_STEP = 0.35, 0.08
BOX_PAD_REL = 1e-7                         # mesh.py:249: pad = 1e-7 * diag
_CHUNK = 1 << 20


class Centering(enum.IntEnum):
    VERTEX = 0
    CELL = 1


class MeshError(Exception):
    pass


class MeshFormatError(MeshError):
    pass


def _gather_corners(vertices: np.ndarray, tets: np.ndarray, lo: int, hi: int) -> np.ndarray:
    return vertices[tets[lo:hi]]  # (n, 4, 3)


def tet_volumes(vertices: np.ndarray, tets: np.ndarray) -> np.ndarray:
    """Signed volume of every tet (det/6 of the edge matrix), chunked."""
    out = np.empty(len(tets))
    for lo in range(0, len(tets), _CHUNK):
        p = _gather_corners(vertices, tets, lo, lo + _CHUNK)
        out[lo:lo + len(p)] = np.linalg.det(p[:, 1:] - p[:, :1]) / 6.0
    return out


class TetMesh:
    """vertices (V,3) f64, tets (T,4) i64, field (V,) or (T,) f64."""

    def __init__(self, vertices, tets, field, centering, *, validate: bool = True):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        self.tets = np.ascontiguousarray(tets, dtype=np.int64).reshape(-1, 4)
        self.field = np.ascontiguousarray(field, dtype=np.float64).reshape(-1)
        self.centering = Centering(centering)
        self.synthetic: Optional[tuple] = None  # (n, field name) for generate_synthetic meshes
        if validate:
            self._validate()
        self.bounds = Box.around(self.vertices)

    def _validate(self) -> None:
        nv, nt = len(self.vertices), len(self.tets)
        if nv == 0 or nt == 0:
            raise MeshFormatError("mesh must have at least one vertex and one tet")
        bad = (self.tets < 0) | (self.tets >= nv)
        if bad.any():
            t = int(np.argmax(bad.any(axis=1)))
            raise MeshFormatError(f"tet {t} has a vertex index out of range (V={nv})")
        want = nv if self.centering == Centering.VERTEX else nt
        if len(self.field) != want:
            raise MeshFormatError(
                f"field length {len(self.field)} does not match "
                f"{self.centering.name.lower()}-centered count {want}")
        diag = float(np.linalg.norm(self.vertices.max(axis=0) - self.vertices.min(axis=0)))
        vols = np.abs(tet_volumes(self.vertices, self.tets))
        deg = np.flatnonzero(vols <= DEGENERACY_REL_TOL * diag ** 3)
        if len(deg):
            raise MeshFormatError(f"degenerate tet {int(deg[0])} (|volume|={vols[deg[0]]:g})")

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def n_tets(self) -> int:
        return len(self.tets)

    def tet_aabbs(self) -> tuple[np.ndarray, np.ndarray]:
        lo = np.empty((self.n_tets, 3))
        hi = np.empty((self.n_tets, 3))
        for a in range(0, self.n_tets, _CHUNK):
            p = _gather_corners(self.vertices, self.tets, a, a + _CHUNK)
            lo[a:a + len(p)] = p.min(axis=1)
            hi[a:a + len(p)] = p.max(axis=1)
        return lo, hi

    def __eq__(self, other) -> bool:
        return (isinstance(other, TetMesh) and self.centering == other.centering
                and np.array_equal(self.vertices, other.vertices)
                and np.array_equal(self.tets, other.tets)
                and np.array_equal(self.field, other.field))


# ----------------------------------------------------------------- TET1 IO

def load_mesh(path) -> TetMesh:
    raw = Path(path).read_bytes()
    if len(raw) < _HEADER.size:
        raise MeshFormatError("file too short for TET1 header")
    magic, centering, nv, nt = _HEADER.unpack_from(raw, 0)
    if magic != MAGIC:
        raise MeshFormatError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if centering not in (0, 1):
        raise MeshFormatError(f"unknown centering byte {centering}")
    nf = nv if centering == 0 else nt
    size = _HEADER.size + 12 * nv + 16 * nt + 4 * nf
    if len(raw) != size:
        raise MeshFormatError(f"file size {len(raw)} != expected {size} bytes")
    off = _HEADER.size
    v = np.frombuffer(raw, "<f4", 3 * nv, off).reshape(nv, 3)
    t = np.frombuffer(raw, "<u4", 4 * nt, off + 12 * nv).reshape(nt, 4)
    f = np.frombuffer(raw, "<f4", nf, off + 12 * nv + 16 * nt)
    return TetMesh(v.astype(np.float64), t.astype(np.int64), f.astype(np.float64),
                   Centering(centering))


def save_mesh(mesh: TetMesh, path) -> None:
    if mesh.n_vertices > 0xFFFFFFFF:
        raise MeshFormatError("too many vertices for u32 indices")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, int(mesh.centering), mesh.n_vertices, mesh.n_tets))
        fh.write(mesh.vertices.astype("<f4").tobytes())
        fh.write(mesh.tets.astype("<u4").tobytes())
        fh.write(mesh.field.astype("<f4").tobytes())


# ------------------------------------------------------- synthetic meshes
# N^3 unit cubes over [0, N]^3, five tets per cube, alternating parity so
# neighbouring cubes share face diagonals (mesh.py:147-231).  Corners are
# numbered 4x + 2y + z.

def _corner(x: int, y: int, z: int) -> int:
    return 4 * x + 2 * y + z


_FIVE_TETS = np.array([
    [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)],
    [(1, 1, 0), (0, 1, 0), (1, 0, 0), (1, 1, 1)],
    [(1, 0, 1), (0, 0, 1), (1, 1, 1), (1, 0, 0)],
    [(0, 1, 1), (1, 1, 1), (0, 0, 1), (0, 1, 0)],
    [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)],
])                                                   # (5 tets, 4 corners, xyz)
_MIRROR = _FIVE_TETS.copy()
_MIRROR[..., 0] = 1 - _MIRROR[..., 0]                 # odd cubes: mirrored in x
# corner offsets (dx, dy, dz) per parity / tet / vertex
CUBE_PATTERNS = np.stack([_FIVE_TETS, _MIRROR])      # (2, 5, 4, 3)


def _radial(p: np.ndarray, n: int) -> np.ndarray:
    d = p - n / 2.0
    return np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])


def _ramp(p: np.ndarray, n: int) -> np.ndarray:
    return p[:, 0].copy()


def _sinusoidal(p: np.ndarray, n: int) -> np.ndarray:
    w = 2.0 * np.pi / n
    return np.sin(w * p[:, 0]) * np.sin(w * p[:, 1]) * np.sin(w * p[:, 2])


def _voidblock(p: np.ndarray, n: int) -> np.ndarray:
    u = p / n
    void = ((u >= VOID_LO) & (u < VOID_HI)).all(axis=1)
    octant = (u[:, 0] >= 0.5).astype(np.int64) + 2 * (u[:, 1] >= 0.5) + 4 * (u[:, 2] >= 0.5)
    vals = VOIDBLOCK_BASE + VOIDBLOCK_STEP * octant
    vals[void] = 0.0
    return vals


ANALYTIC_FIELDS = {"ramp": _ramp, "radial": _radial, "sinusoidal": _sinusoidal,
                   "voidblock": _voidblock}


def synthetic_tets(n: int) -> np.ndarray:
    """(5 n^3, 4) vertex ids, cube-major in (i, j, k) order, 5 tets per cube."""
    g = n + 1
    i, j, k = (a.reshape(-1) for a in np.meshgrid(np.arange(n), np.arange(n), np.arange(n),
                                                   indexing="ij"))
    parity = (i + j + k) % 2
    off = CUBE_PATTERNS[parity]                        # (M, 5, 4, 3)
    vid = ((i[:, None, None] + off[..., 0]) * g + (j[:, None, None] + off[..., 1])) * g \
        + (k[:, None, None] + off[..., 2])
    return vid.reshape(-1, 4).astype(np.int64)


def generate_synthetic(n: int, field: str = "ramp",
                       centering: Centering = Centering.VERTEX) -> TetMesh:
    """Synthetic mesh over [0, n]^3 with an analytic field rounded through f32."""
    if n < 1:
        raise ValueError(f"resolution must be >= 1, got {n}")
    if field not in ANALYTIC_FIELDS:
        raise ValueError(f"unknown field {field!r}; choose from {sorted(ANALYTIC_FIELDS)}")
    centering = Centering(centering)
    g = n + 1
    ax = np.arange(g, dtype=np.float64)
    verts = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), axis=-1).reshape(-1, 3)
    tets = synthetic_tets(n)
    fn = ANALYTIC_FIELDS[field]
    if centering == Centering.VERTEX:
        vals = fn(verts, n)
    else:
        p = verts[tets]
        vals = fn((((p[:, 0] + p[:, 1]) + p[:, 2]) + p[:, 3]) / 4.0, n)
    vals = vals.astype(np.float32).astype(np.float64)
    # the generator's tets are non-degenerate by construction; skip the O(T)
    # volume check for the large benchmark meshes
    mesh = TetMesh(verts, tets, vals, centering, validate=n <= 64)
    mesh.synthetic = (n, field)
    return mesh


# ------------------------------------------------------------ point sampling

def _inverse_edge_matrices(vertices: np.ndarray, tets: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    p0 = vertices[tets[:, 0]]
    e = np.empty((len(tets), 3, 3))
    for c in range(3):  # columns are the edges v_{c+1} - v0 (mesh.py:253)
        e[:, :, c] = vertices[tets[:, c + 1]] - p0
    return p0, np.linalg.inv(e)


class MeshSampler:
    """Host arrays of the point locator: tet_orig (T,3), tet_inv (T,3,3)
    (= MeshSampler.tet_orig / tet_inv of mesh.py:251-254, bit for bit) and
    the padded tet boxes the device BVH is built over (mesh.py:248-250).

    Queries run on the device: sample_many -> tr_field_at_many (K:157-170)."""

    def __init__(self, mesh: TetMesh, leaf_size: int = 8):
        self.mesh = mesh
        self.leaf_size = int(leaf_size)
        syn = getattr(mesh, "synthetic", None)
        if syn is not None:
            # every cube's 5 edge matrices repeat by parity: invert the 10
            # distinct ones (numpy's batched inv is per-matrix LAPACK, so this
            # is bit-identical to inverting all T) and gather
            n = syn[0]
            cube = np.arange(mesh.n_tets) // 5
            i, j, k = cube // (n * n), (cube // n) % n, cube % n
            key = ((i + j + k) % 2) * 5 + np.arange(mesh.n_tets) % 5
            first = np.array([int(np.argmax(key == q)) if (key == q).any() else 0
                              for q in range(10)])
            _, inv10 = _inverse_edge_matrices(mesh.vertices, mesh.tets[first])
            self.tet_inv = np.ascontiguousarray(inv10[key])
            self.tet_orig = np.ascontiguousarray(mesh.vertices[mesh.tets[:, 0]])
        else:
            self.tet_orig, self.tet_inv = _inverse_edge_matrices(mesh.vertices, mesh.tets)
            self.tet_orig = np.ascontiguousarray(self.tet_orig)
            self.tet_inv = np.ascontiguousarray(self.tet_inv)
        self.pad = BOX_PAD_REL * max(mesh.bounds.diagonal(), 1e-30)
        self._device = {}

    def padded_boxes(self) -> tuple[np.ndarray, np.ndarray]:
        lo, hi = self.mesh.tet_aabbs()
        lo -= self.pad
        hi += self.pad
        return lo, hi

    def sample_many(self, points, device=None) -> tuple[np.ndarray, np.ndarray]:
        """(found mask, values) for a batch of points, on the GPU."""
        from .device import sample_points
        found, vals, _ = sample_points(self, points, device=device)
        return found, vals

    def locate_many(self, points, device=None) -> tuple[np.ndarray, np.ndarray]:
        """(tet id or -1, values) for a batch of points, on the GPU."""
        from .device import sample_points
        _, vals, tet = sample_points(self, points, device=device)
        return tet, vals

    def sample(self, point) -> Optional[float]:
        found, vals = self.sample_many(np.asarray(point, dtype=np.float64).reshape(1, 3))
        return float(vals[0]) if found[0] else None


def sample_field(sampler: MeshSampler, point) -> Optional[float]:
    return sampler.sample(point)
