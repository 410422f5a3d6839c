"""Scene/frame recipes shared by the golden-fixture generator (which runs the
REFERENCE package, tests/golden/make_golden.py) and the parity tests (which
build the same scenes with this repo's package).  `pkg` is either module: both
expose generate_synthetic, Centering, TetMesh, TransferFunction,
KdBuildConfig, Scene, Camera, AdaptiveParams with the same semantics.

Recipes follow the reference tests that pin the render path:
  golden_radial4   T/golden_scene.py:13-30 (the CLI golden image scene)
  conftest48       T/conftest.py:33-47
  radial16         T/golden/radial16_scene.json (A5's bundled scene)
  voidcell         T/test_render.py:292-300 (cell-centered)
  a6void / a6fog   T/test_acceptance.py:196-229
  single           T/test_render.py:197-210 (one partition)
  constant         T/test_render.py:303-327 (bitwise single-ray scene)
plus coverage the reference lacks (SURVEY.md §4 gaps): sigma < 1 with p != 2,
a camera inside the mesh, exactly axis-aligned rays, jitter, and the
benchmark scene radial59 (BASELINE config 2).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
ROOT = Path(__file__).resolve().parent.parent

TF_BANDED = {"domain": [0.0, 3.5],
             "rgba": [[0.0, 0.0, 1.0, 0.0], [0.0, 1.0, 1.0, 0.1], [0.0, 1.0, 0.0, 0.5],
                      [1.0, 1.0, 0.0, 0.3], [1.0, 0.0, 0.0, 0.8]]}

VOID_TF_CTRL = [(0.00, 0.1, 0.1, 0.9, 0.0), (0.30, 0.1, 0.5, 0.9, 0.0),
                (0.33, 0.1, 0.9, 0.2, 0.10), (0.50, 0.9, 0.9, 0.1, 0.06),
                (0.70, 0.9, 0.5, 0.1, 0.12), (0.95, 0.9, 0.1, 0.1, 0.08),
                (1.00, 0.9, 0.1, 0.5, 0.08)]


def radial16_tf_doc(n: int = 16) -> dict:
    doc = json.loads((GOLDEN / "radial16_tf.json").read_text())
    doc["domain"] = [0.0, 14.0 * n / 16.0]
    return doc


def _tf(pkg, doc):
    return pkg.TransferFunction.from_json(doc)


def _banded(pkg, domain):
    return pkg.TransferFunction(tuple(domain), np.array(TF_BANDED["rgba"]))


def _void_tf(pkg, void_alpha):
    ctrl = [(x, r, g, b, void_alpha if x <= 0.30 else a) for (x, r, g, b, a) in VOID_TF_CTRL]
    return pkg.TransferFunction.from_control_points(ctrl, domain=(0.0, 1.0), size=64)


def _sin_tf(pkg):
    ctrl = [(0.0, 0.2, 0.2, 0.9, 0.0), (0.35, 0.2, 0.6, 0.9, 0.02), (0.5, 0.9, 0.9, 0.2, 0.3),
            (0.65, 0.9, 0.4, 0.1, 0.05), (1.0, 0.9, 0.1, 0.1, 0.6)]
    return pkg.TransferFunction.from_control_points(ctrl, domain=(-1.0, 1.0), size=256)


def build_scene(pkg, name: str):
    """The scene of recipe `name` built with package `pkg`."""
    V, C = pkg.Centering.VERTEX, pkg.Centering.CELL
    K = pkg.KdBuildConfig
    if name in ("golden_radial4", "conftest48", "inside", "axis"):
        return pkg.Scene.build(pkg.generate_synthetic(4, "radial", V), _tf(pkg, TF_BANDED),
                               kd_config=K(40))
    if name == "radial16":
        return pkg.Scene.build(pkg.generate_synthetic(16, "radial", V),
                               _tf(pkg, radial16_tf_doc(16)), kd_config=K(48))
    if name.startswith("radial") and name[6:].isdigit() and name not in ("radial16",):
        n = int(name[6:])   # radial59 (1e6 tets), radial128 (1e7), radial272 (1e8): SURVEY §8d
        return pkg.Scene.build(pkg.generate_synthetic(n, "radial", V),
                               _tf(pkg, radial16_tf_doc(n)))
    if name.startswith("jitter") and name[6:].isdigit():
        # an unstructured mesh: the radialN generator's interior vertices
        # moved by up to 0.2 cell (seeded) -- leaves no longer align with a grid
        n = int(name[6:])
        m = pkg.generate_synthetic(n, "radial", V)
        v = m.vertices.copy()
        interior = ((v > 0.0) & (v < float(n))).all(axis=1)
        rng = np.random.default_rng(1234)
        v[interior] += rng.uniform(-0.2, 0.2, (int(interior.sum()), 3))
        mesh = pkg.TetMesh(v, m.tets, m.field, V)
        return pkg.Scene.build(mesh, _tf(pkg, radial16_tf_doc(n)))
    if name.startswith("grid") and name[4:].isdigit():
        # the same scene as radialN, generated in HBM without host mesh
        # arrays (grid_scene.py; radial585 = BASELINE config 4, 1e9 tets)
        n = int(name[4:])
        return pkg.GridScene.build(n, _tf(pkg, radial16_tf_doc(n)))
    if name == "voidcell":
        return pkg.Scene.build(pkg.generate_synthetic(3, "voidblock", C),
                               _banded(pkg, (0.0, 1.0)), kd_config=K(16))
    if name in ("a6void", "a6fog"):
        s = pkg.Scene.build(pkg.generate_synthetic(8, "voidblock", V), _void_tf(pkg, 0.0),
                            kd_config=K(max_leaf_elements=5))
        if name == "a6fog":
            s.set_transfer_function(_void_tf(pkg, 0.03))
        return s
    if name == "single":
        return pkg.Scene.build(pkg.generate_synthetic(2, "radial", V), _banded(pkg, (0.0, 1.8)),
                               kd_config=K(max_leaf_elements=10 ** 9))
    if name == "constant":
        m = pkg.generate_synthetic(2, "ramp", V)
        m = pkg.TetMesh(m.vertices, m.tets, np.full(len(m.field), 0.5), V)
        tf = pkg.TransferFunction.constant([0.9, 0.6, 0.2, 0.3], domain=(0.0, 1.0))
        return pkg.Scene.build(m, tf, kd_config=K(10 ** 9), background=[0, 0, 0, 0])
    if name == "sinus":
        return pkg.Scene.build(pkg.generate_synthetic(8, "sinusoidal", V), _sin_tf(pkg),
                               kd_config=K(12))
    raise KeyError(name)


def _grid_alias(name: str) -> str:
    if name.startswith("grid") and name[4:].isdigit():
        return "radial" + name[4:]
    if name.startswith("jitter") and name[6:].isdigit():
        return "radial" + name[6:]
    return name


def camera(pkg, name: str, scale: float = 1.0):
    Cam = pkg.Camera
    name = _grid_alias(name)
    if name == "golden_radial4":
        return Cam(position=[10.0, 6.0, 8.0], look_at=[2.0, 2.0, 2.0], up=[0, 1, 0],
                   fov_y_deg=40.0, width=64, height=64)
    if name == "conftest48":
        return Cam(position=[10.0, 6.0, 8.0], look_at=[2.0, 2.0, 2.0], up=[0, 1, 0],
                   fov_y_deg=40.0, width=48, height=48)
    if name == "inside":
        return Cam(position=[2.3, 1.9, 2.6], look_at=[0.2, 0.5, 0.0], up=[0, 1, 0],
                   fov_y_deg=70.0, width=40, height=32)
    if name == "axis":
        # odd width/height: the centre pixel's ray has exactly zero x and y
        # components, exercising slab's d == 0 branch (K:45-46)
        return Cam(position=[2.0, 2.0, 9.0], look_at=[2.0, 2.0, 2.0], up=[0, 1, 0],
                   fov_y_deg=30.0, width=33, height=31)
    if name.startswith("radial") and name[6:].isdigit() and name != "radial4":
        n = int(name[6:])
        f = n / 16.0
        return Cam(position=[40.0 * f, 26.0 * f, 34.0 * f], look_at=[8.0 * f] * 3, up=[0, 1, 0],
                   fov_y_deg=35.0, width=int(512 * scale), height=int(512 * scale))
    if name == "voidcell":
        return Cam(position=[8, 5, 6], look_at=[1.5, 1.5, 1.5], up=[0, 1, 0], fov_y_deg=40,
                   width=24, height=24)
    if name in ("a6void", "a6fog"):
        return Cam(position=[22, 14, 18], look_at=[4, 4, 4], up=[0, 1, 0], fov_y_deg=38.0,
                   width=128, height=128)
    if name == "single":
        return Cam(position=[6, 4, 5], look_at=[1, 1, 1], up=[0, 1, 0], fov_y_deg=40,
                   width=32, height=32)
    if name == "constant":
        return Cam(position=[5, 3, 4], look_at=[1, 1, 1], up=[0, 1, 0], fov_y_deg=45,
                   width=9, height=7)
    if name == "sinus":
        return Cam(position=[20, 13, 16], look_at=[4, 4, 4], up=[0, 1, 0], fov_y_deg=35,
                   width=96, height=80)
    raise KeyError(name)


def params(pkg, name: str):
    P = pkg.AdaptiveParams
    name = _grid_alias(name)
    if name in ("golden_radial4", "conftest48", "inside", "axis"):
        return P(s1=0.05, s2=0.3, p=2.0, termination_opacity=0.99)
    if name.startswith("radial") and name[6:].isdigit():
        return P(s1=0.08, s2=0.64, p=2.0, termination_opacity=0.9999)
    if name == "voidcell":
        return P(s1=0.1, s2=0.1)
    if name in ("a6void", "a6fog"):
        return P(s1=0.05, s2=0.4, p=2.0, termination_opacity=0.9999)
    if name == "single":
        return P(s1=0.04, s2=0.04)
    if name == "constant":
        return P(s1=0.07, s2=0.07)
    if name == "sinus":
        return P(s1=0.03, s2=0.5, p=6.0, termination_opacity=0.995)
    raise KeyError(name)


# (case id, scene recipe, modes, jitter)
FRAME_CASES = [
    ("golden_radial4", "golden_radial4", ("reference", "skip", "skip-adaptive"), False),
    ("golden_radial4_jitter", "golden_radial4", ("reference", "skip"), True),
    ("conftest48", "conftest48", ("reference", "skip", "skip-adaptive"), False),
    ("inside", "inside", ("reference", "skip", "skip-adaptive"), False),
    ("axis", "axis", ("reference", "skip", "skip-adaptive"), False),
    ("voidcell", "voidcell", ("reference", "skip", "skip-adaptive"), False),
    ("a6void", "a6void", ("reference", "skip", "skip-adaptive"), False),
    ("a6fog", "a6fog", ("reference", "skip", "skip-adaptive"), False),
    ("single", "single", ("reference", "skip"), False),
    ("constant", "constant", ("skip",), False),
    ("sinus", "sinus", ("reference", "skip", "skip-adaptive"), False),
    ("radial16", "radial16", ("reference", "skip", "skip-adaptive"), False),
]

# slow: only hashed, rendered by the generator once
BIG_CASES = [("radial59", "radial59", ("reference", "skip", "skip-adaptive"), False)]

# small enough to store full output arrays
FULL_ARRAY_CASES = {"golden_radial4", "golden_radial4_jitter", "conftest48", "inside", "axis",
                    "voidcell", "single", "constant"}


def point_set(scene, n_random: int, seed: int) -> np.ndarray:
    """Query points for field_at_many parity: random points in and around the
    mesh plus points exactly on vertices, faces and grid planes (where the
    lowest-index tie rule decides)."""
    rng = np.random.default_rng(seed)
    lo, hi = scene.mesh.bounds.lo, scene.mesh.bounds.hi
    ext = hi - lo
    pts = [rng.uniform(lo - 0.1 * ext, hi + 0.1 * ext, size=(n_random, 3))]
    g = rng.integers(0, np.maximum(ext.astype(int), 1) + 1, size=(n_random // 4, 3)) + lo
    pts.append(g.astype(np.float64))                              # grid vertices
    on = rng.uniform(lo, hi, size=(n_random // 4, 3))
    ax = rng.integers(0, 3, size=len(on))
    on[np.arange(len(on)), ax] = np.round(on[np.arange(len(on)), ax])  # grid planes
    pts.append(on)
    d = rng.uniform(lo, hi, size=(n_random // 4, 3))
    d[:, 1] = d[:, 0] + np.round(d[:, 1] - d[:, 0])               # face diagonals
    pts.append(d)
    return np.ascontiguousarray(np.concatenate(pts))
