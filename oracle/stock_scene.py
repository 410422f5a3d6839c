"""Stock reference Scene objects for the reference arm (bench.py --impl reference).

TEST / BASELINE INFRASTRUCTURE ONLY.  The reference arm must time the
reference's own render() (pkg/src/tetray/render.py:161-205 -> the numba
_kernels.render_frame) on the benchmark workload.  The reference's
Scene.build (scene.py:52-68) cannot build radial272 (1e8 tets) in minutes:
its pure-Python median-split BVH (bvh.py:41-98) and KD split
(partitions.py:73-128) need ~40 min and ~40 GB.  So this module assembles the
STOCK dataclasses -- tetray.mesh.TetMesh, MeshSampler, bvh.FlatBVH,
partitions.Partition, scene.Scene, traversal.build_partition_bvh and
transfer.update_transfer_function (via Scene.set_transfer_function) -- around
arrays from the oracle's C restatement of the three heavy builders
(oracle/build.c: generator, KD split, tet BVH), which reproduce the
reference's arrays bit for bit (tests/test_oracle_build.py checks the scene
hashes and the BVH arrays against the stock builders).  The product library
(libtetray_b200.so) is never loaded on this path.
"""

from __future__ import annotations

import numpy as np

from .oracle import FlatBVH as OrcBVH
from .scene import GridMesh, GridSampler, kd_build


def build_stock_scene(tetray, n: int, tf_doc: dict):
    """Scene.build(generate_synthetic(n, "radial", VERTEX), TF(tf_doc)) as stock objects."""
    from tetray import bvh as RB
    from tetray import geometry as RG
    from tetray import mesh as RM
    from tetray import partitions as RP
    from tetray import scene as RS
    from tetray import transfer as RT
    from tetray import traversal as RV

    gm = GridMesh(n, "radial")
    mesh = object.__new__(RM.TetMesh)          # mesh.py:57-72 minus _validate (det of T matrices)
    mesh.vertices, mesh.tets, mesh.field = gm.vertices, gm.tets, gm.field
    mesh.centering = RM.Centering.VERTEX
    mesh.bounds = RG.AABB.from_points(gm.vertices)

    sampler = object.__new__(RM.MeshSampler)  # mesh.py:245-254
    sampler.mesh = mesh
    pad = 1e-7 * max(mesh.bounds.diagonal(), 1e-30)
    lo, hi = gm.tet_aabbs(pad)
    b = OrcBVH(lo, hi, 8)
    del lo, hi
    sampler.bvh = RB.FlatBVH(node_lo=b.node_lo, node_hi=b.node_hi, left=b.left, right=b.right,
                             start=b.start, count=b.count, prim=b.prim)
    gs = GridSampler(gm)
    sampler.tet_orig, sampler.tet_inv = gs.tet_orig, gs.tet_inv

    kd = RP.default_config(len(gm.tets))
    ps = kd_build(gm, kd.max_leaf_elements, kd.max_depth)
    partitions = [RP.Partition(id=p, bounds=RG.AABB(ps.lo[p].copy(), ps.hi[p].copy()),
                               element_ids=ps.element_ids(p).copy(),
                               value_range=(float(ps.vrange[p, 0]), float(ps.vrange[p, 1])))
                  for p in range(len(ps))]
    scene = RS.Scene(mesh=mesh, sampler=sampler, partitions=partitions, kd_config=kd,
                     traversal_config=RV.TraversalConfig.for_diagonal(mesh.bounds.diagonal()))
    scene.bvh = RV.build_partition_bvh(scene.partitions)
    scene.set_transfer_function(RT.TransferFunction.from_json(tf_doc))
    return scene


def stock_bvh_equal(a, b) -> bool:
    return all(np.array_equal(getattr(a, k), getattr(b, k))
               for k in ("node_lo", "node_hi", "left", "right", "start", "count", "prim"))
