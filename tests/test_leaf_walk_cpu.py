"""The leaf walk (TrPLeaf.walk, tr_leaf_walk; render.cu walk_leaf) restated on
the CPU: its answer must be the lowest-index tet accepting the point
(K:93-136, the -1e-9 slack of K:128, the first-hit rule of K:119) for
points inside a leaf's exclusive box -- on the generator's cubes (where the
walk certifies every tet), on an unstructured mesh, and on leaves whose tets
overlap (where certificates must be withheld)."""

import ctypes as C

import numpy as np
import pytest

TOL = 1e-9
TAU = 1e-6   # TR_WALK_TAU


@pytest.fixture(scope="module")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B


def bary(inv, orig, p):
    """K:121-128 in the device's order (Appendix A)."""
    q = p - orig
    l1 = (inv[0, 0] * q[0] + inv[0, 1] * q[1]) + inv[0, 2] * q[2]
    l2 = (inv[1, 0] * q[0] + inv[1, 1] * q[1]) + inv[1, 2] * q[2]
    l3 = (inv[2, 0] * q[0] + inv[2, 1] * q[1]) + inv[2, 2] * q[2]
    l0 = ((1.0 - l1) - l2) - l3
    return np.array([l0, l1, l2, l3])


def entry(walk, i):
    return (int(walk[i >> 1]) >> (16 * (i & 1))) & 0xFFFF


def scan(inv, orig, ids, p):
    """Lowest-index accepting tet of the leaf (records in id order)."""
    for k in np.argsort(ids):
        if (bary(inv[k], orig[k], p) >= -TOL).all():
            return int(k)
    return -1


def predict(w, pred, lo, p):
    """render.cu walk_leaf's start: the first tet, or its neighbour across the
    face the f32 predictor puts p beyond."""
    i = int(w[4]) & 7
    if pred is None:
        return i
    x = (p - lo.astype(np.float64)).astype(np.float32)
    r = np.asarray(pred, np.float32).reshape(3, 4)
    l123 = r[:, :3] @ x + r[:, 3]
    l = np.concatenate([[np.float32(1.0) - l123.sum()], l123])
    f = int(np.argmin(l))
    if l[f] < -1e-4:
        nb = (entry(w, i) >> (3 * f)) & 7
        if nb < 8:
            i = nb
    return i


def walk(inv, orig, ids, w, p, pred=None, lo=None):
    """render.cu walk_leaf."""
    n = len(ids)
    if int(w[4]) >> 31:
        i, seen = predict(w, pred, lo, p), 0
        if i >= n:
            i = int(w[4]) & 7
        for _ in range(n):
            seen |= 1 << i
            e = entry(w, i)
            l = bary(inv[i], orig[i], p)
            if (l >= -TOL).all():
                if (e >> 12) & 1 and (l >= TAU).all():
                    return i, True
                break
            f = int(np.argmin(l))
            nb = (e >> (3 * f)) & 7
            if nb == i or (seen >> nb) & 1:
                break
            i = nb
    return scan(inv, orig, ids, p), False


def leaf_tables(B, verts, tets, leaf_sets, with_pred=False):
    """tr_leaf_walk over leaves given as lists of tet ids (ascending); the
    exclusive-box corner ex_lo is set to the leaf's vertex minimum."""
    from paper_1908_01906_b200 import _lib
    recs = np.concatenate([np.asarray(s, np.uint32) for s in leaf_sets])
    leaves = np.zeros(len(leaf_sets), dtype=_lib.PLEAF_DTYPE)
    off = 0
    for i, s in enumerate(leaf_sets):
        leaves[i]["start"], leaves[i]["count"] = off, len(s)
        leaves[i]["ex_lo"] = verts[tets[s]].reshape(-1, 3).min(axis=0)
        off += len(s)
    verts = np.ascontiguousarray(verts, np.float64)
    tets = np.ascontiguousarray(tets, np.int64)
    pred = np.zeros((len(leaves), 12), np.float32)
    _lib.check(_lib.lib().tr_leaf_walk(len(leaves), _lib.vptr(leaves), _lib.vptr(recs),
                                       _lib.vptr(verts), _lib.vptr(tets), _lib.vptr(pred)),
               "tr_leaf_walk")
    return (leaves, recs, pred) if with_pred else (leaves, recs)


def inverses(verts, tets):
    p = verts[tets]
    e = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]], axis=-1)
    return np.linalg.inv(e), p[:, 0].copy()


def test_generator_cubes_walk_from_the_central_tet(B):
    m = B.generate_synthetic(2, "radial", B.Centering.VERTEX)
    cubes = [list(range(5 * c, 5 * c + 5)) for c in range(8)]
    leaves, _ = leaf_tables(B, m.vertices, m.tets, cubes)
    for lf in leaves:
        w = lf["walk"]
        assert int(w[4]) >> 31 and int(w[4]) & 7 == 4          # the central tet first
        for i in range(5):
            assert (entry(w, i) >> 12) & 1, "every tet of a cube is certified"
        nb = {(entry(w, 4) >> (3 * f)) & 7 for f in range(4)}
        assert nb == {0, 1, 2, 3}                               # one corner per face
        for i in range(4):                                      # corners: 1 inner face
            assert sum(((entry(w, i) >> (3 * f)) & 7) != i for f in range(4)) == 1
    # the device build of the generator's grid uses the same tables
    from paper_1908_01906_b200 import _lib
    assert _lib.lib().tr_leaf_walk(0, None, None, None, None, None) == 0
    two = np.zeros(24, np.float32)
    walk16 = np.zeros(16, np.uint32)
    assert _lib.lib().tr_grid_walk_pred(1e-7, _lib.vptr(two), _lib.vptr(walk16)) == 0
    lv, _, preds = leaf_tables(B, m.vertices, m.tets, cubes, with_pred=True)
    # an interior-cube class predictor = the per-leaf one up to the pad shift
    assert np.allclose(two[:12], preds[0], atol=1e-5)
    # the class walk tables (the march's analytic grid path) = the per-leaf
    # tables of an even and an odd cube
    assert np.array_equal(walk16[:8], lv[0]["walk"]) and np.array_equal(walk16[8:], lv[1]["walk"])


def _check_points(inv, orig, ids, w, pts, pred=None, lo=None):
    certified = 0
    for p in pts:
        want = scan(inv, orig, ids, p)
        got, cert = walk(inv, orig, ids, w, p)
        assert got == want
        if pred is not None:
            got_p, _ = walk(inv, orig, ids, w, p, pred, lo)
            assert got_p == want
        certified += cert
    return certified


def test_walk_equals_lowest_index_scan_on_cubes(B):
    m = B.generate_synthetic(3, "radial", B.Centering.VERTEX)
    inv_all, orig_all = inverses(m.vertices, m.tets)
    rng = np.random.default_rng(3)
    cubes = [list(range(5 * c, 5 * c + 5)) for c in range(27)]
    leaves, _, preds = leaf_tables(B, m.vertices, m.tets, cubes, with_pred=True)
    total = cert = hit = 0
    for c, lf, pr in zip(cubes, leaves, preds):
        lo = m.vertices[m.tets[c]].reshape(-1, 3).min(axis=0)
        pts = lo + rng.uniform(0, 1, (150, 3))
        # points on the cube's face diagonals and inner faces (ties)
        pts[:30, 1] = lo[1] + (pts[:30, 0] - lo[0])
        pts[30:50, 0] = lo[0] + np.round(pts[30:50, 0] - lo[0])
        ids = np.array(c)
        cert += _check_points(inv_all[c], orig_all[c], ids, lf["walk"], pts, pr, lf["ex_lo"])
        for p in pts[50:]:   # off the ties: the predicted start is the containing tet
            hit += predict(lf["walk"], pr, lf["ex_lo"], p) == scan(inv_all[c], orig_all[c], ids, p)
        total += len(pts)
    assert cert > 0.5 * total   # most points end on a certified tet
    assert hit > 0.98 * (total - 50 * len(cubes))


def test_walk_equals_scan_on_unstructured_leaves(B):
    """Jittered generator mesh (tests/cases.py jitterN): leaves of up to 8
    tets from the real point-BVH build; random points in each leaf's tets."""
    import cases
    from paper_1908_01906_b200.device import _padded_boxes, build_point_bvh
    sc = cases.build_scene(B, "jitter6")
    lo, hi = _padded_boxes(sc)
    nodes, leaves, pids, grid, lists = build_point_bvh(lo, hi)
    from paper_1908_01906_b200 import _lib
    verts = np.ascontiguousarray(sc.mesh.vertices)
    tets = np.ascontiguousarray(sc.mesh.tets)
    pred = np.zeros((len(leaves), 12), np.float32)
    _lib.check(_lib.lib().tr_leaf_walk(len(leaves), _lib.vptr(leaves), _lib.vptr(pids),
                                       _lib.vptr(verts), _lib.vptr(tets), _lib.vptr(pred)),
               "tr_leaf_walk")
    inv_all, orig_all = inverses(verts, tets)
    rng = np.random.default_rng(11)
    n_valid = 0
    for lf, pr in zip(leaves[::3], pred[::3]):
        s, n = int(lf["start"]), int(lf["count"])
        ids = pids[s:s + n].astype(np.int64)
        n_valid += int(lf["walk"][4]) >> 31
        pv = verts[tets[ids]]                       # (n, 4, 3)
        lam = rng.dirichlet(np.ones(4), size=(n, 12))
        pts = np.einsum("nkv,nva->nka", lam, pv).reshape(-1, 3)
        _check_points(inv_all[ids], orig_all[ids], ids, lf["walk"], pts, pr, lf["ex_lo"])
    assert n_valid > 0


def test_overlapping_tets_are_not_certified(B):
    """A leaf whose higher-id tet overlaps a lower-id one: the higher one
    must not be certified (the lowest index wins inside the overlap)."""
    base = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    verts = np.concatenate([base, base + 0.1, base, base + [1.0, 0, 0]])
    tets = np.arange(16).reshape(4, 4)
    # leaf 0: tet 0 and its shifted copy (overlap); leaf 1: tet 0 and an exact
    # duplicate (tet 2); leaf 2: tet 0 and a disjoint neighbour (tet 3)
    leaves, _ = leaf_tables(B, verts, tets, [[0, 1], [0, 2], [0, 3]])
    for lf, cert_hi in zip(leaves, (False, False, True)):
        w = lf["walk"]
        assert (entry(w, 0) >> 12) & 1                 # nothing below tet 0
        assert bool((entry(w, 1) >> 12) & 1) == cert_hi
    inv_all, orig_all = inverses(verts, tets)
    rng = np.random.default_rng(2)
    pts = rng.uniform(-0.1, 1.2, (400, 3))
    for lf, ids in zip(leaves, ([0, 1], [0, 2], [0, 3])):
        ids = np.array(ids)
        _check_points(inv_all[ids], orig_all[ids], ids, lf["walk"], pts)


def test_leaves_over_eight_tets_get_no_table(B):
    m = B.generate_synthetic(2, "radial", B.Centering.VERTEX)
    leaves, _ = leaf_tables(B, m.vertices, m.tets, [list(range(10))])
    assert int(leaves[0]["walk"][4]) == 0


def test_walk_equals_scan_on_delaunay_leaves(B):
    """Random Delaunay tetrahedralizations (scipy): conforming but irregular
    meshes with slivers; leaves = 8 consecutive tets along a Morton-like sort
    of their centroids.  The walk (with and without the predictor) must
    return the lowest-index accepting tet for points in and around every
    leaf's tets, including points on shared faces, edges and vertices."""
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(17)
    for trial in range(3):
        pts = rng.uniform(0.0, 4.0, (120, 3))
        tri = Delaunay(pts)
        tets = tri.simplices.astype(np.int64)
        p = pts[tets]
        e = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]], axis=-1)
        vol = np.abs(np.linalg.det(e))
        keep = vol > 1e-6                       # the reference rejects degenerate tets
        tets = tets[keep]
        cen = pts[tets].mean(axis=1)
        order = np.lexsort((cen[:, 2], cen[:, 1], np.floor(cen[:, 0])))
        leaf_sets = [sorted(order[k:k + 8].tolist()) for k in range(0, len(order), 8)]
        leaves, _, preds = leaf_tables(B, pts, tets, leaf_sets, with_pred=True)
        inv_all, orig_all = inverses(pts, tets)
        for lf, pr, ids in zip(leaves, preds, leaf_sets):
            ids = np.array(ids)
            pv = pts[tets[ids]]
            lam = rng.dirichlet(np.ones(4), size=(len(ids), 10))
            q = np.einsum("nkv,nva->nka", lam, pv).reshape(-1, 3)
            faces = pv[:, :3].mean(axis=1)             # on a face
            edges = 0.5 * (pv[:, 0] + pv[:, 1])         # on an edge
            verts = pv[:, 3]                            # a vertex
            out = q + rng.normal(0.0, 0.05, q.shape)    # near the leaf, maybe outside it
            allp = np.concatenate([q, faces, edges, verts, out])
            _check_points(inv_all[ids], orig_all[ids], ids, lf["walk"], allp, pr, lf["ex_lo"])
