"""Soundness of the device point-location structure, checked on the CPU.

The kernel (csrc/render.cu: field_at / locate_full / scan_leaf) answers a
query either from the current leaf's EXCLUSIVE box (scan that leaf's ids in
ascending order) or by a full min-id-pruned descent.  Both are exact only if
(1) the f32 node boxes contain every padded tet box, (2) no other leaf's box
meets the interior of a leaf's exclusive box and (3) leaf ids are ascending.
This test walks the same arrays in numpy and requires the reference's
lowest-index answer (tests/golden/reference_points.npz) from BOTH paths.
"""

import numpy as np
import pytest

import cases as C

TOL = 1e-9


@pytest.fixture(scope="module")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B


def bary_ok(inv, orig, t, p):
    q = p - orig[t]
    A = inv[t]
    l1 = A[0, 0] * q[0] + A[0, 1] * q[1] + A[0, 2] * q[2]
    l2 = A[1, 0] * q[0] + A[1, 1] * q[1] + A[1, 2] * q[2]
    l3 = A[2, 0] * q[0] + A[2, 1] * q[1] + A[2, 2] * q[2]
    l0 = 1.0 - l1 - l2 - l3
    return l0 >= -TOL and l1 >= -TOL and l2 >= -TOL and l3 >= -TOL


def scan(ids, leaf, inv, orig, p, best):
    s, c = int(leaf["start"]), int(leaf["count"])
    for t in ids[s:s + c]:
        if t >= best:
            break
        if bary_ok(inv, orig, int(t), p):
            return int(t)
    return best


def in_box(p, lo, hi):
    return bool(np.all(p >= lo.astype(np.float64)) and np.all(p <= hi.astype(np.float64)))


def full(nodes, leaves, ids, inv, orig, p):
    best, best_leaf = 2 ** 32 - 1, -1
    stack = [0]
    while stack:
        n = nodes[stack.pop()]
        for c, (lo, hi) in enumerate(((n["lo0"], n["hi0"]), (n["lo1"], n["hi1"]))):
            ch, mn = int(n["child"][c]), int(n["minid"][c])
            if ch == -2 ** 31 or mn >= best or not in_box(p, lo, hi):
                continue
            if ch < 0:
                b = scan(ids, leaves[~ch], inv, orig, p, best)
                if b != best:
                    best, best_leaf = b, ~ch
            else:
                stack.append(ch)
    return (best if best != 2 ** 32 - 1 else -1), best_leaf


@pytest.mark.parametrize("recipe", ["golden_radial4", "voidcell", "sinus"])
def test_exclusive_leaf_and_full_descent_agree_with_reference(B, recipe):
    from paper_1908_01906_b200.device import _padded_boxes, build_point_bvh
    sc = C.build_scene(B, recipe)
    lo, hi = _padded_boxes(sc)
    nodes, leaves, ids, grid, _ = build_point_bvh(lo, hi)
    # (1) f32 child boxes contain the f64 padded boxes of everything below
    for n in nodes:
        for c, (blo, bhi) in enumerate(((n["lo0"], n["hi0"]), (n["lo1"], n["hi1"]))):
            ch = int(n["child"][c])
            if ch < 0 and ch != -2 ** 31:
                lf = leaves[~ch]
                t = ids[lf["start"]:lf["start"] + lf["count"]]
                assert (blo.astype(np.float64) <= lo[t]).all() and (bhi.astype(np.float64) >= hi[t]).all()
                assert np.all(np.diff(t.astype(np.int64)) > 0)
                assert int(n["minid"][c]) == int(t[0])
    fx = np.load(C.GOLDEN / "reference_points.npz")
    pts, want = fx[f"{recipe}/pts"], fx[f"{recipe}/tet"]
    inv, orig = sc.sampler.tet_inv, sc.sampler.tet_orig
    hits = 0
    for p, w in zip(pts[:1500], want[:1500]):
        got, leaf = full(nodes, leaves, ids, inv, orig, p)
        assert got == w
        # exclusive-leaf path from every leaf whose exclusive box strictly holds p
        for L in range(len(leaves)):
            lf = leaves[L]
            if np.all(p > lf["ex_lo"].astype(np.float64)) and np.all(p < lf["ex_hi"].astype(np.float64)):
                b = scan(ids, lf, inv, orig, p, 2 ** 32 - 1)
                assert (b if b != 2 ** 32 - 1 else -1) == w
                hits += 1
    assert hits > 100


def test_exclusive_boxes_are_disjoint_from_other_leaf_boxes(B):
    from paper_1908_01906_b200.device import _padded_boxes, build_point_bvh
    sc = C.build_scene(B, "sinus")
    lo, hi = _padded_boxes(sc)
    nodes, leaves, ids, grid, _ = build_point_bvh(lo, hi)
    boxes = []
    for lf in leaves:
        t = ids[lf["start"]:lf["start"] + lf["count"]]
        boxes.append((lo[t].min(axis=0), hi[t].max(axis=0)))
    for a, lf in enumerate(leaves):
        elo, ehi = lf["ex_lo"].astype(np.float64), lf["ex_hi"].astype(np.float64)
        if not np.all(elo < ehi):
            continue
        for b, (blo, bhi) in enumerate(boxes):
            if a == b:
                continue
            # open exclusive box vs closed leaf box: interiors must not meet
            assert np.any(blo >= ehi) or np.any(bhi <= elo), (a, b)


def test_native_boxes_and_parallel_build_invariants(B):
    """tr_tet_boxes equals numpy's padded boxes bit for bit; the task-parallel
    point-BVH build (used above 2^18 tets) keeps every structural invariant."""
    from paper_1908_01906_b200.device import _padded_boxes, build_point_bvh
    m = B.generate_synthetic(40, "radial", B.Centering.VERTEX)   # 320,000 tets
    sc = type("S", (), {})()
    sc.mesh = m
    lo, hi = _padded_boxes(sc)
    nlo, nhi = m.tet_aabbs()
    pad = 1e-7 * max(m.bounds.diagonal(), 1e-30)
    assert np.array_equal(lo, nlo - pad) and np.array_equal(hi, nhi + pad)
    nodes, leaves, ids, grid, _ = build_point_bvh(lo, hi)
    assert np.array_equal(np.sort(ids), np.arange(m.n_tets, dtype=np.uint32))
    starts, counts = leaves["start"].astype(np.int64), leaves["count"].astype(np.int64)
    assert np.array_equal(np.sort(starts), np.concatenate([[0], np.cumsum(counts[np.argsort(starts)])[:-1]]))
    # every reference is in range and every leaf / node is referenced exactly once
    ch = nodes["child"].reshape(-1)
    internal = ch[ch >= 0]
    leafref = ~ch[(ch < 0) & (ch != -2 ** 31)]
    assert np.array_equal(np.sort(internal), np.arange(1, len(nodes)))
    assert np.array_equal(np.sort(leafref), np.arange(len(leaves)))
    # min-id labels and f32 boxes bound their subtrees (bottom-up over nodes)
    sub_min = np.full(len(nodes), 2 ** 32 - 1, dtype=np.int64)
    sub_lo = np.full((len(nodes), 3), np.inf)
    sub_hi = np.full((len(nodes), 3), -np.inf)
    leaf_min = np.array([ids[s:s + c].min() for s, c in zip(starts, counts)], dtype=np.int64)
    leaf_lo = np.array([lo[ids[s:s + c]].min(axis=0) for s, c in zip(starts, counts)])
    leaf_hi = np.array([hi[ids[s:s + c]].max(axis=0) for s, c in zip(starts, counts)])
    order = np.argsort(-np.arange(len(nodes)))
    parent_done = np.zeros(len(nodes), bool)
    # resolve children before parents: iterate until stable (children have larger ids
    # within each spliced subtree, so a few passes suffice)
    for _ in range(64):
        changed = False
        for i in order:
            if parent_done[i]:
                continue
            vals = []
            ok = True
            for c in range(2):
                x = int(nodes[i]["child"][c])
                if x == -2 ** 31:
                    continue
                if x < 0:
                    vals.append((leaf_min[~x], leaf_lo[~x], leaf_hi[~x]))
                elif parent_done[x]:
                    vals.append((sub_min[x], sub_lo[x], sub_hi[x]))
                else:
                    ok = False
            if not ok:
                continue
            for c, (mn, blo, bhi) in zip(range(2), vals):
                assert int(nodes[i]["minid"][c]) == mn
                assert (nodes[i][f"lo{c}"].astype(np.float64) <= blo).all()
                assert (nodes[i][f"hi{c}"].astype(np.float64) >= bhi).all()
            sub_min[i] = min(v[0] for v in vals)
            sub_lo[i] = np.min([v[1] for v in vals], axis=0)
            sub_hi[i] = np.max([v[2] for v in vals], axis=0)
            parent_done[i] = changed = True
        if parent_done.all() or not changed:
            break
    assert parent_done.all()
