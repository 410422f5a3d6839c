"""The trace pass's BSP enumeration (csrc/render.cu: bsp_next_interval),
restated in Python over the arrays the device uses, must reproduce the
reference's own traversal (_kernels.trace_intervals, K:233-259) on the
fixture rays, and the oracle's on random rays of other scenes.  CPU only."""

import json
import math

import numpy as np
import pytest

import cases as C


@pytest.fixture(scope="module")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B


def slab(o, d, lo, hi):
    t0, t1 = -math.inf, math.inf
    for a in range(3):
        if d[a] != 0.0:
            inv = 1.0 / d[a]
            x, y = (lo[a] - o[a]) * inv, (hi[a] - o[a]) * inv
            if x > y:
                x, y = y, x
            if x > t0:
                t0 = x
            if y < t1:
                t1 = y
        elif o[a] < lo[a] or o[a] > hi[a]:
            return 1.0, 0.0
    return t0, t1


def bsp_trace(nodes, pids, root, plo, phi, active, o, d, eps, kbuf=16):
    """Python statement of bsp_begin / bsp_enumerate_next / bsp_next_interval."""
    stack = []
    r0, r1 = slab(o, d, root[:3], root[3:])
    if r0 <= r1 and r1 > 0.0:
        stack.append((0, r0, r1))
    buf = []

    def enumerate_next():
        while stack:
            node, tn, tf = stack.pop()
            while True:
                if tf <= 0.0:
                    break
                info, aux, split = int(nodes[node]["info"]), int(nodes[node]["aux"]), float(nodes[node]["split"])
                if info < 0:
                    for k in range(aux):
                        p = int(pids[~info + k])
                        if not active[p]:
                            continue
                        pa, pb = slab(o, d, plo[p], phi[p])
                        if pa > pb or not pb > 0.0:
                            continue
                        assert len(buf) < kbuf, "candidate buffer overflow"
                        buf.append((p, pa, pb))
                    return
                ax, left, right = info & 3, node + 1, info >> 2
                if d[ax] == 0.0:
                    if o[ax] < split:
                        node = left
                    elif o[ax] > split:
                        node = right
                    else:
                        stack.append((right, tn, tf))
                        node = left
                    continue
                ts = (split - o[ax]) * (1.0 / d[ax])
                near, far = (left, right) if d[ax] > 0.0 else (right, left)
                if ts < tn:
                    node = far
                elif ts > tf:
                    node = near
                else:
                    stack.append((far, ts, tf))
                    node, tf = near, ts

    out = []
    t_min, last = 0.0, -1
    while True:
        thr = t_min + (0.0 if last < 0 else eps)
        while True:
            best = None
            for p, pa, pb in buf:
                if p == last or pb <= thr:
                    continue
                a_cl = pa if pa > t_min else t_min
                if best is None or a_cl < best[1] or (a_cl == best[1] and p < best[0]):
                    best = (p, a_cl, pb)
            if not stack:
                break
            tn = stack[-1][1]
            if best is not None and best[1] < (tn if tn > t_min else t_min):
                break
            enumerate_next()
        if best is None:
            return out
        out.append(best)
        t_min, last = best[2] - eps, best[0]
        buf[:] = [c for c in buf if not c[2] < t_min]


def _arrays(B, sc, active):
    from paper_1908_01906_b200.device import build_partition_bsp
    nodes, pids, root = build_partition_bsp(sc.bvh.box_lo, sc.bvh.box_hi)
    return nodes, pids, root


def test_bsp_reproduces_reference_traversal_fixture(B):
    misc = json.loads((C.GOLDEN / "reference_misc.json").read_text())
    sc = C.build_scene(B, "radial16")
    active = sc.meta_state()[0]
    nodes, pids, root = _arrays(B, sc, active)
    eps = sc.traversal_config.epsilon
    for ray in misc["trace_radial16"]:
        got = bsp_trace(nodes, pids, root, sc.bvh.box_lo, sc.bvh.box_hi, active,
                        np.array(ray["o"]), np.array(ray["d"]), eps)
        assert [g[0] for g in got] == ray["ids"]
        assert [g[1] for g in got] == ray["enter"]
        assert [g[2] for g in got] == ray["exit"]


@pytest.mark.parametrize("recipe", ["a6void", "sinus", "inside", "single"])
def test_bsp_matches_oracle_on_random_rays(B, recipe):
    import ctypes as Ct
    from oracle.oracle import OracleScene, _p, lib
    sc = C.build_scene(B, recipe)
    o = OracleScene(sc)
    active = np.ascontiguousarray(sc.meta_state()[0], dtype=np.uint8)
    nodes, pids, root = _arrays(B, sc, active)
    eps = sc.traversal_config.epsilon
    rng = np.random.default_rng(5)
    lo, hi = sc.mesh.bounds.lo, sc.mesh.bounds.hi
    for i in range(300):
        org = rng.uniform(lo - 3, hi + 3)
        dirn = rng.normal(size=3)
        if i % 10 == 0:
            dirn[rng.integers(3)] = 0.0      # axis-parallel components
            org = np.round(org)              # on split planes
        dirn /= np.linalg.norm(dirn)
        ids = np.zeros(512, np.int64)
        en = np.zeros(512)
        ex = np.zeros(512)
        k = lib().orc_trace_intervals(_p(org, Ct.c_double), _p(dirn, Ct.c_double), 0.0, math.inf,
                                      eps, *o.part_args(active), 512, _p(ids, Ct.c_int64),
                                      _p(en, Ct.c_double), _p(ex, Ct.c_double))
        got = bsp_trace(nodes, pids, root, sc.bvh.box_lo, sc.bvh.box_hi, active, org, dirn, eps)
        assert [g[0] for g in got] == ids[:k].tolist()
        assert [g[1] for g in got] == en[:k].tolist()
        assert [g[2] for g in got] == ex[:k].tolist()
