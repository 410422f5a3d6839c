"""The candidate-list interval resolution (csrc/render.cu: cand_sort_kernel
ordering + cand_next_interval with its dead-prefix hint, 4-slot window and
early exits on the stored next-group key), restated in Python, produces exactly next_interval's sequence
(K:173-230: skip the excluded id and exits <= t_min + excl, winner = min of
(max(entry, t_min), pid)) over random candidate sets with overlapping boxes,
equal entries, degenerate intervals and the trace's t_min = b - eps updates
(K:390-391).  CPU only: this pins the algorithm; the GPU tests pin the kernels."""

import math

import numpy as np
import pytest


def f32_rd(x: float) -> float:
    """__double2float_rd: round toward -inf to float32."""
    f = float(np.float32(x))
    if f > x:
        f = float(np.nextafter(np.float32(f), np.float32(-np.inf)))
    return f


def next_interval_ref(cands, t_min, excl, last):
    thr = t_min + excl
    best, best_a, best_b = -1, math.inf, math.inf
    for pa, pb, pid in cands:
        if pid == last or pb <= thr:
            continue
        a_cl = pa if pa > t_min else t_min
        if a_cl >= math.inf:
            continue
        if a_cl < best_a or (a_cl == best_a and pid < best):
            best, best_a, best_b = pid, a_cl, pb
    return best, best_a, best_b


class Resolver:
    """cand_next_interval over the slots as cand_sort_kernel orders them."""

    def __init__(self, cands):
        keyed = sorted(range(len(cands)), key=lambda i: (f32_rd(cands[i][0]), i))
        self.slots = [cands[i] for i in keyed]
        self.n = len(cands)
        self.dead, self.dead_thr = 0, -math.inf
        self.win_base, self.win = None, None
        self.loads = 0

    def group(self, i0):
        if self.win_base != i0:
            self.win_base = i0
            self.win = [self.slots[i] if i < self.n else (0.0, -math.inf, -1) for i in range(i0, i0 + 4)]
            self.loads += 1
        return self.win

    def next(self, t_min, excl, last):
        thr = t_min + excl
        best, best_a, best_b = -1, math.inf, math.inf
        if thr < self.dead_thr:
            self.dead = 0
        self.dead_thr = thr
        prefix = True
        i0 = self.dead & ~3
        while i0 < self.n:
            g = self.group(i0)
            if f32_rd(g[0][0]) > best_a:
                break
            for u, (pa, pb, pid) in enumerate(g):
                if pb <= thr:
                    if prefix and i0 + u + 1 > self.dead:
                        self.dead = min(i0 + u + 1, self.n)
                    continue
                prefix = False
                if pid == last:
                    continue
                a_cl = pa if pa > t_min else t_min
                if a_cl >= math.inf:
                    continue
                if a_cl < best_a or (a_cl == best_a and pid < best):
                    best, best_a, best_b = pid, a_cl, pb
            # the next group's first key is stored with this group's last slot
            if i0 + 4 < self.n and f32_rd(self.slots[i0 + 4][0]) > best_a:
                break
            i0 += 4
        return best, best_a, best_b


def walk(step_fn, eps):
    """The trace's interval loop (K:360-391) with a given next_interval."""
    out, t_min, last = [], 0.0, -1
    for _ in range(200):
        excl = 0.0 if last < 0 else eps
        pid, a, b = step_fn(t_min, excl, last)
        if pid < 0:
            break
        out.append((pid, a, b))
        t_min = b - eps
        last = pid
    return out


def random_cands(rng, n, kind):
    if kind == "tiled":      # partition boxes tiling the ray: exits = next entries
        cuts = np.sort(rng.uniform(0.0, 50.0, n + 1))
        pa, pb = cuts[:-1], cuts[1:]
    elif kind == "overlap":  # refined boxes overlapping their neighbours
        c = np.sort(rng.uniform(0.0, 50.0, n))
        w = rng.exponential(2.0, n)
        pa, pb = c - w * rng.uniform(0, 1, n), c + w
    else:                    # ties, degenerate and behind-the-origin entries
        pa = np.round(rng.uniform(-5.0, 30.0, n), 1)
        pb = pa + np.round(rng.exponential(1.0, n), 1)
        deg = rng.uniform(size=n) < 0.1
        pb[deg] = pa[deg]   # zero-length boxes along the ray
    pid = rng.permutation(4 * n + 3)[:n]
    keep = pb > 0.0          # the raster keeps exits > 0
    return [(float(a), float(b), int(p)) for a, b, p, k in zip(pa, pb, pid, keep) if k and a <= b]


@pytest.mark.parametrize("kind", ["tiled", "overlap", "ties"])
def test_candidate_resolution_equals_next_interval(kind):
    rng = np.random.default_rng({"tiled": 1, "overlap": 2, "ties": 3}[kind])
    total_loads = total_steps = 0
    for trial in range(400):
        n = int(rng.integers(0, 49))
        cands = random_cands(rng, n, kind)
        eps = float(rng.choice([1e-4, 1e-3, 0.05, 0.3]))
        want = walk(lambda t, e, l: next_interval_ref(cands, t, e, l), eps)
        r = Resolver(cands)
        got = walk(r.next, eps)
        assert got == want, (kind, trial)
        total_loads += r.loads
        total_steps += len(got)
    if kind == "tiled" and total_steps:
        # the register window serves most steps: about one 4-slot load per
        # 3-4 intervals
        assert total_loads < 0.35 * total_steps
