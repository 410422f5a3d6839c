// host_build.cpp -- native host-side producers of the device-resident scene.
//
// These replace the reference's Python scene-build steps whose outputs feed
// the hot path:
//   * KD partitions            partitions.py:73-128  (exact semantics, ids in DFS order)
//   * point-location BVH       mesh.py:246-250, bvh.py:41-98 (own design: BVH2,
//                              cube-preserving splits, exclusive leaf boxes)
//   * partition BVH            traversal.py:82-91 (own design: BVH2, f64 boxes)
//   * TF partition metadata    transfer.py:95-141 (numpy reduction order reproduced)
//   * adaptive step sizes      _kernels.py:20-22 (glibc pow, bit-identical)
//   * tet record packing       mesh.py:251-254 arrays -> 128 B records
#include <algorithm>
#include <array>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "glibc_pow.cuh"
#include "tetray_b200.h"
#include "tr_internal.h"

struct TrHostBuf {
    virtual ~TrHostBuf() {}
};

namespace {

// ------------------------------------------------------------ float rounding
inline float f32_down(double x) {
    float f = (float)x;
    if ((double)f > x) f = std::nextafter(f, -INFINITY);
    return f;
}
inline float f32_up(double x) {
    float f = (float)x;
    if ((double)f < x) f = std::nextafter(f, INFINITY);
    return f;
}

// ============================================================ KD partitions
struct KdBuf : TrHostBuf {
    std::vector<int64_t> offsets{0};
    std::vector<int64_t> ids;
    std::vector<double> leaf_lo, leaf_hi, lo, hi, vrange;
};

struct KdCtx {
    const double *V;
    const int64_t *tets;
    int64_t max_leaf, max_depth;
    std::vector<double> blo, bhi, cen;  // (T,3) tet boxes and centroids
    std::vector<double> emin, emax;     // per-element value range
    KdBuf *out;
};

// np.median of vals (partitions.py:105): odd n -> middle, even n -> (a+b)/2.
double np_median(std::vector<double> &v) {
    size_t n = v.size(), k = n / 2;
    std::nth_element(v.begin(), v.begin() + k, v.end());
    double b = v[k];
    if (n % 2 == 1) return b;
    double a = *std::max_element(v.begin(), v.begin() + k);
    return (a + b) / 2.0;
}

void kd_emit(KdCtx &C, std::vector<int64_t> &ids, const double *nlo, const double *nhi) {
    // partitions.py:88-97: sorted ids, value range, bounds refined to the
    // box of the contained elements' vertices intersected with the leaf box.
    std::sort(ids.begin(), ids.end());
    KdBuf &O = *C.out;
    double vmin = INFINITY, vmax = -INFINITY;
    double plo[3] = {INFINITY, INFINITY, INFINITY}, phi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t t : ids) {
        vmin = std::min(vmin, C.emin[t]);
        vmax = std::max(vmax, C.emax[t]);
        for (int a = 0; a < 3; ++a) {
            plo[a] = std::min(plo[a], C.blo[3 * t + a]);
            phi[a] = std::max(phi[a], C.bhi[3 * t + a]);
        }
    }
    for (int a = 0; a < 3; ++a) {
        O.leaf_lo.push_back(nlo[a]);
        O.leaf_hi.push_back(nhi[a]);
        O.lo.push_back(std::max(plo[a], nlo[a]));
        O.hi.push_back(std::min(phi[a], nhi[a]));
    }
    O.vrange.push_back(vmin);
    O.vrange.push_back(vmax);
    O.ids.insert(O.ids.end(), ids.begin(), ids.end());
    O.offsets.push_back((int64_t)O.ids.size());
}

void kd_split(KdCtx &C, std::vector<int64_t> ids, const double *nlo, const double *nhi,
              int64_t depth) {
    const int64_t n = (int64_t)ids.size();
    if (n <= C.max_leaf || depth >= C.max_depth) {
        kd_emit(C, ids, nlo, nhi);
        return;
    }
    // np.argmax: first longest node axis
    int axis = 0;
    double ext = nhi[0] - nlo[0];
    for (int a = 1; a < 3; ++a)
        if (nhi[a] - nlo[a] > ext) { ext = nhi[a] - nlo[a]; axis = a; }
    std::vector<double> vals(n);
    for (int64_t i = 0; i < n; ++i) vals[i] = C.cen[3 * ids[i] + axis];
    const double m = np_median(vals);
    std::vector<int64_t> left, right, flat;
    left.reserve(n / 2 + 16);
    right.reserve(n / 2 + 16);
    for (int64_t t : ids) {
        bool l = C.blo[3 * t + axis] < m, r = C.bhi[3 * t + axis] > m;
        if (l) left.push_back(t);
        if (r) right.push_back(t);
        if (!l && !r) flat.push_back(t);  // flat on the plane -> right (closed) side
    }
    if (!flat.empty()) {
        std::vector<int64_t> merged(right.size() + flat.size());
        std::merge(right.begin(), right.end(), flat.begin(), flat.end(), merged.begin());
        right.swap(merged);
    }
    if (((int64_t)left.size() == n && (int64_t)right.size() == n) || left.empty() ||
        right.empty()) {
        kd_emit(C, ids, nlo, nhi);
        return;
    }
    std::vector<int64_t>().swap(ids);
    double lhi[3] = {nhi[0], nhi[1], nhi[2]}, rlo[3] = {nlo[0], nlo[1], nlo[2]};
    lhi[axis] = m;
    rlo[axis] = m;
    kd_split(C, std::move(left), nlo, lhi, depth + 1);
    kd_split(C, std::move(right), rlo, nhi, depth + 1);
}

// ------------------------------------------- KD partitions of a cube grid
// The same KD build (kd_split above, partitions.py:73-128) evaluated in closed
// form on the synthetic generator's mesh (mesh.py:147-231): N^3 unit cubes,
// five tets per cube, every tet spanning its whole cube on each axis, and
// per axis the five centroids of a cube at offsets {.25, .25, .5, .75, .75}
// (for both cube parities).  A node's elements are therefore always all tets
// of an integer cube range, np.median is a closed form over those offsets,
// the straddle tests split the range at the median (integer median: disjoint
// halves; otherwise the median's cube slab goes to both sides), and the
// value range is the field at the range's extreme vertices (the f32-rounded
// field is monotone in the vertex distance).  tests/test_grid_scene.py checks
// it against kd_split on generated meshes.
struct GridKdCtx {
    int64_t n;
    int32_t field;  // 0 ramp (x), 1 radial (|p - n/2|)
    int64_t max_leaf, max_depth;
    bool with_ids;
    KdBuf *out;
};

double grid_field(const GridKdCtx &C, const double p[3]) {
    if (C.field == 0) return (double)(float)p[0];
    const double h = (double)C.n / 2.0;  // mesh.py _radial: p - n / 2.0
    const double d0 = p[0] - h, d1 = p[1] - h, d2 = p[2] - h;
    return (double)(float)std::sqrt((d0 * d0 + d1 * d1) + d2 * d2);
}

void gkd_emit(GridKdCtx &C, const int64_t r0[3], const int64_t r1[3], const double *nlo,
              const double *nhi) {
    KdBuf &O = *C.out;
    const int64_t n = C.n;
    if (C.with_ids) {
        std::vector<int64_t> ids;
        for (int64_t x = r0[0]; x <= r1[0]; ++x)
            for (int64_t y = r0[1]; y <= r1[1]; ++y)
                for (int64_t z = r0[2]; z <= r1[2]; ++z) {
                    const int64_t c = (x * n + y) * n + z;
                    for (int k = 0; k < 5; ++k) ids.push_back(5 * c + k);
                }
        O.ids.insert(O.ids.end(), ids.begin(), ids.end());
    }
    const int64_t cnt = 5 * (r1[0] - r0[0] + 1) * (r1[1] - r0[1] + 1) * (r1[2] - r0[2] + 1);
    O.offsets.push_back(O.offsets.back() + cnt);
    // extreme vertices of [r0, r1 + 1]: nearest to / farthest from the field's minimum
    double pmin[3], pmax[3];
    for (int a = 0; a < 3; ++a) {
        const double lo = (double)r0[a], hi = (double)(r1[a] + 1);
        if (C.field == 0) { pmin[a] = lo; pmax[a] = (a == 0) ? hi : lo; continue; }
        const double h = (double)C.n / 2.0;
        const double cl = std::min(std::max(h, lo), hi);     // nearest real coordinate
        const double f = std::floor(cl), c = std::ceil(cl);  // nearest vertex coordinate
        pmin[a] = (cl - f <= c - cl) ? f : c;
        pmax[a] = (h - lo >= hi - h) ? lo : hi;
    }
    O.vrange.push_back(grid_field(C, pmin));
    O.vrange.push_back(grid_field(C, pmax));
    for (int a = 0; a < 3; ++a) {
        O.leaf_lo.push_back(nlo[a]);
        O.leaf_hi.push_back(nhi[a]);
        O.lo.push_back(std::max((double)r0[a], nlo[a]));
        O.hi.push_back(std::min((double)(r1[a] + 1), nhi[a]));
    }
}

void gkd_split(GridKdCtx &C, const int64_t r0[3], const int64_t r1[3], const double *nlo,
               const double *nhi, int64_t depth) {
    int64_t cnt[3];
    for (int a = 0; a < 3; ++a) cnt[a] = r1[a] - r0[a] + 1;
    const int64_t n = 5 * cnt[0] * cnt[1] * cnt[2];
    if (n <= C.max_leaf || depth >= C.max_depth) { gkd_emit(C, r0, r1, nlo, nhi); return; }
    int axis = 0;
    double ext = nhi[0] - nlo[0];
    for (int a = 1; a < 3; ++a)
        if (nhi[a] - nlo[a] > ext) { ext = nhi[a] - nlo[a]; axis = a; }
    // sorted centroid coordinates on `axis`: slab s holds 2S values at
    // u+.25, S at u+.5, 2S at u+.75 (S = 5-tet cubes per slab / 1)
    const int64_t S = n / (5 * cnt[axis]);
    auto val = [&](int64_t pos) {
        const int64_t s = pos / (5 * S), r = pos % (5 * S);
        const double off = (r < 2 * S) ? 0.25 : ((r < 3 * S) ? 0.5 : 0.75);
        return (double)(r0[axis] + s) + off;
    };
    const int64_t k = n / 2;
    const double m = (n % 2) ? val(k) : (val(k - 1) + val(k)) / 2.0;  // np.median
    // left: blo = u < m; right: bhi = u + 1 > m (no element is flat on m)
    const double fm = std::floor(m);
    const int64_t lmax = (fm == m) ? (int64_t)m - 1 : (int64_t)fm;
    const int64_t rmin = (int64_t)fm;
    const bool left_empty = lmax < r0[axis], right_empty = rmin > r1[axis];
    const bool both_full = lmax >= r1[axis] && rmin <= r0[axis];
    if (left_empty || right_empty || both_full) { gkd_emit(C, r0, r1, nlo, nhi); return; }
    int64_t l1[3] = {r1[0], r1[1], r1[2]}, q0[3] = {r0[0], r0[1], r0[2]};
    l1[axis] = std::min(r1[axis], lmax);
    q0[axis] = std::max(r0[axis], rmin);
    double lhi[3] = {nhi[0], nhi[1], nhi[2]}, rlo[3] = {nlo[0], nlo[1], nlo[2]};
    lhi[axis] = m;
    rlo[axis] = m;
    gkd_split(C, r0, l1, nlo, lhi, depth + 1);
    gkd_split(C, q0, r1, rlo, nhi, depth + 1);
}

// ====================================================== point-location BVH
struct PBuf : TrHostBuf {
    std::vector<TrPNode> nodes;
    std::vector<TrPLeaf> leaves;
    std::vector<uint32_t> ids;
    std::vector<std::array<double, 6>> leaf_box;  // exact f64 union boxes
    // uniform grid of leaf candidates (a hint only: the exclusive box proves it)
    std::vector<int32_t> grid;
    int32_t gdim[3] = {1, 1, 1};
    double gorg[3] = {0, 0, 0}, gscale[3] = {1, 1, 1};
    double coverage = 0.0;   // mean fraction of a cell covered by its candidate's exclusive box
};

constexpr int32_t CHILD_NONE = INT32_MIN;

struct PRef {
    int32_t child;
    uint32_t minid;
    double lo[3], hi[3];
};

struct PCtx {
    const double *lo, *hi;
    std::vector<double> key;  // box centres
    std::vector<uint32_t> idx;
    int leaf_max;
    PBuf *out;
};

PRef p_make_leaf(PCtx &C, PBuf &O, int64_t b, int64_t e) {
    std::sort(C.idx.begin() + b, C.idx.begin() + e);
    TrPLeaf L{};
    L.start = (uint32_t)O.ids.size();
    L.count = (uint32_t)(e - b);
    PRef r;
    for (int a = 0; a < 3; ++a) { r.lo[a] = INFINITY; r.hi[a] = -INFINITY; }
    for (int64_t k = b; k < e; ++k) {
        uint32_t t = C.idx[k];
        O.ids.push_back(t);
        for (int a = 0; a < 3; ++a) {
            r.lo[a] = std::min(r.lo[a], C.lo[3 * (size_t)t + a]);
            r.hi[a] = std::max(r.hi[a], C.hi[3 * (size_t)t + a]);
        }
    }
    for (int a = 0; a < 3; ++a) { L.ex_lo[a] = 1.0f; L.ex_hi[a] = 0.0f; }  // filled later
    O.leaves.push_back(L);
    O.leaf_box.push_back({r.lo[0], r.lo[1], r.lo[2], r.hi[0], r.hi[1], r.hi[2]});
    r.child = ~(int32_t)(O.leaves.size() - 1);
    r.minid = C.idx[b];
    return r;
}

void p_set_child(TrPNode &N, int c, const PRef &r) {
    float *lo = c == 0 ? N.lo0 : N.lo1, *hi = c == 0 ? N.hi0 : N.hi1;
    for (int a = 0; a < 3; ++a) { lo[a] = f32_down(r.lo[a]); hi[a] = f32_up(r.hi[a]); }
    N.child[c] = r.child;
    N.minid[c] = r.minid;
}

// Split position for [b, e): the object median on the axis of largest centre
// extent, moved to the nearest change of key (three-way partition) so boxes
// with equal centres never straddle a split.  -1: no split possible.
int64_t p_choose_split(PCtx &C, int64_t b, int64_t e);

PRef p_build(PCtx &C, PBuf &O, int64_t b, int64_t e) {
    const int64_t n = e - b;
    if (n <= C.leaf_max) return p_make_leaf(C, O, b, e);
    int64_t split = p_choose_split(C, b, e);
    if (split < 0) {
        if (n <= 64) return p_make_leaf(C, O, b, e);
        split = b + n / 2;  // identical centres everywhere: force a split
    }
    const size_t ni = O.nodes.size();
    O.nodes.push_back(TrPNode{});
    PRef l = p_build(C, O, b, split);
    PRef r = p_build(C, O, split, e);
    TrPNode &N = O.nodes[ni];
    p_set_child(N, 0, l);
    p_set_child(N, 1, r);
    PRef me;
    me.child = (int32_t)ni;
    me.minid = std::min(l.minid, r.minid);
    for (int a = 0; a < 3; ++a) { me.lo[a] = std::min(l.lo[a], r.lo[a]); me.hi[a] = std::max(l.hi[a], r.hi[a]); }
    return me;
}

// Append subtree buffer S (built separately) to O, relocating node, leaf and
// id indices; returns the relocated reference to its root.
PRef p_splice(PBuf &O, PBuf &S, PRef r) {
    const int32_t node_off = (int32_t)O.nodes.size(), leaf_off = (int32_t)O.leaves.size();
    const uint32_t id_off = (uint32_t)O.ids.size();
    for (TrPNode N : S.nodes) {
        for (int c = 0; c < 2; ++c) {
            if (N.child[c] >= 0) N.child[c] += node_off;
            else if (N.child[c] != CHILD_NONE) N.child[c] = ~(~N.child[c] + leaf_off);
        }
        O.nodes.push_back(N);
    }
    for (TrPLeaf L : S.leaves) { L.start += id_off; O.leaves.push_back(L); }
    O.leaf_box.insert(O.leaf_box.end(), S.leaf_box.begin(), S.leaf_box.end());
    O.ids.insert(O.ids.end(), S.ids.begin(), S.ids.end());
    PBuf().nodes.swap(S.nodes);
    if (r.child >= 0) r.child += node_off;
    else r.child = ~(~r.child + leaf_off);
    return r;
}

// Task-parallel top levels (disjoint index ranges), sequential below.
PRef p_build_par(PCtx &C, PBuf &O, int64_t b, int64_t e, int depth) {
    const int64_t n = e - b;
    if (n < (int64_t)(1 << 18) || depth >= 10) return p_build(C, O, b, e);
    const int64_t split = p_choose_split(C, b, e);
    if (split < 0) return p_build(C, O, b, e);
    const size_t ni = O.nodes.size();
    O.nodes.push_back(TrPNode{});
    PBuf Lb, Rb;
    PRef l, r;
#pragma omp task shared(C, Lb, l)
    l = p_build_par(C, Lb, b, split, depth + 1);
#pragma omp task shared(C, Rb, r)
    r = p_build_par(C, Rb, split, e, depth + 1);
#pragma omp taskwait
    l = p_splice(O, Lb, l);
    r = p_splice(O, Rb, r);
    TrPNode &N = O.nodes[ni];
    p_set_child(N, 0, l);
    p_set_child(N, 1, r);
    PRef me;
    me.child = (int32_t)ni;
    me.minid = std::min(l.minid, r.minid);
    for (int a = 0; a < 3; ++a) { me.lo[a] = std::min(l.lo[a], r.lo[a]); me.hi[a] = std::max(l.hi[a], r.hi[a]); }
    return me;
}

int64_t p_choose_split(PCtx &C, int64_t b, int64_t e) {
    const int64_t n = e - b;
    double klo[3] = {INFINITY, INFINITY, INFINITY}, khi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t k = b; k < e; ++k)
        for (int a = 0; a < 3; ++a) {
            double v = C.key[3 * (size_t)C.idx[k] + a];
            klo[a] = std::min(klo[a], v);
            khi[a] = std::max(khi[a], v);
        }
    int order[3] = {0, 1, 2};
    std::sort(order, order + 3, [&](int x, int y) { return khi[x] - klo[x] > khi[y] - klo[y]; });
    int64_t split = -1;
    for (int oi = 0; oi < 3 && split < 0; ++oi) {
        int a = order[oi];
        if (!(khi[a] > klo[a])) continue;
        auto key = [&](uint32_t t) { return C.key[3 * (size_t)t + a]; };
        int64_t mid = b + n / 2;
        std::nth_element(C.idx.begin() + b, C.idx.begin() + mid, C.idx.begin() + e,
                         [&](uint32_t x, uint32_t y) { return key(x) < key(y) || (key(x) == key(y) && x < y); });
        double v = key(C.idx[mid]);
        // three-way partition so boxes with equal centres (e.g. the 5 tets of
        // one cube) never straddle a split
        auto p1 = std::partition(C.idx.begin() + b, C.idx.begin() + e, [&](uint32_t t) { return key(t) < v; });
        auto p2 = std::partition(p1, C.idx.begin() + e, [&](uint32_t t) { return key(t) == v; });
        int64_t s1 = p1 - C.idx.begin(), s2 = p2 - C.idx.begin();
        int64_t best = -1;
        for (int64_t s : {s1, s2})
            if (s > b && s < e && (best < 0 || std::llabs(s - mid) < std::llabs(best - mid))) best = s;
        split = best;
    }
    return split;
}

inline bool boxes_meet(const double *a, const double *b) {  // closed boxes [lo(3), hi(3)]
    for (int k = 0; k < 3; ++k)
        if (a[k] > b[3 + k] || b[k] > a[3 + k]) return false;
    return true;
}

// Exclusive box of every leaf: its box minus (greedy axis cuts) every other
// leaf box that meets it.  Rounded inward to f32 and tested with strict
// inequalities, a point inside it lies in no other leaf's box.
void p_exclusive_boxes(PBuf &O) {
    const int64_t nl = (int64_t)O.leaves.size();
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t L = 0; L < nl; ++L) {
        const double *B = O.leaf_box[L].data();
        double E[6];
        std::memcpy(E, B, sizeof E);
        int32_t stack[128];
        int sp = 0;
        stack[sp++] = 0;
        while (sp > 0) {
            const TrPNode &N = O.nodes[stack[--sp]];
            for (int c = 0; c < 2; ++c) {
                int32_t ch = N.child[c];
                if (ch == CHILD_NONE) continue;
                const float *lo = c == 0 ? N.lo0 : N.lo1, *hi = c == 0 ? N.hi0 : N.hi1;
                double cb[6] = {lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]};
                if (!boxes_meet(cb, B)) continue;
                if (ch >= 0) { stack[sp++] = ch; continue; }
                int64_t M = ~ch;
                if (M == L) continue;
                const double *Mb = O.leaf_box[M].data();
                if (!boxes_meet(Mb, E)) continue;
                // candidate cuts: keep the part of E below Mb.lo[a] or above Mb.hi[a]
                double best_vol = -1.0, cut_val = 0.0;
                int cut_axis = -1, cut_side = 0;
                for (int a = 0; a < 3; ++a) {
                    for (int side = 0; side < 2; ++side) {
                        double nlo = E[a], nhi = E[3 + a];
                        if (side == 0) { if (!(Mb[a] > E[a])) continue; nhi = Mb[a]; }
                        else { if (!(Mb[3 + a] < E[3 + a])) continue; nlo = Mb[3 + a]; }
                        double vol = 1.0;
                        for (int q = 0; q < 3; ++q) {
                            double lo_q = q == a ? nlo : E[q], hi_q = q == a ? nhi : E[3 + q];
                            vol *= std::max(0.0, hi_q - lo_q);
                        }
                        if (vol > best_vol) { best_vol = vol; cut_axis = a; cut_side = side; cut_val = side == 0 ? nhi : nlo; }
                    }
                }
                if (cut_axis < 0) {  // Mb covers E: nothing exclusive is left
                    E[0] = 1.0; E[3] = 0.0;
                    sp = 0;
                    break;
                }
                if (cut_side == 0) E[3 + cut_axis] = cut_val; else E[cut_axis] = cut_val;
            }
        }
        TrPLeaf &LF = O.leaves[L];
        for (int a = 0; a < 3; ++a) {
            LF.ex_lo[a] = f32_up(E[a]);
            LF.ex_hi[a] = f32_down(E[3 + a]);
        }
        if (!(E[0] <= E[3])) { LF.ex_lo[0] = 1.0f; LF.ex_hi[0] = 0.0f; }
    }
}

// Uniform grid over the leaves: each cell names the leaf whose exclusive box
// covers most of it.  Sized for about one leaf per cell.
void p_build_grid(PBuf &O) {
    const int64_t nl = (int64_t)O.leaves.size();
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (const auto &b : O.leaf_box)
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], b[a]); hi[a] = std::max(hi[a], b[3 + a]); }
    double ext[3], vol = 1.0;
    for (int a = 0; a < 3; ++a) { ext[a] = std::max(hi[a] - lo[a], 1e-300); vol *= ext[a]; }
    const double side = std::cbrt(vol / (double)std::max<int64_t>(nl, 1));
    int64_t cells = 1;
    for (int a = 0; a < 3; ++a) {
        // rounded, not ceiled: leaves of a regular mesh (one cube each) then
        // get one cell each instead of cells straddling two leaves
        double d = std::round(ext[a] / side);
        O.gdim[a] = (int32_t)std::min(std::max(d, 1.0), 2048.0);
        cells *= O.gdim[a];
        O.gorg[a] = lo[a];
        O.gscale[a] = (double)O.gdim[a] / ext[a];
    }
    O.grid.assign((size_t)cells, -1);
    std::vector<double> best((size_t)cells, 0.0);
    for (int64_t L = 0; L < nl; ++L) {
        const TrPLeaf &lf = O.leaves[L];
        double e0[3], e1[3];
        bool ok = true;
        for (int a = 0; a < 3; ++a) {
            e0[a] = lf.ex_lo[a];
            e1[a] = lf.ex_hi[a];
            ok = ok && e0[a] < e1[a];
        }
        if (!ok) continue;
        int64_t c0[3], c1[3];
        for (int a = 0; a < 3; ++a) {
            c0[a] = std::min<int64_t>(std::max<int64_t>((int64_t)std::floor((e0[a] - O.gorg[a]) * O.gscale[a]), 0), O.gdim[a] - 1);
            c1[a] = std::min<int64_t>(std::max<int64_t>((int64_t)std::floor((e1[a] - O.gorg[a]) * O.gscale[a]), 0), O.gdim[a] - 1);
        }
        for (int64_t x = c0[0]; x <= c1[0]; ++x)
            for (int64_t y = c0[1]; y <= c1[1]; ++y)
                for (int64_t z = c0[2]; z <= c1[2]; ++z) {
                    const int64_t c[3] = {x, y, z};
                    double ov = 1.0;
                    for (int a = 0; a < 3; ++a) {
                        double cl = O.gorg[a] + (double)c[a] / O.gscale[a];
                        double ch = O.gorg[a] + (double)(c[a] + 1) / O.gscale[a];
                        ov *= std::max(0.0, std::min(e1[a], ch) - std::max(e0[a], cl));
                    }
                    const size_t ci = (size_t)((x * O.gdim[1] + y) * O.gdim[2] + z);
                    if (ov > best[ci]) { best[ci] = ov; O.grid[ci] = (int32_t)L; }
                }
    }
    double cell_vol = 1.0, cov = 0.0;
    for (int a = 0; a < 3; ++a) cell_vol /= O.gscale[a];
    for (double b : best) cov += std::min(b / cell_vol, 1.0);
    O.coverage = cells > 0 ? cov / (double)cells : 0.0;
}

// ------------------------------------------------ cell candidate lists
// For meshes whose leaves do not line up with the grid (unstructured tets:
// leaf boxes overlap, exclusive boxes shrink), the exact fallback per point
// is a finer uniform grid whose cell lists EVERY record whose padded tet box
// (mesh.py:248-250) meets the cell, in ascending tet id: a point's lowest-id
// containing tet is the first accepting entry (the padded box of a tet that
// accepts the point contains it, K:100-101).  Cell ranges use the kernel's
// own expression floor((x - org) * scale) on the box corners, which is
// monotone, so the lists are conservative.  Cells above max_list entries
// are marked (offset high bit) and the kernel uses the BVH descent there.
struct CBuf : TrHostBuf {
    int32_t dim[3] = {1, 1, 1};
    double org[3] = {0, 0, 0}, scale[3] = {1, 1, 1};
    std::vector<uint32_t> off;    // n_cells + 1; bit 31 of off[c]: overflowed cell
    std::vector<uint32_t> recs;   // record positions
    std::vector<float> tbox;      // 8 floats per record: padded box rounded outward, pad
};

// ============================================================ partition BVH
struct BBuf : TrHostBuf {
    std::vector<TrBNode> nodes;
};

struct BRef {
    int32_t child;
    double lo[3], hi[3];
};

BRef b_build(BBuf &O, const double *lo, const double *hi, std::vector<int32_t> &idx, int64_t b,
             int64_t e) {
    if (e - b == 1) {
        BRef r;
        r.child = ~idx[b];
        for (int a = 0; a < 3; ++a) { r.lo[a] = lo[3 * idx[b] + a]; r.hi[a] = hi[3 * idx[b] + a]; }
        return r;
    }
    double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t k = b; k < e; ++k)
        for (int a = 0; a < 3; ++a) {
            double c = 0.5 * (lo[3 * idx[k] + a] + hi[3 * idx[k] + a]);
            clo[a] = std::min(clo[a], c);
            chi[a] = std::max(chi[a], c);
        }
    int axis = 0;
    for (int a = 1; a < 3; ++a)
        if (chi[a] - clo[a] > chi[axis] - clo[axis]) axis = a;
    int64_t mid = b + (e - b) / 2;
    std::nth_element(idx.begin() + b, idx.begin() + mid, idx.begin() + e, [&](int32_t x, int32_t y) {
        double cx = lo[3 * x + axis] + hi[3 * x + axis], cy = lo[3 * y + axis] + hi[3 * y + axis];
        return cx < cy || (cx == cy && x < y);
    });
    size_t ni = O.nodes.size();
    O.nodes.push_back(TrBNode{});
    BRef l = b_build(O, lo, hi, idx, b, mid);
    BRef r = b_build(O, lo, hi, idx, mid, e);
    TrBNode &N = O.nodes[ni];
    const BRef *cs[2] = {&l, &r};
    BRef me;
    me.child = (int32_t)ni;
    for (int a = 0; a < 3; ++a) { me.lo[a] = INFINITY; me.hi[a] = -INFINITY; }
    for (int c = 0; c < 2; ++c) {
        N.child[c] = cs[c]->child;
        for (int a = 0; a < 3; ++a) {
            N.box[c][a] = cs[c]->lo[a];
            N.box[c][3 + a] = cs[c]->hi[a];
            me.lo[a] = std::min(me.lo[a], cs[c]->lo[a]);
            me.hi[a] = std::max(me.hi[a], cs[c]->hi[a]);
        }
    }
    return me;
}

// ====================================================== partition BSP tree
// Axis-aligned BSP over the partition boxes, built by greedy separating cuts
// (for KD-derived partitions the original split planes always separate).
// A set that no plane separates becomes one multi-partition leaf.
struct KBuf : TrHostBuf {
    std::vector<TrKNode> nodes;
    std::vector<int32_t> leaf_pids;
    double root_lo[3], root_hi[3];
};

int32_t k_build(KBuf &O, const double *lo, const double *hi, std::vector<int32_t> &ids, int depth) {
    const int32_t me = (int32_t)O.nodes.size();
    O.nodes.push_back(TrKNode{});
    const int64_t n = (int64_t)ids.size();
    int best_axis = -1;
    int64_t best_i = -1, best_bal = INT64_MAX;
    double best_s = 0.0;
    if (n > 1 && depth < 60) {
        std::vector<int32_t> ord(ids);
        for (int a = 0; a < 3; ++a) {
            std::sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
                const double lx = lo[3 * x + a], ly = lo[3 * y + a];
                return lx < ly || (lx == ly && x < y);
            });
            double pref = -INFINITY;
            for (int64_t i = 1; i < n; ++i) {
                pref = std::max(pref, hi[3 * ord[i - 1] + a]);
                const double l = lo[3 * ord[i] + a];
                if (pref <= l) {
                    const int64_t bal = std::llabs(2 * i - n);
                    if (bal < best_bal) { best_bal = bal; best_i = i; best_axis = a; best_s = l; }
                }
            }
        }
    }
    if (best_axis < 0) {  // leaf (one partition, or boxes no plane separates)
        O.nodes[me].info = ~(int32_t)O.leaf_pids.size();
        O.nodes[me].aux = (int32_t)n;
        O.nodes[me].split = 0.0;
        std::sort(ids.begin(), ids.end());
        O.leaf_pids.insert(O.leaf_pids.end(), ids.begin(), ids.end());
        return me;
    }
    // members split exactly as the winning sweep did: the first best_i by (lo, id)
    std::vector<int32_t> L, R;
    {
        std::vector<int32_t> ord(ids);
        const int a = best_axis;
        std::sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
            const double lx = lo[3 * x + a], ly = lo[3 * y + a];
            return lx < ly || (lx == ly && x < y);
        });
        L.assign(ord.begin(), ord.begin() + best_i);
        R.assign(ord.begin() + best_i, ord.end());
    }
    std::vector<int32_t>().swap(ids);
    O.nodes[me].split = best_s;
    O.nodes[me].aux = 0;
    k_build(O, lo, hi, L, depth + 1);  // left child = me + 1 (pre-order)
    const int32_t r = k_build(O, lo, hi, R, depth + 1);
    O.nodes[me].info = (r << 2) | best_axis;
    return me;
}

// ============================================================ TF metadata
// numpy's pairwise summation of a contiguous float64 vector (add.reduce).
double np_pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

void tf_lookup(const double *T, int64_t n, double lo, double hi, double v, double *rgba) {
    tr_tf_sample_host(T, n, lo, hi, v, rgba);
}

}  // namespace

// Shared with the device code's host-side checks: K:74-90 on the host.
void tr_tf_sample_host(const double *T, int64_t n, double lo, double hi, double v, double *rgba) {
    double u = (v - lo) / (hi - lo) * (double)(n - 1);
    if (u <= 0.0) { std::memcpy(rgba, T, 32); return; }
    if (u >= (double)(n - 1)) { std::memcpy(rgba, T + 4 * (n - 1), 32); return; }
    int64_t j = (int64_t)std::floor(u);
    double f = u - (double)j;
    for (int c = 0; c < 4; ++c) rgba[c] = T[4 * j + c] + f * (T[4 * (j + 1) + c] - T[4 * j + c]);
}

extern "C" {

int tr_kd_build(int64_t n_vertices, const double *vertices, int64_t n_tets, const int64_t *tets,
                const double *field, int32_t centering, const double *mesh_lo,
                const double *mesh_hi, int64_t max_leaf_elements, int64_t max_depth,
                TrHostBuf **out) {
    if (!out || !vertices || !tets || !field || n_tets <= 0 || max_leaf_elements < 1 ||
        max_depth < 1)
        return tr_fail(TR_EINVAL, "tr_kd_build: invalid arguments");
    try {
        KdBuf *K = new KdBuf();
        KdCtx C;
        C.V = vertices;
        C.tets = tets;
        C.max_leaf = max_leaf_elements;
        C.max_depth = max_depth;
        C.out = K;
        C.blo.resize(3 * n_tets);
        C.bhi.resize(3 * n_tets);
        C.cen.resize(3 * n_tets);
        C.emin.resize(n_tets);
        C.emax.resize(n_tets);
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < n_tets; ++t) {
            const int64_t *tv = tets + 4 * t;
            for (int a = 0; a < 3; ++a) {
                double v0 = vertices[3 * tv[0] + a], v1 = vertices[3 * tv[1] + a];
                double v2 = vertices[3 * tv[2] + a], v3 = vertices[3 * tv[3] + a];
                C.blo[3 * t + a] = std::min(std::min(v0, v1), std::min(v2, v3));
                C.bhi[3 * t + a] = std::max(std::max(v0, v1), std::max(v2, v3));
                C.cen[3 * t + a] = (((v0 + v1) + v2) + v3) / 4.0;  // mesh.vertices[tets].mean(axis=1)
            }
            if (centering == 0) {
                double f0 = field[tv[0]], f1 = field[tv[1]], f2 = field[tv[2]], f3 = field[tv[3]];
                C.emin[t] = std::min(std::min(f0, f1), std::min(f2, f3));
                C.emax[t] = std::max(std::max(f0, f1), std::max(f2, f3));
            } else {
                C.emin[t] = C.emax[t] = field[t];
            }
        }
        std::vector<int64_t> all(n_tets);
        for (int64_t t = 0; t < n_tets; ++t) all[t] = t;
        kd_split(C, std::move(all), mesh_lo, mesh_hi, 0);
        *out = K;
        return TR_OK;
    } catch (const std::bad_alloc &) {
        return tr_fail(TR_ENOMEM, "tr_kd_build: out of host memory");
    }
}

int tr_kd_build_grid(int64_t n, int32_t field, int64_t max_leaf_elements, int64_t max_depth,
                     int32_t with_ids, TrHostBuf **out) {
    if (!out || n < 1 || n > (1 << 20) || (field != 0 && field != 1) || max_leaf_elements < 1 ||
        max_depth < 1 || (with_ids && n > 256))
        return tr_fail(TR_EINVAL, "tr_kd_build_grid: invalid arguments");
    try {
        KdBuf *K = new KdBuf();
        GridKdCtx C{n, field, max_leaf_elements, max_depth, with_ids != 0, K};
        const int64_t r0[3] = {0, 0, 0}, r1[3] = {n - 1, n - 1, n - 1};
        const double lo[3] = {0.0, 0.0, 0.0}, hi[3] = {(double)n, (double)n, (double)n};
        gkd_split(C, r0, r1, lo, hi, 0);
        *out = K;
        return TR_OK;
    } catch (const std::bad_alloc &) {
        return tr_fail(TR_ENOMEM, "tr_kd_build_grid: out of host memory");
    }
}

int tr_kd_sizes(const TrHostBuf *b, int64_t *sizes2) {
    auto K = dynamic_cast<const KdBuf *>(b);
    if (!K || !sizes2) return tr_fail(TR_EINVAL, "tr_kd_sizes: not a KD result");
    sizes2[0] = (int64_t)K->offsets.size() - 1;
    sizes2[1] = (int64_t)K->ids.size();
    return TR_OK;
}

int tr_kd_copy(const TrHostBuf *b, int64_t *offsets, int64_t *ids, double *leaf_lo,
               double *leaf_hi, double *lo, double *hi, double *vrange) {
    auto K = dynamic_cast<const KdBuf *>(b);
    if (!K) return tr_fail(TR_EINVAL, "tr_kd_copy: not a KD result");
    auto cp = [](void *dst, const auto &v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(offsets, K->offsets);
    cp(ids, K->ids);
    cp(leaf_lo, K->leaf_lo);
    cp(leaf_hi, K->leaf_hi);
    cp(lo, K->lo);
    cp(hi, K->hi);
    cp(vrange, K->vrange);
    return TR_OK;
}

int tr_pbvh_build(int64_t n_tets, const double *box_lo, const double *box_hi, int32_t leaf_max,
                  TrHostBuf **out) {
    if (!out || n_tets <= 0 || n_tets >= (int64_t)INT32_MAX || leaf_max < 1 || leaf_max > 64)
        return tr_fail(TR_EINVAL, "tr_pbvh_build: invalid arguments");
    try {
        PBuf *O = new PBuf();
        PCtx C;
        C.lo = box_lo;
        C.hi = box_hi;
        C.leaf_max = leaf_max;
        C.out = O;
        C.key.resize(3 * (size_t)n_tets);
        C.idx.resize(n_tets);
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < n_tets; ++t) {
            C.idx[t] = (uint32_t)t;
            for (int a = 0; a < 3; ++a) C.key[3 * t + a] = 0.5 * (box_lo[3 * t + a] + box_hi[3 * t + a]);
        }
        O->nodes.reserve(2 * (size_t)n_tets / 4 + 4);
        PRef root;
#pragma omp parallel
#pragma omp single
        root = p_build_par(C, *O, 0, n_tets, 0);  // an internal root lands at index 0
        if (root.child < 0) {  // whole mesh is one leaf: root node with one child
            TrPNode N{};
            p_set_child(N, 0, root);
            for (int a = 0; a < 3; ++a) { N.lo1[a] = 1.0f; N.hi1[a] = 0.0f; }
            N.child[1] = CHILD_NONE;
            N.minid[1] = UINT32_MAX;
            O->nodes.push_back(N);
        }
        p_exclusive_boxes(*O);
        p_build_grid(*O);
        *out = O;
        return TR_OK;
    } catch (const std::bad_alloc &) {
        return tr_fail(TR_ENOMEM, "tr_pbvh_build: out of host memory");
    }
}

double tr_pbvh_coverage(const TrHostBuf *b) {
    auto P = dynamic_cast<const PBuf *>(b);
    return P ? P->coverage : 0.0;
}

int tr_cells_build(const TrHostBuf *b, const double *box_lo, const double *box_hi, int32_t refine,
                   int32_t max_list, TrHostBuf **out) {
    auto P = dynamic_cast<const PBuf *>(b);
    if (!P || !box_lo || !box_hi || !out || refine < 1 || refine > 8 || max_list < 1)
        return tr_fail(TR_EINVAL, "tr_cells_build: invalid arguments");
    try {
        CBuf *Cb = new CBuf();
        int64_t n_cells = 1;
        for (int a = 0; a < 3; ++a) {
            Cb->dim[a] = (int32_t)std::min<int64_t>((int64_t)P->gdim[a] * refine, 4096);
            Cb->org[a] = P->gorg[a];
            Cb->scale[a] = P->gscale[a] * (double)Cb->dim[a] / (double)P->gdim[a];
            n_cells *= Cb->dim[a];
        }
        const int64_t nrec = (int64_t)P->ids.size();
        auto crange = [&](const double *lo, const double *hi, int64_t c0[3], int64_t c1[3]) {
            for (int a = 0; a < 3; ++a) {
                const double f0 = (lo[a] - Cb->org[a]) * Cb->scale[a], f1 = (hi[a] - Cb->org[a]) * Cb->scale[a];
                c0[a] = std::min<int64_t>(std::max<int64_t>((int64_t)std::floor(f0), 0), Cb->dim[a] - 1);
                c1[a] = std::min<int64_t>(std::max<int64_t>((int64_t)std::floor(f1), 0), Cb->dim[a] - 1);
            }
        };
        std::vector<uint32_t> cnt((size_t)n_cells, 0u);
        for (int64_t k = 0; k < nrec; ++k) {   // pass 1: counts
            const uint32_t t = P->ids[k];
            int64_t c0[3], c1[3];
            crange(box_lo + 3 * (size_t)t, box_hi + 3 * (size_t)t, c0, c1);
            for (int64_t x = c0[0]; x <= c1[0]; ++x)
                for (int64_t y = c0[1]; y <= c1[1]; ++y)
                    for (int64_t z = c0[2]; z <= c1[2]; ++z)
                        ++cnt[(size_t)((x * Cb->dim[1] + y) * Cb->dim[2] + z)];
        }
        Cb->off.assign((size_t)n_cells + 1, 0u);
        uint64_t total = 0;
        for (int64_t c = 0; c < n_cells; ++c) {
            Cb->off[c] = (uint32_t)total;
            if (cnt[c] <= (uint32_t)max_list) total += cnt[c];
            if (total >= 0x7fffffffull) { delete Cb; return tr_fail(TR_ENOMEM, "tr_cells_build: lists too large"); }
        }
        Cb->off[n_cells] = (uint32_t)total;
        Cb->recs.assign((size_t)total, 0u);
        std::vector<uint32_t> fill((size_t)n_cells, 0u);
        for (int64_t k = 0; k < nrec; ++k) {   // pass 2: fill in record order
            const uint32_t t = P->ids[k];
            int64_t c0[3], c1[3];
            crange(box_lo + 3 * (size_t)t, box_hi + 3 * (size_t)t, c0, c1);
            for (int64_t x = c0[0]; x <= c1[0]; ++x)
                for (int64_t y = c0[1]; y <= c1[1]; ++y)
                    for (int64_t z = c0[2]; z <= c1[2]; ++z) {
                        const size_t c = (size_t)((x * Cb->dim[1] + y) * Cb->dim[2] + z);
                        if (cnt[c] <= (uint32_t)max_list) Cb->recs[Cb->off[c] + fill[c]++] = (uint32_t)k;
                    }
        }
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t c = 0; c < n_cells; ++c) {   // ascending tet id within each cell
            if (cnt[c] > (uint32_t)max_list) continue;
            std::sort(Cb->recs.begin() + Cb->off[c], Cb->recs.begin() + Cb->off[c] + cnt[c],
                      [&](uint32_t x, uint32_t y) { return P->ids[x] < P->ids[y]; });
        }
        for (int64_t c = 0; c < n_cells; ++c)
            if (cnt[c] > (uint32_t)max_list) Cb->off[c] |= 0x80000000u;
        Cb->tbox.assign((size_t)nrec * 8, 0.0f);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < nrec; ++k) {
            const uint32_t t = P->ids[k];
            for (int a = 0; a < 3; ++a) {
                Cb->tbox[8 * (size_t)k + a] = f32_down(box_lo[3 * (size_t)t + a]);
                Cb->tbox[8 * (size_t)k + 3 + a] = f32_up(box_hi[3 * (size_t)t + a]);
            }
        }
        *out = Cb;
        return TR_OK;
    } catch (const std::bad_alloc &) {
        return tr_fail(TR_ENOMEM, "tr_cells_build: out of host memory");
    }
}

int tr_cells_sizes(const TrHostBuf *b, int64_t *sizes3) {
    auto Cb = dynamic_cast<const CBuf *>(b);
    if (!Cb || !sizes3) return tr_fail(TR_EINVAL, "tr_cells_sizes: not a cell list");
    sizes3[0] = (int64_t)Cb->off.size() - 1;
    sizes3[1] = (int64_t)Cb->recs.size();
    sizes3[2] = (int64_t)Cb->tbox.size() / 8;
    return TR_OK;
}

int tr_cells_copy(const TrHostBuf *b, int32_t *dims3, double *org3, double *scale3, uint32_t *off,
                  uint32_t *recs, float *tbox) {
    auto Cb = dynamic_cast<const CBuf *>(b);
    if (!Cb) return tr_fail(TR_EINVAL, "tr_cells_copy: not a cell list");
    for (int a = 0; a < 3; ++a) {
        if (dims3) dims3[a] = Cb->dim[a];
        if (org3) org3[a] = Cb->org[a];
        if (scale3) scale3[a] = Cb->scale[a];
    }
    if (off) std::memcpy(off, Cb->off.data(), Cb->off.size() * sizeof(uint32_t));
    if (recs && !Cb->recs.empty()) std::memcpy(recs, Cb->recs.data(), Cb->recs.size() * sizeof(uint32_t));
    if (tbox && !Cb->tbox.empty()) std::memcpy(tbox, Cb->tbox.data(), Cb->tbox.size() * sizeof(float));
    return TR_OK;
}

int tr_pbvh_sizes(const TrHostBuf *b, int64_t *s) {
    auto P = dynamic_cast<const PBuf *>(b);
    if (!P || !s) return tr_fail(TR_EINVAL, "tr_pbvh_sizes: not a point BVH");
    s[0] = (int64_t)P->nodes.size();
    s[1] = (int64_t)P->leaves.size();
    s[2] = (int64_t)P->ids.size();
    s[3] = (int64_t)P->grid.size();
    return TR_OK;
}

int tr_pbvh_grid(const TrHostBuf *b, int32_t *dims3, double *org3, double *scale3,
                 int32_t *cells) {
    auto P = dynamic_cast<const PBuf *>(b);
    if (!P) return tr_fail(TR_EINVAL, "tr_pbvh_grid: not a point BVH");
    for (int a = 0; a < 3; ++a) {
        if (dims3) dims3[a] = P->gdim[a];
        if (org3) org3[a] = P->gorg[a];
        if (scale3) scale3[a] = P->gscale[a];
    }
    if (cells) std::memcpy(cells, P->grid.data(), P->grid.size() * sizeof(int32_t));
    return TR_OK;
}

int tr_pbvh_copy(const TrHostBuf *b, TrPNode *nodes, TrPLeaf *leaves, uint32_t *ids) {
    auto P = dynamic_cast<const PBuf *>(b);
    if (!P) return tr_fail(TR_EINVAL, "tr_pbvh_copy: not a point BVH");
    if (nodes) std::memcpy(nodes, P->nodes.data(), P->nodes.size() * sizeof(TrPNode));
    if (leaves) std::memcpy(leaves, P->leaves.data(), P->leaves.size() * sizeof(TrPLeaf));
    if (ids) std::memcpy(ids, P->ids.data(), P->ids.size() * sizeof(uint32_t));
    return TR_OK;
}

int tr_bbvh_build(int64_t n_parts, const double *lo, const double *hi, TrHostBuf **out) {
    if (!out || n_parts <= 0 || n_parts >= (int64_t)INT32_MAX)
        return tr_fail(TR_EINVAL, "tr_bbvh_build: invalid arguments");
    try {
        BBuf *O = new BBuf();
        std::vector<int32_t> idx(n_parts);
        for (int64_t i = 0; i < n_parts; ++i) idx[i] = (int32_t)i;
        if (n_parts == 1) {
            TrBNode N{};
            N.child[0] = ~0;
            N.child[1] = CHILD_NONE;
            for (int a = 0; a < 3; ++a) {
                N.box[0][a] = lo[a]; N.box[0][3 + a] = hi[a];
                N.box[1][a] = 1.0; N.box[1][3 + a] = 0.0;
            }
            O->nodes.push_back(N);
        } else {
            b_build(*O, lo, hi, idx, 0, n_parts);
        }
        *out = O;
        return TR_OK;
    } catch (const std::bad_alloc &) {
        return tr_fail(TR_ENOMEM, "tr_bbvh_build: out of host memory");
    }
}

int tr_bbvh_sizes(const TrHostBuf *b, int64_t *n) {
    auto B = dynamic_cast<const BBuf *>(b);
    if (!B || !n) return tr_fail(TR_EINVAL, "tr_bbvh_sizes: not a partition BVH");
    *n = (int64_t)B->nodes.size();
    return TR_OK;
}

int tr_bbvh_copy(const TrHostBuf *b, TrBNode *nodes) {
    auto B = dynamic_cast<const BBuf *>(b);
    if (!B || !nodes) return tr_fail(TR_EINVAL, "tr_bbvh_copy: not a partition BVH");
    std::memcpy(nodes, B->nodes.data(), B->nodes.size() * sizeof(TrBNode));
    return TR_OK;
}

int tr_bnodes_activity(int64_t n_nodes, const TrBNode *nodes, const uint8_t *active,
                       uint8_t *out) {
    if (!nodes || !active || !out || n_nodes <= 0)
        return tr_fail(TR_EINVAL, "tr_bnodes_activity: invalid arguments");
    // children always have larger indices than their parent (pre-order build)
    for (int64_t i = n_nodes - 1; i >= 0; --i) {
        uint8_t bits = 0;
        for (int c = 0; c < 2; ++c) {
            int32_t ch = nodes[i].child[c];
            bool any = false;
            if (ch == CHILD_NONE) any = false;
            else if (ch < 0) any = active[~ch] != 0;
            else any = out[ch] != 0;
            if (any) bits |= (uint8_t)(1u << c);
        }
        out[i] = bits;
    }
    return TR_OK;
}

int tr_bbvh_activity(const TrHostBuf *b, const uint8_t *active, uint8_t *out) {
    auto B = dynamic_cast<const BBuf *>(b);
    if (!B) return tr_fail(TR_EINVAL, "tr_bbvh_activity: not a partition BVH");
    return tr_bnodes_activity((int64_t)B->nodes.size(), B->nodes.data(), active, out);
}

int tr_kbsp_build(int64_t n_parts, const double *lo, const double *hi, TrHostBuf **out) {
    if (!out || n_parts <= 0 || n_parts >= (int64_t)(INT32_MAX >> 3))
        return tr_fail(TR_EINVAL, "tr_kbsp_build: invalid arguments");
    try {
        KBuf *O = new KBuf();
        for (int a = 0; a < 3; ++a) { O->root_lo[a] = INFINITY; O->root_hi[a] = -INFINITY; }
        std::vector<int32_t> ids(n_parts);
        for (int64_t i = 0; i < n_parts; ++i) {
            ids[i] = (int32_t)i;
            for (int a = 0; a < 3; ++a) {
                O->root_lo[a] = std::min(O->root_lo[a], lo[3 * i + a]);
                O->root_hi[a] = std::max(O->root_hi[a], hi[3 * i + a]);
            }
        }
        k_build(*O, lo, hi, ids, 0);
        *out = O;
        return TR_OK;
    } catch (const std::bad_alloc &) {
        return tr_fail(TR_ENOMEM, "tr_kbsp_build: out of host memory");
    }
}

int tr_kbsp_sizes(const TrHostBuf *b, int64_t *sizes2) {
    auto K = dynamic_cast<const KBuf *>(b);
    if (!K || !sizes2) return tr_fail(TR_EINVAL, "tr_kbsp_sizes: not a BSP");
    sizes2[0] = (int64_t)K->nodes.size();
    sizes2[1] = (int64_t)K->leaf_pids.size();
    return TR_OK;
}

int tr_kbsp_copy(const TrHostBuf *b, TrKNode *nodes, int32_t *leaf_pids, double *root6) {
    auto K = dynamic_cast<const KBuf *>(b);
    if (!K) return tr_fail(TR_EINVAL, "tr_kbsp_copy: not a BSP");
    if (nodes) std::memcpy(nodes, K->nodes.data(), K->nodes.size() * sizeof(TrKNode));
    if (leaf_pids) std::memcpy(leaf_pids, K->leaf_pids.data(), K->leaf_pids.size() * sizeof(int32_t));
    if (root6)
        for (int a = 0; a < 3; ++a) { root6[a] = K->root_lo[a]; root6[3 + a] = K->root_hi[a]; }
    return TR_OK;
}

int tr_knodes_activity(int64_t n_nodes, const TrKNode *nodes, const int32_t *leaf_pids,
                       const uint8_t *active, uint8_t *out) {
    if (!nodes || !leaf_pids || !active || !out || n_nodes <= 0)
        return tr_fail(TR_EINVAL, "tr_knodes_activity: invalid arguments");
    for (int64_t i = n_nodes - 1; i >= 0; --i) {  // children follow their parent
        const TrKNode &N = nodes[i];
        uint8_t any = 0;
        if (N.info < 0) {
            const int32_t s = ~N.info;
            for (int32_t k = 0; k < N.aux && !any; ++k) any = active[leaf_pids[s + k]] != 0;
        } else {
            any = (out[i + 1] | out[N.info >> 2]) ? 1 : 0;
        }
        out[i] = any;
    }
    return TR_OK;
}

// ============================================================ leaf walk tables
//
// K:93-136 returns the LOWEST-index tet whose barycentrics are all >= -1e-9.
// Inside a leaf's exclusive box only the leaf's tets can contain the point,
// and the kernels used to test them in id order (a regular cube: 3.3 record
// loads per sample, the central tet -- a third of the volume -- last).  The
// walk starts at the largest tet and steps across the most violated face;
// a tet that accepts the point with every barycentric >= TR_WALK_TAU is the
// answer when it is CERTIFIED against every lower-id tet of the leaf (below);
// anything else falls back to the id-order scan, so the result is always
// the reference's.
namespace {

constexpr long double W_TOL = 1e-9L;     // K:15
constexpr long double W_M1 = 1e-8L;      // margin beyond the slack
constexpr long double W_TAU = (long double)TR_WALK_TAU;

struct TetL {
    long double v[4][3];
    long double inv[3][3];
    bool ok;
};

TetL tet_geo(const double *const vp[4]) {
    TetL T;
    for (int i = 0; i < 4; ++i)
        for (int a = 0; a < 3; ++a) T.v[i][a] = vp[i][a];
    long double e[3][3];   // columns: v1-v0, v2-v0, v3-v0 (mesh.py:253)
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) e[a][c] = T.v[c + 1][a] - T.v[0][a];
    const long double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                            e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                            e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
    T.ok = det != 0.0L && std::isfinite((double)det);
    if (!T.ok) return T;
    T.inv[0][0] = (e[1][1] * e[2][2] - e[1][2] * e[2][1]) / det;
    T.inv[0][1] = (e[0][2] * e[2][1] - e[0][1] * e[2][2]) / det;
    T.inv[0][2] = (e[0][1] * e[1][2] - e[0][2] * e[1][1]) / det;
    T.inv[1][0] = (e[1][2] * e[2][0] - e[1][0] * e[2][2]) / det;
    T.inv[1][1] = (e[0][0] * e[2][2] - e[0][2] * e[2][0]) / det;
    T.inv[1][2] = (e[0][2] * e[1][0] - e[0][0] * e[1][2]) / det;
    T.inv[2][0] = (e[1][0] * e[2][1] - e[1][1] * e[2][0]) / det;
    T.inv[2][1] = (e[0][1] * e[2][0] - e[0][0] * e[2][1]) / det;
    T.inv[2][2] = (e[0][0] * e[1][1] - e[0][1] * e[1][0]) / det;
    return T;
}

void bary_l(const TetL &T, const long double p[3], long double l[4]) {
    long double q[3];
    for (int a = 0; a < 3; ++a) q[a] = p[a] - T.v[0][a];
    for (int r = 0; r < 3; ++r) l[r + 1] = T.inv[r][0] * q[0] + T.inv[r][1] * q[1] + T.inv[r][2] * q[2];
    l[0] = 1.0L - l[1] - l[2] - l[3];
}

// No point that tet K accepts with every barycentric >= TAU is accepted by
// tet J (barycentrics >= -1e-9): (A) a face plane of J has K shrunk to
// barycentrics >= TAU / 2 beyond -(slack + margin), or (B) a face plane of
// K has J inflated by (slack + margin) below TAU / 2.  Convexity: checking
// the 4 vertices of the shrunk / inflated tet covers it.  The device's
// rounding of either tet's barycentrics (<= 1e-10, `certifiable` below) is
// covered by the TAU / 2 and 1e-8 margins.
bool separated(const TetL &J, const TetL &K) {
    long double w[4][3], u[4][3], sk[3] = {0, 0, 0}, sj[3] = {0, 0, 0};
    for (int i = 0; i < 4; ++i)
        for (int a = 0; a < 3; ++a) { sk[a] += K.v[i][a]; sj[a] += J.v[i][a]; }
    const long double s = W_TOL + W_M1;
    for (int i = 0; i < 4; ++i)
        for (int a = 0; a < 3; ++a) {
            w[i][a] = (1.0L - 2.0L * W_TAU) * K.v[i][a] + 0.5L * W_TAU * sk[a];
            u[i][a] = (1.0L + 4.0L * s) * J.v[i][a] - s * sj[a];
        }
    long double lw[4][4], lu[4][4];
    for (int i = 0; i < 4; ++i) { bary_l(J, w[i], lw[i]); bary_l(K, u[i], lu[i]); }
    for (int f = 0; f < 4; ++f) {
        bool a_ok = true, b_ok = true;
        for (int i = 0; i < 4; ++i) {
            a_ok = a_ok && lw[i][f] <= -(W_TOL + W_M1);
            b_ok = b_ok && lu[i][f] <= 0.5L * W_TAU;
        }
        if (a_ok || b_ok) return true;
    }
    return false;
}

// The table of one leaf: n <= 8 tets, vertex ids vid[i][4], positions vp[i][4],
// tet ids ids[i] (ascending or not).
void walk_table(int n, const int64_t (*vid)[4], const double *const (*vp)[4], const int64_t *ids,
                uint32_t walk[8], const float *ex_lo = nullptr, TrLeafPred *pred = nullptr) {
    for (int k = 0; k < 8; ++k) walk[k] = 0;
    if (pred) std::memset(pred, 0, sizeof(TrLeafPred));
    if (n < 1 || n > 8) return;
    TetL geo[8];
    long double vmax = 0.0L, imax = 0.0L, vol_best = -1.0L;
    int first = 0;
    for (int i = 0; i < n; ++i) {
        geo[i] = tet_geo(vp[i]);
        if (!geo[i].ok) return;
        long double isum = 0.0L;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) isum += std::fabs(geo[i].inv[r][c]);
        imax = std::max(imax, isum);
        for (int q = 0; q < 4; ++q)
            for (int a = 0; a < 3; ++a) vmax = std::max(vmax, (long double)std::fabs(vp[i][q][a]));
        // volume ~ 1 / |det(inv)|: the largest tet has the smallest inverse
        const long double (&m)[3][3] = geo[i].inv;
        const long double dinv = std::fabs(m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                                           m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                                           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]));
        const long double vol = 1.0L / dinv;
        if (vol > vol_best) { vol_best = vol; first = i; }
    }
    // the device's barycentric rounding error is a few ulp of |inv| * |coords|;
    // it must stay far below the 1e-8 and TAU / 2 margins
    const bool certifiable = imax * (vmax + 1.0L) * 0x1p-51L < 1e-10L;
    for (int i = 0; i < n; ++i) {
        uint32_t e = 0;
        for (int f = 0; f < 4; ++f) {
            int64_t fa[3], m = 0;
            for (int q = 0; q < 4; ++q)
                if (q != f) fa[m++] = vid[i][q];
            std::sort(fa, fa + 3);
            int nb = i;
            for (int j = 0; j < n && nb == i; ++j) {
                if (j == i) continue;
                int hits = 0;
                for (int q = 0; q < 4; ++q)
                    hits += (vid[j][q] == fa[0]) + (vid[j][q] == fa[1]) + (vid[j][q] == fa[2]);
                if (hits == 3) nb = j;
            }
            e |= (uint32_t)nb << (3 * f);
        }
        bool cert = certifiable;
        for (int j = 0; j < n && cert; ++j)
            if (ids[j] < ids[i]) cert = separated(geo[j], geo[i]);
        if (cert) e |= 1u << 12;
        walk[i >> 1] |= e << (16 * (i & 1));
    }
    walk[4] = (uint32_t)first | (1u << 31);
    if (pred && ex_lo) {   // l_r(p) = inv_r . (p - v0) = inv_r . (p - lo) + inv_r . (lo - v0)
        const TetL &F = geo[first];
        for (int r = 0; r < 3; ++r) {
            long double d = 0.0L;
            for (int c = 0; c < 3; ++c) {
                pred->row[r][c] = (float)F.inv[r][c];
                d += F.inv[r][c] * ((long double)ex_lo[c] - F.v[0][c]);
            }
            pred->row[r][3] = (float)d;
        }
    }
}

}  // namespace

static void walk_table_cube(int parity, uint32_t walk[8], const float *ex_lo, TrLeafPred *pred) {
    // mesh.py:151-163: corner c = 4x + 2y + z; odd cubes mirror x (c ^ 4)
    static const int P[5][4] = {{0, 4, 2, 1}, {6, 2, 4, 7}, {5, 1, 7, 4}, {3, 7, 1, 2}, {4, 2, 1, 7}};
    double pos[8][3];
    for (int c = 0; c < 8; ++c) {
        pos[c][0] = (c >> 2) & 1; pos[c][1] = (c >> 1) & 1; pos[c][2] = c & 1;
    }
    int64_t vid[5][4], ids[5];
    const double *vp[5][4];
    for (int k = 0; k < 5; ++k) {
        ids[k] = k;
        for (int q = 0; q < 4; ++q) {
            const int c = parity ? (P[k][q] ^ 4) : P[k][q];
            vid[k][q] = c;
            vp[k][q] = pos[c];
        }
    }
    walk_table(5, vid, vp, ids, walk, ex_lo, pred);
}

void tr_walk_table_cube(int parity, uint32_t walk[8]) { walk_table_cube(parity, walk, nullptr, nullptr); }

int tr_grid_walk_pred(double pad, TrLeafPred *pred2, uint32_t *walk16) {
    if (!pred2 || !(pad >= 0.0)) return tr_fail(TR_EINVAL, "tr_grid_walk_pred: invalid arguments");
    const float lo[3] = {(float)pad, (float)pad, (float)pad};   // an interior cube at the origin
    uint32_t w[2][8];
    walk_table_cube(0, w[0], lo, pred2);
    walk_table_cube(1, w[1], lo, pred2 + 1);
    if (walk16) std::memcpy(walk16, w, sizeof w);
    return TR_OK;
}

extern "C" int tr_leaf_walk(int64_t n_leaves, TrPLeaf *leaves, const uint32_t *rec_ids,
                            const double *vertices, const int64_t *tets, TrLeafPred *pred) {
    if (n_leaves < 0 || (n_leaves > 0 && (!leaves || !vertices || !tets)))
        return tr_fail(TR_EINVAL, "tr_leaf_walk: invalid arguments");
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t L = 0; L < n_leaves; ++L) {
        TrPLeaf &lf = leaves[L];
        const int n = (int)std::min<uint32_t>(lf.count, 9);
        int64_t vid[8][4], ids[8];
        const double *vp[8][4];
        if (n > 8) {
            for (int k = 0; k < 8; ++k) lf.walk[k] = 0;
            if (pred) std::memset(pred + L, 0, sizeof(TrLeafPred));
            continue;
        }
        for (int i = 0; i < n; ++i) {
            const int64_t t = rec_ids ? (int64_t)rec_ids[lf.start + i] : (int64_t)lf.start + i;
            ids[i] = t;
            for (int q = 0; q < 4; ++q) {
                vid[i][q] = tets[4 * t + q];
                vp[i][q] = vertices + 3 * vid[i][q];
            }
        }
        walk_table(n, vid, vp, ids, lf.walk, lf.ex_lo, pred ? pred + L : nullptr);
    }
    return TR_OK;
}

void tr_host_free(TrHostBuf *b) { delete b; }

int tr_pack_tets(int64_t n_tets, const int64_t *tets, const double *tet_orig,
                 const double *tet_inv, const double *field, int32_t centering,
                 const uint32_t *order, TrTetRecord *out) {
    if (n_tets <= 0 || !tets || !tet_orig || !tet_inv || !field || !out)
        return tr_fail(TR_EINVAL, "tr_pack_tets: invalid arguments");
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n_tets; ++k) {
        const int64_t t = order ? (int64_t)order[k] : k;
        TrTetRecord &R = out[k];
        std::memcpy(R.inv, tet_inv + 9 * t, 72);
        std::memcpy(R.orig, tet_orig + 3 * t, 24);
        if (centering == 0) {
            for (int i = 0; i < 4; ++i) R.f[i] = field[tets[4 * t + i]];
        } else {
            R.f[0] = field[t];
            R.f[1] = R.f[2] = R.f[3] = 0.0;
        }
    }
    return TR_OK;
}

int tr_tet_boxes(int64_t n_tets, const double *vertices, const int64_t *tets, double pad,
                 double *lo, double *hi) {
    if (n_tets <= 0 || !vertices || !tets || !lo || !hi)
        return tr_fail(TR_EINVAL, "tr_tet_boxes: invalid arguments");
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_tets; ++t) {
        const int64_t *tv = tets + 4 * t;
        for (int a = 0; a < 3; ++a) {
            const double v0 = vertices[3 * tv[0] + a], v1 = vertices[3 * tv[1] + a];
            const double v2 = vertices[3 * tv[2] + a], v3 = vertices[3 * tv[3] + a];
            lo[3 * t + a] = std::min(std::min(v0, v1), std::min(v2, v3)) - pad;
            hi[3 * t + a] = std::max(std::max(v0, v1), std::max(v2, v3)) + pad;
        }
    }
    return TR_OK;
}

int tr_tf_meta(int64_t n_parts, const double *vrange, const double *T, int64_t n, double lo,
               double hi, double *max_opacity, double *raw_variance, double *sigma,
               uint8_t *active) {
    if (n_parts <= 0 || !vrange || !T || n < 2 || !(lo < hi))
        return tr_fail(TR_EINVAL, "tr_tf_meta: invalid arguments");
    std::vector<double> raw(n_parts), mop(n_parts);
    int err = 0;
#pragma omp parallel
    {
        std::vector<double> rows, W, D;
#pragma omp for schedule(dynamic, 16)
        for (int64_t p = 0; p < n_parts; ++p) {
            // transfer.py:_overlapping_colors: interpolated ends + table rows inside
            double rmin = vrange[2 * p], rmax = vrange[2 * p + 1];
            if (rmin > rmax) { err = 1; continue; }
            double u_min = (rmin - lo) / (hi - lo) * (double)(n - 1);
            double u_max = (rmax - lo) / (hi - lo) * (double)(n - 1);
            // Python int(floor(.)) semantics, clamped so the cast cannot overflow
            double fl = std::min(std::max(std::floor(u_min), -2.0), (double)n + 2.0);
            double cl = std::min(std::max(std::ceil(u_max), -2.0), (double)n + 2.0);
            int64_t j0 = std::max((int64_t)fl + 1, (int64_t)0);
            int64_t j1 = std::min((int64_t)cl - 1, n - 1);
            rows.clear();
            double c[4];
            tf_lookup(T, n, lo, hi, rmin, c);
            rows.insert(rows.end(), c, c + 4);
            for (int64_t j = j0; j <= j1; ++j) rows.insert(rows.end(), T + 4 * j, T + 4 * j + 4);
            tf_lookup(T, n, lo, hi, rmax, c);
            rows.insert(rows.end(), c, c + 4);
            const int64_t k = (int64_t)rows.size() / 4;
            // compute_partition_meta: opacity-weighted RGB, axis-0 mean
            // (sequential), per-row squared distance (sequential over 3),
            // mean over rows (numpy pairwise sum)
            W.resize(3 * k);
            double amax = -INFINITY;
            for (int64_t i = 0; i < k; ++i) {
                double a = rows[4 * i + 3];
                amax = (a > amax) ? a : amax;
                for (int q = 0; q < 3; ++q) W[3 * i + q] = rows[4 * i + q] * a;
            }
            double mean[3];
            for (int q = 0; q < 3; ++q) {
                double s = W[q];
                for (int64_t i = 1; i < k; ++i) s += W[3 * i + q];
                mean[q] = s / (double)k;
            }
            D.resize(k);
            for (int64_t i = 0; i < k; ++i) {
                double d0 = W[3 * i] - mean[0], d1 = W[3 * i + 1] - mean[1], d2 = W[3 * i + 2] - mean[2];
                D[i] = ((d0 * d0) + (d1 * d1)) + (d2 * d2);
            }
            raw[p] = np_pairwise_sum(D.data(), k) / (double)k;
            mop[p] = amax;
        }
    }
    if (err) return tr_fail(TR_EINVAL, "tr_tf_meta: invalid value range (min > max)");
    // normalize_variances (transfer.py:127-141)
    double vmin = raw[0], vmax = raw[0];
    for (int64_t p = 1; p < n_parts; ++p) { vmin = std::min(vmin, raw[p]); vmax = std::max(vmax, raw[p]); }
    for (int64_t p = 0; p < n_parts; ++p) {
        double s = (vmax == vmin) ? 1.0 : (raw[p] - vmin) / (vmax - vmin);
        if (sigma) sigma[p] = s;
        if (max_opacity) max_opacity[p] = mop[p];
        if (raw_variance) raw_variance[p] = raw[p];
        if (active) active[p] = mop[p] > 0.0 ? 1 : 0;
    }
    return TR_OK;
}

#if TR_HAVE_GLIBC_POW
static const uint64_t H_POW_LOG[] = TR_POW_LOG_INIT;
static const uint64_t H_POW_EXP_HEAD[] = TR_POW_EXP_HEAD_INIT;
static const uint64_t H_POW_EXP_TAB[] = TR_POW_EXP_TAB_INIT;
#endif

int tr_pow_glibc_available(void) { return TR_HAVE_GLIBC_POW; }

double tr_pow_glibc_host(double x, double y, int32_t *exact) {
#if TR_HAVE_GLIBC_POW
    if (!tr_pow_glibc_supported(x, y)) {
        if (exact) *exact = 0;
        return std::pow(x, y);
    }
    bool ex = false;
    const double r = tr_pow_glibc(x, y, H_POW_LOG, H_POW_LOG + 9, H_POW_EXP_HEAD, H_POW_EXP_TAB, &ex);
    if (exact) *exact = ex ? 1 : 0;
    return r;
#else
    if (exact) *exact = 0;
    return std::pow(x, y);
#endif
}

double tr_step_size(double s1, double s2, double p, double sigma) {
    double m = (1.0 < sigma) ? 1.0 : sigma;  // Python min(sigma, 1.0)
    double v = s1 + (s2 - s1) * std::pow(std::fabs(m - 1.0), p);
    return (s1 > v) ? s1 : v;  // Python max(v, s1)
}

double tr_opacity_correction(double alpha, double s, double s1) {
    return 1.0 - std::pow(1.0 - alpha, s / s1);
}

int tr_step_sizes(int64_t n, const double *sigma, double s1, double s2, double p, double *out) {
    return tr_epoch_steps(n, sigma, s1, s2, p, out, nullptr);
}

int tr_epoch_steps(int64_t n, const double *sigma, double s1, double s2, double p, double *step,
                   double *step_ratio) {
    if (n < 0 || (n > 0 && (!sigma || (!step && !step_ratio))))
        return tr_fail(TR_EINVAL, "tr_epoch_steps: invalid arguments");
    // ~20 ns per pow: threads only pay off for very large partition counts
#pragma omp parallel for schedule(static) if (n > 262144)
    for (int64_t i = 0; i < n; ++i) {
        const double s = tr_step_size(s1, s2, p, sigma[i]);
        if (step) step[i] = s;
        if (step_ratio) { step_ratio[2 * i] = s; step_ratio[2 * i + 1] = s / s1; }  // K:27 exponent
    }
    return TR_OK;
}

}  // extern "C"
