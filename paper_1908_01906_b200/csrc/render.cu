// render.cu -- sm_100a kernels of the tetray hot path.
//
//   tr_render_frame   replaces _kernels.render_frame   (pkg/src/tetray/_kernels.py:312-398)
//   tr_field_at_many  replaces _kernels.field_at_many  (K:157-170)
//   tr_scatter_tiles  multi-GPU merge of disjoint pixel tiles
//
// Arithmetic contract: every fp64 expression is
// evaluated in the reference's (Python left-to-right) order and this file is
// compiled with -fmad=false, so no multiply-add is contracted; / and sqrt
// are IEEE round-to-nearest.  Results are therefore bit-identical to the
// numba reference, except glibc pow in skip-adaptive mode.
//
// A frame is three kernels per ray chunk:
//   trace_intervals_kernel  one thread per ray, 8x4 pixel tiles per warp: the
//       exact front-to-back partition-interval sequence (K:360-391 calling
//       next_interval K:173-230) over a BVH2 with f64 child boxes, pruned by
//       per-epoch subtree activity bits, kept as partition ids; rays with
//       nothing to march are finished here, the rest get a cost bucket.
//   order_rays_kernel  marching rays sorted into descending cost buckets
//       (longest first, so the frame does not end on one long ray).
//   march_kernel<G>  persistent CTAs; G lanes march ONE ray: each lane
//       shades one consecutive sample (interval and k from the trace's prefix
//       sample counts), then the group composites the G results in sample
//       order with the exact early-termination rule.  Point location: uniform-grid
//       candidate leaf proved by its exclusive box (a point strictly inside
//       it can only lie in that leaf's tets, scanned in ascending id order:
//       first hit = lowest index, the reference's tie rule K:119), else a
//       full min-id-pruned BVH descent.
//   Per-partition samples are added per interval with 64-bit integer atomics
//   (exact, order independent).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>

#include "glibc_pow.cuh"
#include "grid_layout.cuh"
#include "tetray_b200.h"
#include "tr_internal.h"

namespace {

constexpr double BARY_TOL = 1e-9;  // K:15
constexpr int TILE_W = 8, TILE_H = 4;
constexpr int PSTACK = 64;
constexpr int BSTACK = 64;
#ifndef TR_MARCH_BLOCK
#define TR_MARCH_BLOCK 256   // A/B knob: threads per march CTA
#endif
#ifndef TR_MARCH_MINB
#define TR_MARCH_MINB 3      // A/B knob: resident march CTAs per SM the registers are budgeted for
#endif
constexpr int MARCH_BLOCK = TR_MARCH_BLOCK;
constexpr int MB = TR_MARCH_MINB;
constexpr int TRACE_BLOCK = 128;
constexpr int IV_CAP = 64;           // partition ids per ray kept in the scratch list
constexpr int CAND_CAP = 48;         // partition slabs per ray kept by the candidate raster
constexpr int N_BUCKETS = 64;        // ray-cost buckets (4 per octave) for longest-first order
constexpr int32_t CHILD_NONE = INT32_MIN;
constexpr unsigned FULL = 0xffffffffu;

// Optional kernel statistics (TR_FLAG_STATS): counters read back with
// tr_kernel_stats().  Indices:
enum : int {
    ST_ROUNDS = 0,       // group rounds with a ray
    ST_PARTIAL,          // rounds with fewer samples than lanes
    ST_SLOTS,            // lane-samples shaded
    ST_FOUND,            // samples inside a tet
    ST_GRID_HIT,         // located through the grid + exclusive box
    ST_DESCENT,          // full BVH descents
    ST_INLINE_IV,        // next_interval calls in the march (list overflow)
    ST_POW,              // pow() evaluations
    ST_TRACE_IV,         // intervals produced by the trace pass
    ST_TRACE_RAYS,       // rays traced
    ST_BSP_OVERFLOW,     // rays redone with the BVH (BSP buffer or stack overflow)
    ST_BSP_CELLS,        // BSP leaf cells enumerated
    ST_TRACE_MAX_IV,     // most intervals of one ray (max)
    ST_BSP_NODES,        // BSP nodes visited by the trace
    ST_TRACE_MAX_NODES,  // most BSP nodes visited by one ray (max)
    ST_MAX_RAY_SAMPLES,  // most samples of one ray's stored list (max)
    ST_TILE_CYCLES,      // trace: SM cycles summed over 32-ray tiles (TR_FLAG_TILE_TIMING)
    ST_TILE_MAX_CYCLES,  // trace: most cycles of one tile (max)
    ST_MARCH_T0,         // march (TR_FLAG_TILE_TIMING): earliest CTA start, globaltimer ns (min)
    ST_MARCH_TQ,         // first time a group found the ray queue empty (min)
    ST_MARCH_T1,         // latest CTA end (max)
    ST_COUNT
};
__device__ unsigned long long g_stats[32];

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct RayD {
    double ox, oy, oz, dx, dy, dz;
    double ix, iy, iz;  // 1/d per axis (valid where d != 0), K:36
    bool nx, ny, nz;    // d != 0
};

// K:30-71 (a zero-direction miss returns (1, 0)).
__device__ __forceinline__ void slab(const RayD &r, const double *lo, const double *hi,
                                     double &t0, double &t1) {
    t0 = -INFINITY;
    t1 = INFINITY;
    if (r.nx) {
        double a = (lo[0] - r.ox) * r.ix, b = (hi[0] - r.ox) * r.ix;
        if (a > b) { double t = a; a = b; b = t; }
        if (a > t0) t0 = a;
        if (b < t1) t1 = b;
    } else if (r.ox < lo[0] || r.ox > hi[0]) { t0 = 1.0; t1 = 0.0; return; }
    if (r.ny) {
        double a = (lo[1] - r.oy) * r.iy, b = (hi[1] - r.oy) * r.iy;
        if (a > b) { double t = a; a = b; b = t; }
        if (a > t0) t0 = a;
        if (b < t1) t1 = b;
    } else if (r.oy < lo[1] || r.oy > hi[1]) { t0 = 1.0; t1 = 0.0; return; }
    if (r.nz) {
        double a = (lo[2] - r.oz) * r.iz, b = (hi[2] - r.oz) * r.iz;
        if (a > b) { double t = a; a = b; b = t; }
        if (a > t0) t0 = a;
        if (b < t1) t1 = b;
    } else if (r.oz < lo[2] || r.oz > hi[2]) { t0 = 1.0; t1 = 0.0; return; }
}

// ------------------------------------------------------------ point location

struct PQuery {  // a sample point
    double x, y, z;
};

__device__ __forceinline__ PQuery make_query(double x, double y, double z) {
    PQuery q;
    q.x = x; q.y = y; q.z = z;
    return q;
}

// f32 round-down / round-up copies of a point for conservative tests against
// f32 boxes (the BVH descent and the cell lists; the grid path compares in f64)
struct PQueryF {
    float xd, yd, zd, xu, yu, zu;
};

__device__ __forceinline__ PQueryF make_qf(const PQuery &q) {
    PQueryF f;
    f.xd = __double2float_rd(q.x); f.yd = __double2float_rd(q.y); f.zd = __double2float_rd(q.z);
    f.xu = __double2float_ru(q.x); f.yu = __double2float_ru(q.y); f.zu = __double2float_ru(q.z);
    return f;
}

// conservative: true whenever the exact point lies in the closed box
__device__ __forceinline__ bool in_box(const PQueryF &q, float lx, float ly, float lz, float hx,
                                       float hy, float hz) {
    return !(q.xu < lx) && !(q.xd > hx) && !(q.yu < ly) && !(q.yd > hy) && !(q.zu < lz) &&
           !(q.zd > hz);
}

// exact: true only if the point is strictly inside the f32 box (the floats
// widen to double exactly, so these are exact comparisons)
__device__ __forceinline__ bool strictly_in(const PQuery &q, const float *lo, const float *hi) {
    return q.x > (double)lo[0] && q.x < (double)hi[0] && q.y > (double)lo[1] &&
           q.y < (double)hi[1] && q.z > (double)lo[2] && q.z < (double)hi[2];
}

// 32-B read-only loads (LDG.E.ENL2.256, sm_100): the march is bound by the
// L1 data pipe's wavefronts (ncu: l1tex__data_pipe_lsu_wavefronts ~91% of
// peak), and a warp-wide gather costs about one wavefront per distinct line
// per instruction -- so each 32-B record chunk, TF row, pow table entry and
// leaf header is fetched by one instruction instead of two.
#ifndef TR_LD256
#define TR_LD256 1
#endif
__device__ __forceinline__ double4 ldg256(const void *p) {
    double4 v;
#if TR_LD256
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
#else
    const double2 a = __ldg(reinterpret_cast<const double2 *>(p));
    const double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    v = make_double4(a.x, a.y, b.x, b.y);
#endif
    return v;
}

#ifndef TR_RAY_TIMES
#define TR_RAY_TIMES 0
#endif
#ifndef TR_ROUND_TIMES
#define TR_ROUND_TIMES 0
#endif
#ifndef TR_UNROLL_COMPOSITE
#define TR_UNROLL_COMPOSITE 1   // A/B knob: the round's compositing loop unrolled over G
#endif

// The 96 B of a record the barycentric test reads (inverse + origin).
struct RecM {
    double2 a0, a1, a2, a3, a4, a5;
};

__device__ __forceinline__ RecM load_recm(const TrTetRecord *__restrict__ recs, uint32_t k) {
    const char *r = reinterpret_cast<const char *>(recs + k);
    const double4 c0 = ldg256(r), c1 = ldg256(r + 32), c2 = ldg256(r + 64);
    RecM m;
    m.a0 = make_double2(c0.x, c0.y); m.a1 = make_double2(c0.z, c0.w);
    m.a2 = make_double2(c1.x, c1.y); m.a3 = make_double2(c1.z, c1.w);
    m.a4 = make_double2(c2.x, c2.y); m.a5 = make_double2(c2.z, c2.w);
    return m;
}

// K:121-128: barycentrics of q in a record; true if all >= -BARY_TOL.
__device__ __forceinline__ bool bary_of(const RecM &m, const PQuery &q, double l[4]) {
    const double qx = q.x - m.a4.y, qy = q.y - m.a5.x, qz = q.z - m.a5.y;
    const double l1 = m.a0.x * qx + m.a0.y * qy + m.a1.x * qz;
    const double l2 = m.a1.y * qx + m.a2.x * qy + m.a2.y * qz;
    const double l3 = m.a3.x * qx + m.a3.y * qy + m.a4.x * qz;
    const double l0 = 1.0 - l1 - l2 - l3;
    l[0] = l0; l[1] = l1; l[2] = l2; l[3] = l3;
    return l0 >= -BARY_TOL && l1 >= -BARY_TOL && l2 >= -BARY_TOL && l3 >= -BARY_TOL;
}

__device__ __forceinline__ bool bary_test(const TrTetRecord *__restrict__ recs, uint32_t k,
                                          const PQuery &q, double l[4]) {
    return bary_of(load_recm(recs, k), q, l);
}

#if TR_HAVE_GLIBC_POW
__constant__ unsigned long long c_pow_lhead[] = TR_POW_LOG_HEAD_INIT;
__constant__ unsigned long long c_pow_ehead[] = TR_POW_EXP_HEAD_INIT;
__device__ const __align__(32) unsigned long long d_pow_ltab[] = TR_POW_LOG_TAB_INIT;
__device__ const __align__(16) unsigned long long d_pow_etab[] = TR_POW_EXP_TAB_INIT;
#endif

// x**y as the reference computes it (glibc pow, K:22 / K:27): the restated
// glibc main path where it applies, CUDA pow elsewhere (never reached for
// opacity correction: x = 1 - alpha in [0, 1], y = step/s1 in [1, 2^63)).
__device__ __forceinline__ double ref_pow(double x, double y) {
    if (x == 1.0) return 1.0;  // glibc: pow(1, y) == 1 for every y
#if TR_HAVE_GLIBC_POW
    if (tr_pow_glibc_supported(x, y)) {
        bool exact;
        const double r = tr_pow_glibc(x, y, (const uint64_t *)c_pow_lhead,
                                      (const uint64_t *)d_pow_ltab, (const uint64_t *)c_pow_ehead,
                                      (const uint64_t *)d_pow_etab, &exact);
        // |y log x| >= 512: glibc under/overflows; for x < 1 the result is
        // < 2^-738, so 1 - pow is 1.0 either way
        if (exact || x < 1.0) return r;
    } else if (x == 0.0 && y > 0.0) {
        return 0.0;
    }
#endif
    return pow(x, y);
}

struct SceneK {  // kernel copy of TrDeviceScene
    const TrTetRecord *__restrict__ tets;   // in LEAF order: record k holds tet pleaf_ids[k]
    const TrPNode *__restrict__ pnodes;
    const TrPLeaf *__restrict__ pleaves;
    const uint32_t *__restrict__ pleaf_ids;
    const TrBNode *__restrict__ bnodes;
    const double *__restrict__ part_lo;     // (P,3) partition boxes (next_interval's leaf boxes)
    const double *__restrict__ part_hi;
    const int32_t *__restrict__ pgrid;      // uniform-grid leaf candidates
    const TrPLeaf *__restrict__ pgrid_leaf; // the candidate leaf's header per cell
    const TrKNode *__restrict__ knodes;     // partition BSP (NULL: BVH trace)
    const int32_t *__restrict__ kleaf_pids;
    double kroot_lo[3], kroot_hi[3];
    int32_t gdim[3];
    int32_t centering;
    double gorg[3], gscale[3];
    double mesh_lo[3], mesh_hi[3];
    const uint32_t *__restrict__ cell_off;  // cell candidate lists (NULL: none)
    const uint32_t *__restrict__ cell_recs;
    const float4 *__restrict__ tbox;        // per record: padded box (2 x float4)
    int32_t cdim[3];
    int32_t cells_first;
    double corg[3], cscale[3];
    const float4 *__restrict__ pgrid_pred;  // per cell: 3 float4 rows (TrLeafPred), or NULL
    int32_t pred_classes;                   // 2: pred_class[cube parity] (grid scenes)
    float pred_class[2][12];
    int64_t grid_n;                         // > 0: analytic cube-grid leaves (grid_layout.cuh)
    double grid_pad;
    int32_t grid_brick;
    const uint32_t *__restrict__ class_walk;   // 2 x 8 u32: walk tables of even / odd cubes
};

// Exclusive-leaf path: the records [start, start+count) are the leaf's tets in
// ascending id order, so the first one containing q is the lowest index.
// One record at a time (the fewest record loads).
__device__ __forceinline__ uint32_t scan_leaf_first(const SceneK &S, uint32_t start,
                                                    uint32_t count, const PQuery &q, double l[4]) {
    for (uint32_t k = start; k < start + count; ++k)
        if (bary_of(load_recm(S.tets, k), q, l)) return k;
    return UINT32_MAX;
}

// Pairwise variant: two records in flight per step, tested in order.
__device__ __forceinline__ uint32_t scan_leaf_pairs(const SceneK &S, uint32_t start,
                                                    uint32_t count, const PQuery &q, double l[4]) {
    const uint32_t end = start + count;
    for (uint32_t k = start; k < end; k += 2) {
        const bool has_b = k + 1 < end;
        const RecM A = load_recm(S.tets, k);
        const RecM Bm = load_recm(S.tets, has_b ? k + 1 : k);
        if (bary_of(A, q, l)) return k;
        if (has_b && bary_of(Bm, q, l)) return k + 1;
    }
    return UINT32_MAX;
}

// Leaf walk (TrPLeaf.walk, tr_leaf_walk): start at the leaf's largest tet,
// step across the most violated face; a tet that accepts q with every
// barycentric >= TR_WALK_TAU and carries the CERTIFIED bit is the lowest
// index containing q (no lower-id tet of the leaf can accept it, and only
// the leaf's tets can: q is strictly inside the exclusive box).  Anything
// else -- an uncertified or marginal accept, a step out of the leaf, a
// revisit -- ends in the id-order scan, so the result is always K:119's.
// A regular cube: 1.67 record loads per sample instead of 3.33.
//
// pred (TrLeafPred rows, or NULL): approximate f32 barycentrics of the first
// tet relative to the exclusive box's corner `lo`; when they put q beyond a
// face the walk starts at the neighbour across it instead -- one record load
// for almost every sample (a wrong guess costs a step, never the result).
__device__ __forceinline__ uint32_t walk_leaf(const SceneK &S, const uint32_t *__restrict__ wt,
                                              uint32_t start, uint32_t count, const PQuery &q,
                                              double l[4], bool use_pred = false,
                                              float4 r1 = float4(), float4 r2 = float4(),
                                              float4 r3 = float4(), const float *lo = nullptr) {
    const uint32_t w4 = __ldg(wt + 4);
    if (w4 >> 31) {
        uint32_t i = w4 & 7u, seen = 0;
        if (use_pred) {
            const float x = (float)(q.x - (double)lo[0]), y = (float)(q.y - (double)lo[1]);
            const float z = (float)(q.z - (double)lo[2]);
            const float p1 = r1.x * x + r1.y * y + r1.z * z + r1.w;
            const float p2 = r2.x * x + r2.y * y + r2.z * z + r2.w;
            const float p3 = r3.x * x + r3.y * y + r3.z * z + r3.w;
            const float p0 = 1.0f - p1 - p2 - p3;
            int face = 0;
            float pm = p0;
            if (p1 < pm) { pm = p1; face = 1; }
            if (p2 < pm) { pm = p2; face = 2; }
            if (p3 < pm) { pm = p3; face = 3; }
            if (pm < -1e-4f) {
                const uint32_t e = (__ldg(wt + (i >> 1)) >> (16 * (i & 1u))) & 0xffffu;
                const uint32_t nb = (e >> (3 * face)) & 7u;
                if (nb < count) i = nb;
            }
        }
        for (uint32_t step = 0; step < count; ++step) {
            seen |= 1u << i;
            const uint32_t e = (__ldg(wt + (i >> 1)) >> (16 * (i & 1u))) & 0xffffu;
            if (bary_of(load_recm(S.tets, start + i), q, l)) {
                if (((e >> 12) & 1u) && l[0] >= TR_WALK_TAU && l[1] >= TR_WALK_TAU &&
                    l[2] >= TR_WALK_TAU && l[3] >= TR_WALK_TAU)
                    return start + i;
                break;
            }
            int face = 0;   // the most negative barycentric: q is beyond that face
            double lm = l[0];
            if (l[1] < lm) { lm = l[1]; face = 1; }
            if (l[2] < lm) { lm = l[2]; face = 2; }
            if (l[3] < lm) { face = 3; }
            const uint32_t nb = (e >> (3 * face)) & 7u;
            if (nb == i || ((seen >> nb) & 1u)) break;
            i = nb;
        }
    }
    return scan_leaf_first(S, start, count, q, l);
}

// Full-descent leaf scan: ids ascending; stop at the first id >= best.
__device__ __forceinline__ void scan_leaf_ids(const SceneK &S, uint32_t start, uint32_t count,
                                              const PQuery &q, uint32_t &best, uint32_t &best_pos,
                                              double l[4]) {
    for (uint32_t k = start; k < start + count; ++k) {
        const uint32_t t = S.pleaf_ids ? __ldg(S.pleaf_ids + k) : k;   // NULL: records in id order
        if (t >= best) break;
        double lt[4];
        if (bary_test(S.tets, k, q, lt)) {
            best = t;
            best_pos = k;
            l[0] = lt[0]; l[1] = lt[1]; l[2] = lt[2]; l[3] = lt[3];
            break;
        }
    }
}

// Full descent: lowest-index tet containing q (K:93-136 semantics), pruning
// subtrees whose minimum id cannot beat the best so far.  Returns the record
// position (UINT32_MAX if none) and the leaf it was found in.
__device__ uint32_t locate_full(const SceneK &S, const PQuery &q, double l[4], int32_t &leaf_out) {
    uint32_t best = UINT32_MAX, best_pos = UINT32_MAX;
    int32_t best_leaf = -1;
    const PQueryF qf = make_qf(q);
    int32_t st_node[PSTACK];
    uint32_t st_min[PSTACK];
    int sp = 0;
    int32_t node = 0;
    while (true) {
        const float4 *np = reinterpret_cast<const float4 *>(S.pnodes + node);
        const float4 A = __ldg(np + 0), B = __ldg(np + 1), C = __ldg(np + 2);
        const int4 D = __ldg(reinterpret_cast<const int4 *>(np + 3));
        const int32_t c0 = D.x, c1 = D.y;
        const uint32_t m0 = (uint32_t)D.z, m1 = (uint32_t)D.w;
        bool h0 = m0 < best && in_box(qf, A.x, A.y, A.z, A.w, B.x, B.y);
        bool h1 = c1 != CHILD_NONE && m1 < best && in_box(qf, B.z, B.w, C.x, C.y, C.z, C.w);
        if (h0 && c0 < 0) {
            const uint32_t before = best;
            const TrPLeaf *lf = S.pleaves + (~c0);
            scan_leaf_ids(S, __ldg(&lf->start), __ldg(&lf->count), q, best, best_pos, l);
            if (best != before) best_leaf = ~c0;
            h0 = false;
        }
        if (h1 && c1 < 0) {
            const uint32_t before = best;
            const TrPLeaf *lf = S.pleaves + (~c1);
            scan_leaf_ids(S, __ldg(&lf->start), __ldg(&lf->count), q, best, best_pos, l);
            if (best != before) best_leaf = ~c1;
            h1 = false;
        }
        h0 = h0 && m0 < best;
        h1 = h1 && m1 < best;
        if (h0 && h1) {
            // descend into the lower-min-id child first, defer the other
            if (m0 <= m1) { node = c0; st_node[sp] = c1; st_min[sp] = m1; }
            else { node = c1; st_node[sp] = c0; st_min[sp] = m0; }
            ++sp;
            continue;
        }
        if (h0) { node = c0; continue; }
        if (h1) { node = c1; continue; }
        bool found = false;
        while (sp > 0) {
            --sp;
            if (st_min[sp] < best) { node = st_node[sp]; found = true; break; }
        }
        if (!found) break;
    }
    leaf_out = best_leaf;
    return best_pos;
}

// Cell candidate lists (tr_cells_build; unstructured meshes): the cell's
// records are every tet whose padded box meets the cell, in ascending id, so
// the first one whose box holds q and which accepts q is the lowest-index
// containing tet (K:93-136).  Outside the cell grid no padded box can hold q.
// Returns false when the cell overflowed (the caller runs the BVH descent).
__device__ __forceinline__ bool locate_cells(const SceneK &S, const PQuery &q, double l[4],
                                             uint32_t &pos) {
    pos = UINT32_MAX;
    int64_t c[3];
    const double qv[3] = {q.x, q.y, q.z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double f = (qv[a] - S.corg[a]) * S.cscale[a];   // the builder's expression
        const double dim = (double)S.cdim[a];
        if (!(f >= 0.0) || f >= dim * (1.0 + 1e-12)) return true;   // outside every padded box
        const int64_t ci = (int64_t)f;
        c[a] = ci < S.cdim[a] ? ci : S.cdim[a] - 1;
    }
    const int64_t cell = (c[0] * S.cdim[1] + c[1]) * S.cdim[2] + c[2];
    const uint32_t o0 = __ldg(S.cell_off + cell), o1 = __ldg(S.cell_off + cell + 1) & 0x7fffffffu;
    if (o0 & 0x80000000u) return false;
    const PQueryF qf = make_qf(q);
    for (uint32_t k = o0; k < o1; ++k) {
        const uint32_t r = __ldg(S.cell_recs + k);
        const float4 b0 = __ldg(S.tbox + 2 * r), b1 = __ldg(S.tbox + 2 * r + 1);
        if (!in_box(qf, b0.x, b0.y, b0.z, b0.w, b1.x, b1.y)) continue;
        if (bary_test(S.tets, r, q, l)) { pos = r; return true; }
    }
    return true;
}

struct LeafHint {  // the ray's current leaf: exclusive box + record range, in registers
    float lo[3], hi[3];
    uint32_t start, count;
    const TrPLeaf *hdr;   // the header (walk table)
    bool valid;
};

__device__ __forceinline__ void load_hint(const SceneK &S, int32_t leaf, LeafHint &h) {
    const float4 *p = reinterpret_cast<const float4 *>(S.pleaves + leaf);
    const float4 a = __ldg(p), b = __ldg(p + 1);
    h.lo[0] = a.x; h.lo[1] = a.y; h.lo[2] = a.z;
    h.hi[0] = a.w; h.hi[1] = b.x; h.hi[2] = b.y;
    h.start = __float_as_uint(b.z);
    h.count = __float_as_uint(b.w);
    h.hdr = S.pleaves + leaf;
    h.valid = true;
}

// Grid cell of q (-1: outside the grid).  The cell's candidate leaf is only a
// hint: the caller accepts it after proving q strictly inside its exclusive box.
__device__ __forceinline__ int64_t grid_cell(const SceneK &S, const PQuery &q,
                                             int *parity = nullptr) {
    const double fx = (q.x - S.gorg[0]) * S.gscale[0];
    const double fy = (q.y - S.gorg[1]) * S.gscale[1];
    const double fz = (q.z - S.gorg[2]) * S.gscale[2];
    if (!(fx >= 0.0 && fy >= 0.0 && fz >= 0.0)) return -1;
    const int64_t cx = (int64_t)fx, cy = (int64_t)fy, cz = (int64_t)fz;
    if (cx >= S.gdim[0] || cy >= S.gdim[1] || cz >= S.gdim[2]) return -1;
    if (parity) *parity = (int)((cx + cy + cz) & 1);
    return (cx * S.gdim[1] + cy) * S.gdim[2] + cz;
}

__device__ __forceinline__ void load_leaf(const TrPLeaf *lf, LeafHint &h) {
    const double4 v = ldg256(lf);   // 8 x 32 bit: ex_lo[3], ex_hi[3], start, count
    const long long w0 = __double_as_longlong(v.x), w1 = __double_as_longlong(v.y);
    const long long w2 = __double_as_longlong(v.z), w3 = __double_as_longlong(v.w);
    h.lo[0] = __int_as_float((int)w0); h.lo[1] = __int_as_float((int)(w0 >> 32));
    h.lo[2] = __int_as_float((int)w1); h.hi[0] = __int_as_float((int)(w1 >> 32));
    h.hi[1] = __int_as_float((int)w2); h.hi[2] = __int_as_float((int)(w2 >> 32));
    h.start = (uint32_t)w3;
    h.count = (uint32_t)((unsigned long long)w3 >> 32);
    h.hdr = lf;
    h.valid = true;
}

// K:139-154.  Returns the record position (UINT32_MAX: outside every tet).
// Order: the ray's current exclusive leaf (registers), the grid's candidate
// leaf, else the full descent.  All three return the lowest containing index.
__device__ __forceinline__ uint32_t field_at(const SceneK &S, const PQuery &q, LeafHint &hint,
                                             bool use_hint, bool use_grid, double &v,
                                             bool stats = false, bool grid_indirect = false) {
    double l[4];
    uint32_t pos;
    bool done = false;
    if (use_hint && hint.valid && strictly_in(q, hint.lo, hint.hi)) {
        pos = walk_leaf(S, hint.hdr->walk, hint.start, hint.count, q, l);
        done = true;
    } else if (use_grid) {
        const int64_t gc = grid_cell(S, q);
        if (gc >= 0) {
            LeafHint h;
            if (grid_indirect) {
                const int32_t gl = __ldg(S.pgrid + gc);
                h.valid = false;
                if (gl >= 0) load_leaf(S.pleaves + gl, h);
                else { h.lo[0] = 1.0f; h.hi[0] = 0.0f; h.lo[1] = h.lo[2] = h.hi[1] = h.hi[2] = 0.0f; }
            } else {
                load_leaf(S.pgrid_leaf + gc, h);  // one load: the header is replicated per cell
            }
            if (strictly_in(q, h.lo, h.hi)) {
                pos = walk_leaf(S, h.hdr->walk, h.start, h.count, q, l);
                if (use_hint) hint = h;
                done = true;
                if (stats) atomicAdd(&g_stats[ST_GRID_HIT], 1ull);
            }
        }
    }
    if (!done && use_grid && S.cell_off) done = locate_cells(S, q, l, pos);
    if (!done) {
        int32_t leaf;
        if (stats) atomicAdd(&g_stats[ST_DESCENT], 1ull);
        pos = locate_full(S, q, l, leaf);
        if (use_hint && leaf >= 0) load_hint(S, leaf, hint);
    }
    if (pos == UINT32_MAX) { v = 0.0; return pos; }
    const double2 *r = reinterpret_cast<const double2 *>(S.tets + pos);
    if (S.centering == 0) {
        const double2 f01 = __ldg(r + 6), f23 = __ldg(r + 7);
        v = l[0] * f01.x + l[1] * f01.y + l[2] * f23.x + l[3] * f23.y;
    } else {
        v = __ldg(r + 6).x;
    }
    return pos;
}

// K:74-90.  SHARED: T is the march's shared-memory copy of the table.
template <bool SHARED = false>
__device__ __forceinline__ void tf_sample(const double *__restrict__ T, int64_t n, double lo,
                                          double hi, double v, double c[4]) {
    const double u = (v - lo) / (hi - lo) * (double)(n - 1);
    int64_t j;
    double f;
    bool interp = true;
    if (u <= 0.0) { j = 0; interp = false; }
    else if (u >= (double)(n - 1)) { j = n - 1; interp = false; }
    else { j = (int64_t)floor(u); }
    const double4 a = SHARED ? *reinterpret_cast<const double4 *>(T + 4 * j) : ldg256(T + 4 * j);
    if (!interp) { c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w; return; }
    f = u - (double)j;
    const double4 b = SHARED ? *reinterpret_cast<const double4 *>(T + 4 * j + 4)
                             : ldg256(T + 4 * j + 4);
    c[0] = a.x + f * (b.x - a.x);
    c[1] = a.y + f * (b.y - a.y);
    c[2] = a.z + f * (b.z - a.z);
    c[3] = a.w + f * (b.w - a.w);
}

struct EpochK {
    const uint8_t *__restrict__ knode_active;
    const uint8_t *__restrict__ active;
    const uint8_t *__restrict__ bnode_active;
    const double *__restrict__ step;
    const double *__restrict__ step_ratio;  // (P,2): step, step / s1
    const double *__restrict__ tf;
    int64_t n_tf;
    double tf_lo, tf_hi;
};

struct Acc {
    double r, g, b, a;
};

// K:173-230: first active partition interval, lexicographic min (clamped
// t_enter, pid) among partitions with t_exit > t_min + excl_eps.
__device__ int32_t next_interval(const SceneK &S, const EpochK &E, const RayD &ray, double t_min,
                                 double excl_eps, int32_t excl_id, double &ra, double &rb) {
    int32_t best_id = -1;
    double best_a = INFINITY, best_b = INFINITY;
    const double thr = t_min + excl_eps;
    int32_t st_node[BSTACK];
    double st_a[BSTACK];
    int sp = 0;
    int32_t node = 0;
    double node_a = -INFINITY;
    while (true) {
        if (node_a <= best_a) {
            const TrBNode *N = S.bnodes + node;
            const uint32_t act = __ldg(E.bnode_active + node);
            const int2 ch = __ldg(reinterpret_cast<const int2 *>(&N->child[0]));
            int32_t push_n[2];
            double push_a[2];
            int np = 0;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int32_t child = c == 0 ? ch.x : ch.y;
                if (!((act >> c) & 1u)) continue;  // CHILD_NONE has a clear bit
                const double2 *bp = reinterpret_cast<const double2 *>(&N->box[c][0]);
                const double2 b0 = __ldg(bp), b1 = __ldg(bp + 1), b2 = __ldg(bp + 2);
                const double lo[3] = {b0.x, b0.y, b1.x}, hi[3] = {b1.y, b2.x, b2.y};
                double a, b;
                slab(ray, lo, hi, a, b);
                if (a > b) continue;
                if (b <= thr) continue;
                const double a_cl = (a > t_min) ? a : t_min;
                if (a_cl >= INFINITY) continue;  // t_max = inf (K:366)
                if (a_cl > best_a) continue;
                if (child < 0) {
                    const int32_t pid = ~child;
                    if (pid == excl_id) continue;
                    if (a_cl < best_a || (a_cl == best_a && pid < best_id)) {
                        best_id = pid;
                        best_a = a_cl;
                        best_b = b;
                    }
                } else {
                    push_n[np] = child;
                    push_a[np] = a_cl;
                    ++np;
                }
            }
            if (np == 2) {  // visit the nearer child first
                const int near = push_a[1] < push_a[0] ? 1 : 0;
                st_node[sp] = push_n[1 - near];
                st_a[sp] = push_a[1 - near];
                ++sp;
                node = push_n[near];
                node_a = push_a[near];
                continue;
            }
            if (np == 1) { node = push_n[0]; node_a = push_a[0]; continue; }
        }
        if (sp == 0) break;
        --sp;
        node = st_node[sp];
        node_a = st_a[sp];
    }
    ra = best_a;
    rb = best_b;
    return best_id;
}

// ------------------------------------------------------ BSP interval trace

constexpr int KBUF = 16;
constexpr int KSTACK = 32;

// Exact front-to-back interval sequence of one ray from a resumable BSP
// traversal.  A partition's box lies inside its BSP cell, so the entry of the
// nearest pending cell lower-bounds the clamped entry of every partition not
// yet enumerated: next_interval's winner (K:173-230: min (clamped entry, pid)
// among active partitions with exit > t_min + excl, excluding the last one)
// is certain once it beats max(that bound, t_min) strictly.
struct BspTrace {
    int32_t st_node[KSTACK];
    double st_tn[KSTACK], st_tf[KSTACK];
    int sp;
    int32_t c_pid[KBUF];
    double c_pa[KBUF], c_pb[KBUF];
    int nb;
    int cells;
    int nodes;
    bool overflow;
};

__device__ __forceinline__ double ray_o(const RayD &r, int a) { return a == 0 ? r.ox : (a == 1 ? r.oy : r.oz); }
__device__ __forceinline__ double ray_d(const RayD &r, int a) { return a == 0 ? r.dx : (a == 1 ? r.dy : r.dz); }
__device__ __forceinline__ double ray_i(const RayD &r, int a) { return a == 0 ? r.ix : (a == 1 ? r.iy : r.iz); }

__device__ __forceinline__ void bsp_begin(const SceneK &S, const RayD &ray, BspTrace &T) {
    T.sp = 0;
    T.nb = 0;
    T.cells = 0;
    T.nodes = 0;
    T.overflow = false;
    double r0, r1;
    slab(ray, S.kroot_lo, S.kroot_hi, r0, r1);
    if (r0 <= r1 && r1 > 0.0) {
        T.st_node[0] = 0; T.st_tn[0] = r0; T.st_tf[0] = r1;
        T.sp = 1;
    }
}

// Pop subtrees until one leaf cell has been enumerated into the buffer.
// COUNT: node / cell statistics (TR_FLAG_STATS builds only: T is in local
// memory, so each counter update is a local load and store).
template <bool COUNT>
__device__ void bsp_enumerate_next(const SceneK &S, const EpochK &E, const RayD &ray, BspTrace &T) {
    while (T.sp > 0) {
        --T.sp;
        int32_t node = T.st_node[T.sp];
        double tn = T.st_tn[T.sp], tf = T.st_tf[T.sp];
        bool leaf_done = false;
        while (true) {
            if (tf <= 0.0) break;                         // behind the origin: exits <= 0
            if (COUNT) ++T.nodes;
            const TrKNode *N = S.knodes + node;
            const int32_t info = __ldg(&N->info);   // issued with the activity byte
            if (E.knode_active && !__ldg(E.knode_active + node)) break;
            if (info < 0) {                                // leaf cell: its partitions
                if (COUNT) ++T.cells;
                const int32_t st = ~info, cnt = __ldg(&N->aux);
                for (int32_t k = 0; k < cnt; ++k) {
                    const int32_t pid = __ldg(S.kleaf_pids + st + k);
                    if (!__ldg(E.active + pid)) continue;
                    const double lo[3] = {__ldg(S.part_lo + 3 * pid), __ldg(S.part_lo + 3 * pid + 1),
                                          __ldg(S.part_lo + 3 * pid + 2)};
                    const double hi[3] = {__ldg(S.part_hi + 3 * pid), __ldg(S.part_hi + 3 * pid + 1),
                                          __ldg(S.part_hi + 3 * pid + 2)};
                    double pa, pb;
                    slab(ray, lo, hi, pa, pb);
                    if (pa > pb || !(pb > 0.0)) continue;
                    if (T.nb == KBUF) { T.overflow = true; return; }
                    T.c_pid[T.nb] = pid; T.c_pa[T.nb] = pa; T.c_pb[T.nb] = pb;
                    ++T.nb;
                }
                leaf_done = true;
                break;
            }
            const int axis = info & 3;
            const double sp = __ldg(&N->split);
            const int32_t left = node + 1, right = info >> 2;
            const double d = ray_d(ray, axis), o = ray_o(ray, axis);
            if (d == 0.0) {                                // parallel: one side, or both on the plane
                if (o < sp) { node = left; continue; }
                if (o > sp) { node = right; continue; }
                if (T.sp == KSTACK) { T.overflow = true; return; }
                T.st_node[T.sp] = right; T.st_tn[T.sp] = tn; T.st_tf[T.sp] = tf; ++T.sp;
                node = left;
                continue;
            }
            const double ts = (sp - o) * ray_i(ray, axis);
            const int32_t nearc = d > 0.0 ? left : right, farc = d > 0.0 ? right : left;
            if (ts < tn) { node = farc; continue; }
            if (ts > tf) { node = nearc; continue; }
            if (T.sp == KSTACK) { T.overflow = true; return; }
            T.st_node[T.sp] = farc; T.st_tn[T.sp] = ts; T.st_tf[T.sp] = tf; ++T.sp;
            node = nearc;
            tf = ts;
        }
        if (leaf_done) return;
    }
}

// next_interval (K:173-230) from the BSP state; -1 when the ray is done.
template <bool COUNT>
__device__ int32_t bsp_next_interval(const SceneK &S, const EpochK &E, const RayD &ray,
                                     BspTrace &T, double t_min, double excl, int32_t last,
                                     double &ra, double &rb) {
    const double thr = t_min + excl;
    while (true) {
        int32_t best = -1;
        double best_a = INFINITY, best_b = INFINITY;
        for (int i = 0; i < T.nb; ++i) {
            const int32_t pid = T.c_pid[i];
            const double pb = T.c_pb[i];
            if (pid == last || pb <= thr) continue;
            const double pa = T.c_pa[i];
            const double a_cl = (pa > t_min) ? pa : t_min;
            if (a_cl < best_a || (a_cl == best_a && pid < best)) { best = pid; best_a = a_cl; best_b = pb; }
        }
        if (T.sp == 0) {
            ra = best_a; rb = best_b;
            return best;
        }
        const double tn = T.st_tn[T.sp - 1];
        const double bound = (tn > t_min) ? tn : t_min;
        if (best >= 0 && best_a < bound) {
            ra = best_a; rb = best_b;
            return best;
        }
        bsp_enumerate_next<COUNT>(S, E, ray, T);
        if (T.overflow) return -1;
    }
}

// Drop candidates that no later query can return (exit behind the new t_min).
__device__ __forceinline__ void bsp_compact(BspTrace &T, double t_min) {
    int w = 0;
    for (int i = 0; i < T.nb; ++i) {
        if (T.c_pb[i] < t_min) continue;
        T.c_pid[w] = T.c_pid[i]; T.c_pa[w] = T.c_pa[i]; T.c_pb[w] = T.c_pb[i];
        ++w;
    }
    T.nb = w;
}

// K:300-309 with numba's 64-bit integer promotion.
__device__ __forceinline__ double hash01(int64_t ix, int64_t iy) {
    uint64_t h = ((uint64_t)(uint32_t)ix * 73856093ull) ^ ((uint64_t)(uint32_t)iy * 19349663ull);
    h = (h ^ 61ull) ^ (h >> 16);
    h = h * 9ull;
    h = h ^ (h >> 4);
    h = h * 0x27D4EB2Dull;
    h = h ^ (h >> 15);
    return __ull2double_rn(h) / 4294967296.0;
}


struct FrameK {
    TrFrame f;
    int64_t tiles_x, n_tiles, my_tiles;
    int64_t ray_begin, n_rays;   // this chunk: rays [ray_begin, ray_begin + n_rays) in tile order
    int32_t n_parts;
    int32_t auto_g;              // lanes per ray chosen on the device (march_lane_choice)
    int64_t march_lanes;         // resident march lanes (CTAs x threads) for that choice
    int32_t defer_bg;            // background pixels go to background_kernel (host framebuffer)
    int32_t use_cand;            // modes 1/2: intervals from the rasterised candidate lists
    int32_t raster_sub;          // warps per partition rectangle in the candidate raster
    // brick-sharded frame (tr_brick_*; B_on = 0 otherwise)
    int32_t B_on, B_rank, B_n, B_write_bg, B_zero_foreign;
    const int16_t *B_owner;
    const double *B_lo, *B_hi;
    TrRayState *B_state;
    uint32_t *B_queue, *B_ctr;
    // PEER exchange (B_npeers > 0): states pushed to the peers' inboxes
    uint32_t B_tag;
    int32_t B_npeers;
    TrRayState *const *B_peer_inbox;
    TrRayState *B_inbox;
};

// One stored interval of a ray (16 B): next_interval's clamped entry, the
// partition, and the ray's inclusive prefix count of march_range samples.
struct __align__(16) IvRec {
    double a;
    int32_t pid;     // -1: reference mode's mesh-box interval (K:346-353)
    uint32_t cum;
};
constexpr uint32_t CUM_MAX = 0x7fffffffu;   // longer lists continue inline in the march
constexpr uint32_t CNT_MORE = 0x80000000u;  // cnt word: intervals past the stored list

struct IvBuf {                   // per-chunk scratch
    IvRec *rec;                  // [n_rays][IV_CAP], ray-major
    uint32_t *cnt;               // [n_rays]: n | bucket << 16 | CNT_MORE
    double *tail;                // [n_rays]: t_min after the last stored interval (CNT_MORE only)
    uint32_t *order;             // marching rays, most expensive first
    uint32_t *hist, *cursor;     // [N_BUCKETS] each; bucket 0 = nothing to march
    uint32_t *trace_ctr;         // next 32-ray tile of the trace pass
    unsigned long long *ray_stats;  // [0] sum, [1] max of the rays' stored sample counts
    uint32_t *gsel;              // lanes per ray chosen for this chunk (auto mode)
    uint32_t *n_bg;              // deferred background rays, listed from the top of `order`
    double *cand_pa, *cand_pb;   // [CAND_CAP][n_rays] active partition slabs (use_cand), slot-major
    int32_t *cand_pid;           //   so a warp's 32 rays read one slot in one coalesced load
    float *cand_nkey;            // [CAND_CAP][n_rays] the next slot's sort key (+inf after the last)
    uint32_t *ccount;            // [n_rays] slabs found (> CAND_CAP: the ray takes the BSP)
    double *rinv;                // [3][n_rays] 1/d per axis (0 where d == 0) for the raster
    unsigned long long *totals;  // frame totals (trace-finished rays add their visited)
};

__device__ __forceinline__ uint32_t cost_bucket(double cost) {
    if (!(cost > 0.0)) return 0;
    const int b = (int)(4.0f * __log2f((float)cost + 1.0f));
    return (uint32_t)(b < 1 ? 1 : (b < N_BUCKETS - 1 ? b : N_BUCKETS - 1));
}

struct Pixel {
    int64_t ix, iy, out;
    bool valid;
};

// chunk-local ray index -> pixel (8x4 tiles, tile t of rank r is slot t/count)
__device__ __forceinline__ Pixel ray_pixel(const FrameK &F, int64_t rr) {
    const TrFrame &fr = F.f;
    const int64_t g = F.ray_begin + rr;
    const int64_t j = g >> 5;
    const int lane = (int)(g & 31);
    const int64_t tile = (int64_t)fr.shard_rank + (int64_t)fr.shard_count * j;
    Pixel p;
    p.ix = (tile % F.tiles_x) * TILE_W + (lane % TILE_W);
    p.iy = (tile / F.tiles_x) * TILE_H + (lane / TILE_W);
    p.valid = j < F.my_tiles && p.ix < fr.width && p.iy < fr.height;
    p.out = fr.compact ? g : p.iy * fr.width + p.ix;
    return p;
}

// K:330-339 (left-to-right evaluation, no contraction)
__device__ __forceinline__ RayD make_ray(const TrFrame &fr, int64_t ix, int64_t iy) {
    const double sx = (((double)ix + 0.5) / (double)fr.width) * 2.0 - 1.0;
    const double sy = 1.0 - (((double)iy + 0.5) / (double)fr.height) * 2.0;
    double dx = fr.cam_fwd[0] + sx * fr.aspect * fr.tan_half * fr.cam_right[0] + sy * fr.tan_half * fr.cam_up[0];
    double dy = fr.cam_fwd[1] + sx * fr.aspect * fr.tan_half * fr.cam_right[1] + sy * fr.tan_half * fr.cam_up[1];
    double dz = fr.cam_fwd[2] + sx * fr.aspect * fr.tan_half * fr.cam_right[2] + sy * fr.tan_half * fr.cam_up[2];
    const double dn = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
    dx *= dn; dy *= dn; dz *= dn;
    RayD ray;
    ray.ox = fr.cam_pos[0]; ray.oy = fr.cam_pos[1]; ray.oz = fr.cam_pos[2];
    ray.dx = dx; ray.dy = dy; ray.dz = dz;
    ray.nx = dx != 0.0; ray.ny = dy != 0.0; ray.nz = dz != 0.0;
    ray.ix = ray.nx ? 1.0 / dx : 0.0;
    ray.iy = ray.ny ? 1.0 / dy : 0.0;
    ray.iz = ray.nz ? 1.0 / dz : 0.0;
    return ray;
}

// Samples march_range takes on [a, b): k = 0 always, then every k >= 1 with
// t_k = a + (k + phase) * step < b (K:277-280).  fl(a + fl(fl(k + phase) *
// step)) is monotone in k, so the count is the first k >= 1 with t_k >= b,
// found from the real-valued estimate and corrected with the exact expression.
__device__ __forceinline__ int64_t interval_samples(double a, double b, double step,
                                                    double phase) {
    const double est = ceil((b - a) / step - phase);
    int64_t k = (est > 1.0) ? (int64_t)fmin(est, 4.0e15) : 1;
    while (k > 1 && a + ((double)(k - 1) + phase) * step >= b) --k;
    while (a + ((double)k + phase) * step < b) ++k;
    return k;
}

__device__ __forceinline__ void write_pixel(const TrFrame &fr, const TrOutputs &O, int64_t out,
                                            const Acc &acc, int64_t samples, int32_t visited) {
    const double r = acc.r + (1.0 - acc.a) * fr.bg[0];  // K:393-396
    const double g = acc.g + (1.0 - acc.a) * fr.bg[1];
    const double bl = acc.b + (1.0 - acc.a) * fr.bg[2];
    const double al = acc.a + (1.0 - acc.a) * fr.bg[3];
    double *px = O.rgba + 4 * out;
    if ((reinterpret_cast<uintptr_t>(px) & 31) == 0) {
        // one 32-byte store: one PCIe write when the framebuffer is host memory
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};"
                     :: "l"(px), "d"(r), "d"(g), "d"(bl), "d"(al) : "memory");
    } else {
        reinterpret_cast<double2 *>(px)[0] = make_double2(r, g);
        reinterpret_cast<double2 *>(px)[1] = make_double2(bl, al);
    }
    O.samples[out] = samples;
    O.visited[out] = visited;
}

// Mode 0 under brick sharding: the mesh-box interval [ta, b) cut where the
// ray leaves each brick box (front to back).  Every record keeps a = ta and
// pid = -1 - brick; cum = samples with t < the brick's exit (the forced
// k = 0 sample counts in the first), the last = ns.  The march takes the
// sample index itself as k in mode 0, so positions are unchanged.
__device__ uint32_t brick_cut(const FrameK &F, const RayD &ray, double ta, double b, double phase,
                              int64_t ns, IvRec *rec) {
    constexpr int MAXB = 64;
    double ex[MAXB];
    int16_t id[MAXB];
    int m = 0;
    for (int k = 0; k < F.B_n && k < MAXB; ++k) {
        const double lo[3] = {F.B_lo[3 * k], F.B_lo[3 * k + 1], F.B_lo[3 * k + 2]};
        const double hi[3] = {F.B_hi[3 * k], F.B_hi[3 * k + 1], F.B_hi[3 * k + 2]};
        double ea, eb;
        slab(ray, lo, hi, ea, eb);
        if (ea > eb || eb <= ta || ea >= b) continue;
        // insertion by exit (convex, disjoint boxes: exits order like entries)
        int q = m++;
        while (q > 0 && ex[q - 1] > eb) { ex[q] = ex[q - 1]; id[q] = id[q - 1]; --q; }
        ex[q] = eb; id[q] = (int16_t)k;
    }
    if (m == 0) { ex[0] = b; id[0] = 0; m = 1; }   // degenerate: the whole interval on brick 0
    uint32_t n = 0;
    for (int q = 0; q < m; ++q) {
        int64_t c = (q == m - 1 || ex[q] >= b) ? ns : interval_samples(ta, ex[q], F.f.s1, phase);
        if (c > ns) c = ns;
        IvRec r; r.a = ta; r.pid = -1 - (int32_t)id[q]; r.cum = (uint32_t)c;
        rec[n++] = r;
        if (c == ns) break;
    }
    return n;
}

// next_interval (K:173-230) over the ray's complete candidate list: the
// active partitions whose slab it hits.  Same rule as the BVH / BSP
// enumerations: skip the excluded id and exits <= t_min + excl, winner = the
// lexicographic minimum of (max(entry, t_min), pid).
// The last 4-slot group a ray loaded (consecutive intervals mostly reuse it).
struct CandWin {
    uint32_t base;   // first slot (a multiple of 4); UINT32_MAX: empty
    double pa[4], pb[4];
    int32_t pid[4];
    float nkey3;     // sort key of slot base + 4
};

__device__ __forceinline__ int32_t cand_next_interval(const IvBuf &iv, int64_t n_rays, int64_t rr,
                                                      uint32_t n, uint32_t &dead, double &dead_thr,
                                                      CandWin &w, double t_min, double excl,
                                                      int32_t last, double &ra, double &rb) {
    const double thr = t_min + excl;
    int32_t best = -1;
    double best_a = INFINITY, best_b = INFINITY;
    // skip the prefix whose exits are <= thr: still dead while thr >= the
    // threshold they were skipped at (fl(fl(b - eps) + eps) can step back an ulp)
    if (thr < dead_thr) dead = 0;
    dead_thr = thr;
    bool prefix = true;   // still in the run of dead slots from `dead`
    // aligned groups; slots below `dead` in the first one are dead again
    for (uint32_t i0 = dead & ~3u; i0 < n; i0 += 4) {
        if (w.base != i0) {
            w.base = i0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {   // four slots' loads in flight together
                const int64_t o = (int64_t)(i0 + u) * n_rays + rr;
                const bool ok = i0 + u < n;
                w.pa[u] = ok ? __ldg(iv.cand_pa + o) : 0.0;
                w.pb[u] = ok ? __ldg(iv.cand_pb + o) : -INFINITY;
                w.pid[u] = ok ? __ldg(iv.cand_pid + o) : -1;
            }
            w.nkey3 = i0 + 4 < n ? __ldg(iv.cand_nkey + (int64_t)(i0 + 3) * n_rays + rr) : INFINITY;
        }
        const double *pa = w.pa, *pb = w.pb;
        const int32_t *pid = w.pid;
        // slots ascend by entry rounded down to float: nothing later can win
        if ((double)__double2float_rd(pa[0]) > best_a) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (pb[u] <= thr) {   // dead for good (also the padding, pb = -inf)
                if (prefix && i0 + u + 1 > dead) dead = min(i0 + u + 1, n);
                continue;
            }
            prefix = false;
            if (pid[u] == last) continue;
            const double a_cl = (pa[u] > t_min) ? pa[u] : t_min;
            if (a_cl >= INFINITY) continue;   // t_max = inf (K:366)
            if (a_cl < best_a || (a_cl == best_a && pid[u] < best)) { best = pid[u]; best_a = a_cl; best_b = pb[u]; }
        }
        // the next group's first key (kept with this group's last slot)
        // bounds every later slot: stop without loading it
        if (i0 + 4 < n && (double)w.nkey3 > best_a) break;
    }
    ra = best_a;
    rb = best_b;
    return best;
}

// chunk-local ray of pixel (ix, iy), -1 if another rank's or chunk's
__device__ __forceinline__ int64_t pixel_ray(const FrameK &F, uint32_t ix, uint32_t iy) {
    uint32_t tile = (iy / TILE_H) * (uint32_t)F.tiles_x + ix / TILE_W;
    const uint32_t cnt = (uint32_t)F.f.shard_count;
    if (cnt > 1) {
        if (tile % cnt != (uint32_t)F.f.shard_rank) return -1;
        tile /= cnt;
    }
    const int64_t g = (int64_t)tile * 32 + (iy % TILE_H) * TILE_W + (ix % TILE_W) - F.ray_begin;
    return (g >= 0 && g < F.n_rays) ? g : -1;
}

// 1/d per axis of every ray of the chunk (make_ray, K:330-338) for the raster.
__global__ void __launch_bounds__(256) ray_table_kernel(FrameK F, IvBuf iv) {
    const int64_t rr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (rr >= F.n_rays) return;
    iv.ccount[rr] = 0;
    const Pixel px = ray_pixel(F, rr);
    double a = 0.0, b = 0.0, c = 0.0;
    if (px.valid) {
        const RayD ray = make_ray(F.f, px.ix, px.iy);
        a = ray.ix; b = ray.iy; c = ray.iz;
    }
    iv.rinv[rr] = a;
    iv.rinv[F.n_rays + rr] = b;
    iv.rinv[2 * F.n_rays + rr] = c;
}

// Candidate raster: one CTA per active partition walks the pixels of its
// box's screen rectangle (conservative: corners projected, 2 px margin, the
// whole frame if a corner is not in front of the camera) and appends the
// partition to every ray whose exact slab test (the trace's own make_ray and
// slab) hits it with an exit > 0.  Work is spread over partitions x pixels,
// so no ray's front-to-back walk sets the pass time.
__global__ void __launch_bounds__(256, 4) cand_raster_kernel(SceneK S, EpochK E, FrameK F, IvBuf iv) {
    const TrFrame &fr = F.f;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    // work item = (partition, sub): `sub` takes every RASTER_SUB-th row of
    // the partition's rectangle, so large rectangles spread over warps
    const int64_t nsub = F.raster_sub;
    for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < F.n_parts * nsub; u += warps) {
        const int64_t pid = u / nsub, sub = u % nsub;
        if (!__ldg(E.active + pid)) continue;   // warp-uniform
        const double lo[3] = {__ldg(S.part_lo + 3 * pid), __ldg(S.part_lo + 3 * pid + 1), __ldg(S.part_lo + 3 * pid + 2)};
        const double hi[3] = {__ldg(S.part_hi + 3 * pid), __ldg(S.part_hi + 3 * pid + 1), __ldg(S.part_hi + 3 * pid + 2)};
        // lanes 0-7 project one box corner each
        double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
        bool full = false;
        if (lane < 8) {
            const int c = lane;
            const double v[3] = {((c & 1) ? hi[0] : lo[0]) - fr.cam_pos[0],
                                 ((c & 2) ? hi[1] : lo[1]) - fr.cam_pos[1],
                                 ((c & 4) ? hi[2] : lo[2]) - fr.cam_pos[2]};
            const double z = v[0] * fr.cam_fwd[0] + v[1] * fr.cam_fwd[1] + v[2] * fr.cam_fwd[2];
            const double len = fabs(v[0]) + fabs(v[1]) + fabs(v[2]);
            if (!(z > 1e-6 * len)) {
                full = true;
            } else {
                const double sx = (v[0] * fr.cam_right[0] + v[1] * fr.cam_right[1] + v[2] * fr.cam_right[2]) /
                                  z / (fr.aspect * fr.tan_half);
                const double sy = (v[0] * fr.cam_up[0] + v[1] * fr.cam_up[1] + v[2] * fr.cam_up[2]) / z / fr.tan_half;
                x0 = x1 = (sx + 1.0) * 0.5 * (double)fr.width - 0.5;
                y0 = y1 = (1.0 - sy) * 0.5 * (double)fr.height - 0.5;
            }
        }
        full = __any_sync(FULL, full);
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) {
            x0 = fmin(x0, __shfl_xor_sync(FULL, x0, off)); x1 = fmax(x1, __shfl_xor_sync(FULL, x1, off));
            y0 = fmin(y0, __shfl_xor_sync(FULL, y0, off)); y1 = fmax(y1, __shfl_xor_sync(FULL, y1, off));
        }
        x0 = __shfl_sync(FULL, x0, 0); x1 = __shfl_sync(FULL, x1, 0);
        y0 = __shfl_sync(FULL, y0, 0); y1 = __shfl_sync(FULL, y1, 0);
        int64_t ix0 = 0, ix1 = fr.width - 1, iy0 = 0, iy1 = fr.height - 1;
        if (!full) {
            if (!(x1 >= -2.0) || !(x0 <= (double)fr.width + 1.0) || !(y1 >= -2.0) ||
                !(y0 <= (double)fr.height + 1.0))
                continue;   // off screen
            ix0 = (int64_t)fmax(floor(x0) - 2.0, 0.0);
            ix1 = (int64_t)fmin(ceil(x1) + 2.0, (double)(fr.width - 1));
            iy0 = (int64_t)fmax(floor(y0) - 2.0, 0.0);
            iy1 = (int64_t)fmin(ceil(y1) + 2.0, (double)(fr.height - 1));
        }
        // only the pixel rows of this ray chunk's tiles
        const int64_t cnt = fr.shard_count;
        const int64_t t_first = fr.shard_rank + cnt * (F.ray_begin >> 5);
        const int64_t t_last = fr.shard_rank + cnt * ((F.ray_begin + F.n_rays - 1) >> 5);
        iy0 = max(iy0, (t_first / F.tiles_x) * TILE_H);
        iy1 = min(iy1, (t_last / F.tiles_x) * TILE_H + TILE_H - 1);
        iy0 += sub;   // this warp's rows: iy0 + sub, iy0 + sub + nsub, ...
        if (iy0 > iy1) continue;
        // columns enumerated per row: every column of the rectangle, or
        // (sharded frame) only this rank's tiles -- tile ty * tiles_x + tx is
        // the rank's when it is == rank (mod shard_count), so on one tile row
        // its tile columns step by shard_count: ceil(span / count) + 1 of them
        // (8 columns each) cover the rectangle, and the raster's work shrinks
        // with the rank count like the rest of the frame's
        const uint32_t shards = (uint32_t)cnt;
        const uint32_t tc0 = (uint32_t)ix0 / TILE_W;
        uint32_t rw = (uint32_t)(ix1 - ix0 + 1);
        if (shards > 1) rw = TILE_W * (((uint32_t)ix1 / TILE_W - tc0 + shards) / shards + 1);
        const uint32_t nrow = (uint32_t)((iy1 - iy0) / nsub + 1), npx = rw * nrow;
        // (row, column) of pixel k stepped incrementally: no division per pixel
        const uint32_t dcol = 32u % rw, drow = 32u / rw;
        uint32_t col = (uint32_t)lane % rw, row = (uint32_t)lane / rw;
        for (uint32_t k = lane; k < npx; k += 32, col += dcol, row += drow) {
            if (col >= rw) { col -= rw; ++row; }
            const uint32_t iy = (uint32_t)iy0 + row * (uint32_t)nsub;
            uint32_t ix = (uint32_t)ix0 + col;
            if (shards > 1) {   // the col / 8-th tile of the rank's on this tile row
                const uint32_t first = (iy / TILE_H * (uint32_t)F.tiles_x + tc0) % shards;
                const uint32_t tx = tc0 + ((uint32_t)fr.shard_rank + shards - first) % shards +
                                    col / TILE_W * shards;
                ix = tx * TILE_W + col % TILE_W;
                if (ix < (uint32_t)ix0 || ix > (uint32_t)ix1) continue;
            }
            const int64_t rr = pixel_ray(F, ix, iy);
            if (rr < 0) continue;
            RayD ray;   // the trace's make_ray, from the per-ray table (slab needs o, 1/d)
            ray.ox = fr.cam_pos[0]; ray.oy = fr.cam_pos[1]; ray.oz = fr.cam_pos[2];
            ray.ix = __ldg(iv.rinv + rr); ray.iy = __ldg(iv.rinv + F.n_rays + rr);
            ray.iz = __ldg(iv.rinv + 2 * F.n_rays + rr);
            ray.nx = ray.ix != 0.0; ray.ny = ray.iy != 0.0; ray.nz = ray.iz != 0.0;
            double pa, pb;
            slab(ray, lo, hi, pa, pb);
            if (pa > pb || !(pb > 0.0)) continue;
            const uint32_t slot = atomicAdd(iv.ccount + rr, 1u);
            if (slot < (uint32_t)CAND_CAP) {
                const int64_t o = (int64_t)slot * F.n_rays + rr;
                iv.cand_pa[o] = pa; iv.cand_pb[o] = pb; iv.cand_pid[o] = (int32_t)pid;
            }
        }
    }
}

// Each ray's candidates in ascending (entry, pid) order, so that
// cand_next_interval can stop at the first entry beyond its best and skip
// the dead prefix.  One warp per ray: a bitonic network over the lanes for
// up to 32 slabs, a rank sort (rank = number of smaller keys) beyond.  Keys
// are distinct (one slab per partition).
__device__ __forceinline__ bool cand_less(double a, int32_t ia, double b, int32_t ib) {
    return a < b || (a == b && ia < ib);
}

// order-preserving bits of a float
__device__ __forceinline__ uint32_t float_key(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

constexpr int SORT_THREADS = 256;

__global__ void __launch_bounds__(SORT_THREADS) cand_sort_kernel(FrameK F, IvBuf iv) {
    // a 32-ray tile staged through shared memory (coalesced global slot rows;
    // rows padded to 33 so a warp reading one ray's column hits 32 banks)
    __shared__ double s_pa[CAND_CAP][33], s_pb[CAND_CAP][33];
    __shared__ int32_t s_pid[CAND_CAP][33];
    __shared__ uint32_t s_n[32], s_nmax;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_tiles = (F.n_rays + 31) / 32;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t r0 = t * 32;
        __syncthreads();
        if (warp == 0) {
            const int64_t rr = r0 + lane;
            uint32_t n = rr < F.n_rays ? iv.ccount[rr] : 0u;
            n = (n >= 2 && n <= (uint32_t)CAND_CAP) ? n : 0u;
            s_n[lane] = n;
            uint32_t m = n;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(FULL, m, off));
            if (lane == 0) s_nmax = m;
        }
        __syncthreads();
        const uint32_t nmax = s_nmax;
        if (nmax == 0) continue;   // CTA-uniform
        for (uint32_t slot = warp; slot < nmax; slot += SORT_THREADS / 32) {
            if ((uint32_t)slot < s_n[lane]) {
                const int64_t o = (int64_t)slot * F.n_rays + r0 + lane;
                s_pa[slot][lane] = iv.cand_pa[o]; s_pb[slot][lane] = iv.cand_pb[o]; s_pid[slot][lane] = iv.cand_pid[o];
            }
        }
        __syncthreads();
        for (int c = warp; c < 32; c += SORT_THREADS / 32) {
            const uint32_t n = s_n[c];
            if (n == 0) continue;   // warp-uniform
            if (n <= 32) {
                // bitonic network on 32-bit keys: the entry rounded down to
                // float (monotone: a later slot never has a smaller entry than
                // an earlier slot's key -- all cand_next_interval's early exit
                // needs), the slot index as payload
                const bool ok = (uint32_t)lane < n;
                uint32_t key = ok ? float_key(__double2float_rd(s_pa[lane][c])) : 0xffffffffu;
                int32_t idx = lane;
                for (int k = 2; k <= 32; k <<= 1) {
                    for (int j = k >> 1; j > 0; j >>= 1) {
                        const uint32_t qk = __shfl_xor_sync(FULL, key, j);
                        const int32_t qi = __shfl_xor_sync(FULL, idx, j);
                        const bool up = (lane & k) == 0, lower = (lane & j) == 0;
                        const bool qless = qk < key || (qk == key && qi < idx);
                        if ((lower == up) ? qless : !qless) { key = qk; idx = qi; }
                    }
                }
                double sa = 0.0, sb = 0.0;
                int32_t sid = 0;
                if (ok) { sa = s_pa[idx][c]; sb = s_pb[idx][c]; sid = s_pid[idx][c]; }
                __syncwarp();
                if (ok) { s_pa[lane][c] = sa; s_pb[lane][c] = sb; s_pid[lane][c] = sid; }
            } else {   // rank sort on the exact keys (entry, pid)
                double pa[2], pb[2];
                int32_t pid[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t i = lane + 32 * h;
                    const bool ok = i < n;
                    pa[h] = ok ? s_pa[i][c] : INFINITY;
                    pb[h] = ok ? s_pb[i][c] : 0.0;
                    pid[h] = ok ? s_pid[i][c] : INT_MAX;
                }
                uint32_t rank[2] = {0u, 0u};
                for (uint32_t j = 0; j < n; ++j) {
                    const double qa = s_pa[j][c];
                    const int32_t qid = s_pid[j][c];
#pragma unroll
                    for (int e = 0; e < 2; ++e) rank[e] += cand_less(qa, qid, pa[e], pid[e]) ? 1u : 0u;
                }
                __syncwarp();
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (lane + 32 * h < n) { s_pa[rank[h]][c] = pa[h]; s_pb[rank[h]][c] = pb[h]; s_pid[rank[h]][c] = pid[h]; }
            }
        }
        __syncthreads();
        for (uint32_t slot = warp; slot < nmax; slot += SORT_THREADS / 32) {
            if ((uint32_t)slot < s_n[lane]) {
                const int64_t o = (int64_t)slot * F.n_rays + r0 + lane;
                iv.cand_pa[o] = s_pa[slot][lane]; iv.cand_pb[o] = s_pb[slot][lane]; iv.cand_pid[o] = s_pid[slot][lane];
                iv.cand_nkey[o] = (uint32_t)slot + 1 < s_n[lane] ? __double2float_rd(s_pa[slot + 1][lane])
                                                                 : INFINITY;
            }
        }
    }
}

// Phase 1 (one thread per ray, 8x4 pixel tiles per warp): the exact
// partition-interval sequence (K:360-391 calling next_interval K:173-230)
// with each interval's clamped entry and the running count of the samples
// march_range would take (K:277-280).  Rays with nothing to march (no hit,
// or only degenerate intervals) are finished here; the others get a cost
// bucket (~4 log2 of their sample count) for longest-first scheduling.
//
// Persistent warps: each warp takes the next 32-ray tile from a counter, so
// the long rays' tiles do not leave a wave tail (the grid is sized to the
// resident warps).
template <bool COUNT>
__global__ void __launch_bounds__(TRACE_BLOCK)
trace_intervals_kernel(SceneK S, EpochK E, FrameK F, IvBuf iv, TrOutputs O) {
    const int lane = threadIdx.x & 31;
    const uint32_t n_tiles = (uint32_t)((F.n_rays + 31) / 32);
    unsigned long long vis_acc = 0, cost_sum = 0;
    uint32_t cost_max = 0;
    while (true) {
    uint32_t tile = 0;
    if (lane == 0) tile = atomicAdd(iv.trace_ctr, 1u);
    tile = __shfl_sync(FULL, tile, 0);
    if (tile >= n_tiles) break;
    const long long tile_t0 = clock64();
    const int64_t rr = (int64_t)tile * 32 + lane;
    uint32_t n = 0, bucket = 0, ray_cost = 0;
    unsigned long long vis_done = 0;
    const bool in_chunk = rr < F.n_rays;
    if (in_chunk) {
        const Pixel px = ray_pixel(F, rr);
        if (px.valid) {
            const RayD ray = make_ray(F.f, px.ix, px.iy);
            const double phase = F.f.jitter ? hash01(px.ix, px.iy) : 0.5;  // K:340
            IvRec *rec = iv.rec + rr * IV_CAP;
            uint32_t cum = 0;
            bool more = false, bsp_redo = false;
            double t_min = 0.0;
            int bsp_cells = 0, bsp_nodes = 0;
            if (F.f.mode == 0) {  // K:346-353: the mesh box is the one interval
                double a, b;
                slab(ray, S.mesh_lo, S.mesh_hi, a, b);
                const double ta = (a > 0.0) ? a : 0.0;
                if (a <= b && b - ta >= F.f.eps) {
                    const int64_t ns = interval_samples(ta, b, F.f.s1, phase);
                    if (ns > (int64_t)CUM_MAX) {
                        more = true;   // the march recomputes it inline
                    } else if (F.B_on) {
                        n = brick_cut(F, ray, ta, b, phase, ns, rec);
                        cum = (uint32_t)ns;
                    } else {
                        IvRec r; r.a = ta; r.pid = -1; r.cum = (uint32_t)ns;
                        rec[0] = r;
                        n = 1;
                        cum = (uint32_t)ns;
                    }
                }
            } else {
                bool use_bsp = S.knodes != nullptr && !(F.f.flags & TR_FLAG_NO_BSP);
                uint32_t n_cand = 0, dead = 0;
                double dead_thr = -INFINITY;
                CandWin win;
                win.base = UINT32_MAX;
                bool cands = false;
                if (F.use_cand) {
                    n_cand = iv.ccount[rr];
                    if (n_cand <= (uint32_t)CAND_CAP) { cands = true; use_bsp = false; }
                }
                BspTrace T;
                if (use_bsp) bsp_begin(S, ray, T);
                for (int attempt = 0; attempt < 2; ++attempt) {
                    int32_t last = -1;
                    n = 0; cum = 0; more = false; t_min = 0.0;
                    while (true) {
                        const double excl = (last < 0) ? 0.0 : F.f.eps;
                        double a, b;
                        const int32_t pid = cands
                            ? cand_next_interval(iv, F.n_rays, rr, n_cand, dead, dead_thr, win, t_min, excl, last, a, b)
                            : use_bsp
                            ? bsp_next_interval<COUNT>(S, E, ray, T, t_min, excl, last, a, b)
                            : next_interval(S, E, ray, t_min, excl, last, a, b);
                        if (pid < 0) break;
                        if (n == IV_CAP) { more = true; break; }
                        int64_t ns = 0;
                        if (b - a >= F.f.eps)   // K:374
                            ns = interval_samples(a, b, (F.f.mode == 2) ? __ldg(E.step + pid) : F.f.s1,
                                                  phase);
                        if ((int64_t)cum + ns > (int64_t)CUM_MAX) { more = true; break; }
                        cum += (uint32_t)ns;
                        IvRec r; r.a = a; r.pid = pid; r.cum = cum;
                        rec[n] = r;
                        ++n;
                        t_min = b - F.f.eps;   // K:390-391
                        last = pid;
                        if (use_bsp) bsp_compact(T, t_min);
                    }
                    if (use_bsp) { bsp_cells += T.cells; bsp_nodes += T.nodes; }
                    if (!(use_bsp && T.overflow)) break;
                    use_bsp = false;  // candidate buffer overflowed: redo with the BVH
                    bsp_redo = true;
                }
            }
            if (more) iv.tail[rr] = t_min;
            if (COUNT) {
                atomicAdd(&g_stats[ST_TRACE_RAYS], 1ull);
                atomicAdd(&g_stats[ST_TRACE_IV], (unsigned long long)n);
                atomicMax(&g_stats[ST_TRACE_MAX_IV], (unsigned long long)n);
                if (bsp_redo) atomicAdd(&g_stats[ST_BSP_OVERFLOW], 1ull);
                atomicAdd(&g_stats[ST_BSP_CELLS], (unsigned long long)bsp_cells);
                atomicAdd(&g_stats[ST_BSP_NODES], (unsigned long long)bsp_nodes);
                atomicMax(&g_stats[ST_TRACE_MAX_NODES], (unsigned long long)bsp_nodes);
                atomicMax(&g_stats[ST_MAX_RAY_SAMPLES], (unsigned long long)cum);
            }
            if (F.B_on) {
                TrRayState z = {};
                z.flags = (cum > 0) ? 1u : 0u;
                if (more) { z.flags = 0u; atomicOr(F.B_ctr + 2, 1u); }
                F.B_state[rr] = z;
            }
            if (F.B_on && !(cum > 0 || more) && !F.B_write_bg) {
                // another rank writes this background pixel
            } else if (cum > 0 || more) {
                bucket = cost_bucket((double)cum + (more ? 1024.0 : 0.0));
            } else {  // nothing to march: background, `visited` = every interval returned
                if (F.defer_bg) {   // listed for background_kernel
                    O.visited[px.out] = (int32_t)n;
                    const unsigned m = __activemask();
                    const int lead = __ffs(m) - 1;
                    unsigned e0 = 0;
                    if (lane == lead) e0 = atomicAdd(iv.n_bg, (unsigned)__popc(m));
                    e0 = __shfl_sync(m, e0, lead) + __popc(m & ((1u << lane) - 1u));
                    iv.order[F.n_rays - 1 - (int64_t)e0] = (uint32_t)rr;
                } else {
                    const Acc zero = {0.0, 0.0, 0.0, 0.0};
                    write_pixel(F.f, O, px.out, zero, 0, (int32_t)n);
                }
                vis_done = n;
            }
            iv.cnt[rr] = n | (bucket << 16) | (more ? CNT_MORE : 0u);
            ray_cost = cum + (more ? 1024u : 0u);
        } else {
            iv.cnt[rr] = 0;
        }
    }
    const unsigned vm = __ballot_sync(FULL, in_chunk);
    if (in_chunk) {
        const unsigned peers = __match_any_sync(vm, bucket);
        if (lane == __ffs(peers) - 1) atomicAdd(iv.hist + bucket, (unsigned)__popc(peers));
    }
    if ((F.f.flags & TR_FLAG_TILE_TIMING) && lane == 0) {
        const unsigned long long dt = (unsigned long long)(clock64() - tile_t0);
        atomicAdd(&g_stats[ST_TILE_CYCLES], dt);
        atomicMax(&g_stats[ST_TILE_MAX_CYCLES], dt);
    }
    vis_acc += vis_done;
    cost_sum += ray_cost;
    cost_max = ray_cost > cost_max ? ray_cost : cost_max;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        vis_acc += __shfl_xor_sync(FULL, vis_acc, off);
        cost_sum += __shfl_xor_sync(FULL, cost_sum, off);
        cost_max = max(cost_max, __shfl_xor_sync(FULL, cost_max, off));
    }
    if (lane == 0 && vis_acc) atomicAdd(iv.totals + 1, vis_acc);
    if (lane == 0 && cost_sum) {
        atomicAdd(iv.ray_stats, cost_sum);
        atomicMax(iv.ray_stats + 1, (unsigned long long)cost_max);
    }
}

// The background pixels the trace listed (F.defer_bg: the framebuffer is
// page-locked host memory), written by BG_CTAS small CTAs on a side stream
// while the march runs.  They fit beside three march CTAs per SM (registers)
// and their dependent-load chain paces them (~BG_CTAS x 64 pixels per ~1 us):
// the PCIe stores trickle out beside the march instead of bursting at the
// start of the trace, where they back up the memory system (measured: +105
// us on the trace for 4.8 MB of background at 512^2).
constexpr int BG_THREADS = 64;
constexpr int BG_CTAS = 8;

__global__ void __launch_bounds__(BG_THREADS)
background_kernel(FrameK F, IvBuf iv, TrOutputs O) {
    const uint32_t n = *iv.n_bg;
    const Acc zero = {0.0, 0.0, 0.0, 0.0};
    for (uint32_t e = blockIdx.x * BG_THREADS + threadIdx.x; e < n; e += gridDim.x * BG_THREADS) {
        const uint32_t rr = iv.order[F.n_rays - 1 - (int64_t)e];
        const Pixel px = ray_pixel(F, rr);
        write_pixel(F.f, O, px.out, zero, 0, O.visited[px.out]);
    }
}

// Marching rays of the chunk in descending cost buckets (order inside a
// bucket is arbitrary; outputs do not depend on it).
__global__ void __launch_bounds__(TRACE_BLOCK)
order_rays_kernel(FrameK F, IvBuf iv) {
    __shared__ uint32_t start[N_BUCKETS];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // lanes per ray: 4, unless the longest ray's rounds at 4 lanes
        // (max / 4) exceed the average lane's share of the work (sum /
        // resident lanes) -- then 16, so long rays stop setting the frame
        // time (1e9-tet scenes: up to 3,600 samples on one ray).  8 lanes
        // measured slower than 4 on radial59/128/272 in every mode except
        // radial272 skip-adaptive (-2%; scripts/lane_sweep.py, profiles/r02)
        const unsigned long long sum = iv.ray_stats[0], mx = iv.ray_stats[1];
        *iv.gsel = (mx * (unsigned long long)F.march_lanes <= 4ull * sum) ? 4u : 16u;
    }
    if (threadIdx.x < N_BUCKETS) {
        uint32_t s = 0;
        for (int b = N_BUCKETS - 1; b > (int)threadIdx.x; --b) s += iv.hist[b];
        start[threadIdx.x] = s;
    }
    __syncthreads();
    const int64_t rr = blockIdx.x * (int64_t)TRACE_BLOCK + threadIdx.x;
    const uint32_t bucket = rr < F.n_rays ? (iv.cnt[rr] >> 16) & 0xffu : 0u;
    const bool valid = bucket != 0;
    const unsigned vm = __ballot_sync(FULL, valid);
    if (!valid) return;
    const unsigned peers = __match_any_sync(vm, bucket);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(iv.cursor + bucket, (unsigned)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    iv.order[start[bucket] + base + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)rr;
}

__device__ __forceinline__ IvRec load_rec(const IvRec *p) {
    const int4 v = __ldg(reinterpret_cast<const int4 *>(p));
    IvRec r;
    r.a = __hiloint2double(v.y, v.x);
    r.pid = v.z;
    r.cum = (uint32_t)v.w;
    return r;
}

// Inline continuation past the stored list (IV_CAP intervals or CUM_MAX
// samples): the next interval with samples, from (t_min, last) (K:360-391).
// Returns false when the ray has no further interval.  Run by one lane.
struct Inline {
    double t_min, a;
    int64_t n, k;      // samples of the current inline interval, samples taken
    int32_t last, pid;
    int32_t visited;   // inline intervals returned so far
    int32_t started;   // mode 0: the mesh-box interval was issued
};

__device__ bool inline_next(const SceneK &S, const EpochK &E, const TrFrame &fr, int64_t ix,
                            int64_t iy, double phase, Inline &L) {
    const RayD ray = make_ray(fr, ix, iy);
    if (fr.mode == 0) {
        if (L.started) return false;
        L.started = 1;
        double a, b;
        slab(ray, S.mesh_lo, S.mesh_hi, a, b);
        const double ta = (a > 0.0) ? a : 0.0;
        if (!(a <= b && b - ta >= fr.eps)) return false;
        L.a = ta; L.pid = -1; L.k = 0;
        L.n = interval_samples(ta, b, fr.s1, phase);
        return true;
    }
    while (true) {
        double a, b;
        const int32_t pid = next_interval(S, E, ray, L.t_min, (L.last < 0) ? 0.0 : fr.eps, L.last, a, b);
        if (pid < 0) return false;
        L.visited += 1;
        L.t_min = b - fr.eps;
        L.last = pid;
        if (b - a >= fr.eps) {
            L.a = a; L.pid = pid; L.k = 0;
            L.n = interval_samples(a, b, (fr.mode == 2) ? __ldg(E.step + pid) : fr.s1, phase);
            return true;
        }
    }
}

// One sample of march_range (K:277-290): position t = a + (k + phase) * step
// (K:278), point location (K:93-136: the grid's candidate leaf proved by its
// exclusive box, else the full descent -- both exact), field
// (K:149-153), TF (K:74-90) and opacity correction (K:27).  Returns
// (ca, r, g, b); found = inside a tet (ca = c = 0 otherwise).
#ifndef TR_RASTER_PX
#define TR_RASTER_PX 262144   // A/B knob: band pixels per candidate-raster warp of a partition
#endif

#if TR_ROUND_TIMES   // diagnostics build: per-thread cycle sums of the march's phases
constexpr int DBG_THREADS = 148 * 8 * 256, DBG_PH = 8;
__device__ unsigned long long g_dbg[DBG_THREADS * DBG_PH];
__device__ __forceinline__ void dbg_add(int ph, long long dt) {
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < DBG_THREADS) g_dbg[t * DBG_PH + ph] += (unsigned long long)dt;
}
#define DBG_T(v) const long long v = clock64()
#else
#define DBG_T(v)
#endif

// The transfer function staged in shared memory once per march CTA: a
// sample's TF lookup (K:74-90) then costs a shared-memory load instead of an
// L1/L2 round trip on its dependent chain.  Only in the 128-thread march of
// reference / skip modes (2-4% faster there; with it the 256-thread
// skip-adaptive march measured 2% slower, so its instantiation has no TF code).
struct MarchTabs {
    const double *tf;   // TF table copy, or NULL (global)
};
constexpr int TABS_TF_MAX = 16384;   // TF tables up to 512 entries are staged
#ifndef TR_TABS_TF   // A/B knob
#define TR_TABS_TF 1
#endif

// dynamic shared memory of a march launch with `block` threads per CTA
__host__ __device__ inline int march_tabs_bytes(int block, int64_t n_tf) {
    return (TR_TABS_TF && block == 128 && n_tf * 32 <= TABS_TF_MAX) ? (int)(n_tf * 32) : 0;
}

template <bool TABS = false>
__device__ __forceinline__ double4 shade_sample(const SceneK &S, const EpochK &E, const TrFrame &fr,
                                                double ox, double oy, double oz, double dx,
                                                double dy, double dz, double a, int64_t k,
                                                double phase, int32_t pid, bool stats,
                                                bool pair_scan, bool use_grid, bool use_cells,
                                                bool &found, const MarchTabs *T = nullptr) {
    double4 sh = make_double4(0.0, 0.0, 0.0, 0.0);
    found = false;
    double step = fr.s1, e = 1.0;
    if (fr.mode == 2) {
        const double2 se = __ldg(reinterpret_cast<const double2 *>(E.step_ratio) + pid);
        step = se.x;
        e = se.y;
    }
    DBG_T(d0);
    const double t = a + ((double)k + phase) * step;
    const PQuery q = make_query(ox + t * dx, oy + t * dy, oz + t * dz);
    if (stats) atomicAdd(&g_stats[ST_SLOTS], 1ull);
    double l[4];
    uint32_t pos = UINT32_MAX;
    bool located = false;
    if (use_grid && S.grid_n > 0 && !(fr.flags & (TR_FLAG_NO_ANALYTIC | TR_FLAG_NO_WALK))) {
        // analytic cube grid (tr_grid_scene_build): the cube, its exclusive box
        // and records follow from the coordinates -- no leaf header load
        const int64_t n = S.grid_n;
        if (q.x >= 0.0 && q.y >= 0.0 && q.z >= 0.0 && q.x < (double)n && q.y < (double)n &&
            q.z < (double)n) {
            const int cx = (int)q.x, cy = (int)q.y, cz = (int)q.z;
            if (q.x > tr_grid::ex_lo(cx, n, S.grid_pad) && q.x < tr_grid::ex_hi(cx, n, S.grid_pad) &&
                q.y > tr_grid::ex_lo(cy, n, S.grid_pad) && q.y < tr_grid::ex_hi(cy, n, S.grid_pad) &&
                q.z > tr_grid::ex_lo(cz, n, S.grid_pad) && q.z < tr_grid::ex_hi(cz, n, S.grid_pad)) {
                const int par = (cx + cy + cz) & 1;
                const float *c = par ? S.pred_class[1] : S.pred_class[0];
                const uint32_t start = 5u * tr_grid::cube_slot32((uint32_t)n, S.grid_brick != 0,
                                                                 (uint32_t)cx, (uint32_t)cy,
                                                                 (uint32_t)cz);
                // the predictor's rows are relative to an interior cube's box corner
                const float lo[3] = {(float)cx + (float)S.grid_pad, (float)cy + (float)S.grid_pad,
                                     (float)cz + (float)S.grid_pad};
                pos = walk_leaf(S, S.class_walk + 8 * par, start, 5u, q, l,
                                !(fr.flags & TR_FLAG_NO_PRED),
                                make_float4(c[0], c[1], c[2], c[3]),
                                make_float4(c[4], c[5], c[6], c[7]),
                                make_float4(c[8], c[9], c[10], c[11]), lo);
                located = true;
                if (stats) atomicAdd(&g_stats[ST_GRID_HIT], 1ull);
            }
        }
    }
    if (!located && use_grid && !(use_cells && S.cells_first)) {
        int par = 0;
        const int64_t gc = grid_cell(S, q, &par);
        if (gc >= 0) {
            LeafHint hh;
            load_leaf(S.pgrid_leaf + gc, hh);
            float4 pr0 = float4(), pr1 = float4(), pr2 = float4();  // walk-start predictor
            bool use_pred = false;
            if (S.pgrid_pred) {
                const float4 *src = S.pgrid_pred + 3 * gc;
                pr0 = __ldg(src); pr1 = __ldg(src + 1); pr2 = __ldg(src + 2);
                use_pred = true;
            } else if (S.pred_classes == 2) {
                const float *c = par ? S.pred_class[1] : S.pred_class[0];
                pr0 = make_float4(c[0], c[1], c[2], c[3]);
                pr1 = make_float4(c[4], c[5], c[6], c[7]);
                pr2 = make_float4(c[8], c[9], c[10], c[11]);
                use_pred = true;
            }
            if (fr.flags & TR_FLAG_NO_PRED) use_pred = false;
            if (strictly_in(q, hh.lo, hh.hi)) {
                if (pair_scan) pos = scan_leaf_pairs(S, hh.start, hh.count, q, l);
                else if (fr.flags & TR_FLAG_NO_WALK) pos = scan_leaf_first(S, hh.start, hh.count, q, l);
                else pos = walk_leaf(S, S.pgrid_leaf[gc].walk, hh.start, hh.count, q, l, use_pred,
                                     pr0, pr1, pr2, hh.lo);
                located = true;
                if (stats) atomicAdd(&g_stats[ST_GRID_HIT], 1ull);
            }
        }
    }
    if (!located && use_cells) located = locate_cells(S, q, l, pos);
    if (!located) {
        int32_t leaf;
        if (stats) atomicAdd(&g_stats[ST_DESCENT], 1ull);
        pos = locate_full(S, q, l, leaf);
    }
    if (pos == UINT32_MAX) return sh;
    DBG_T(d1);
    double v;
    const double2 *rp = reinterpret_cast<const double2 *>(S.tets + pos);
    if (S.centering == 0) {   // K:149-151
        const double4 f = ldg256(rp + 6);
        v = l[0] * f.x + l[1] * f.y + l[2] * f.z + l[3] * f.w;
    } else {                  // K:153
        v = __ldg(rp + 6).x;
    }
    double c[4];
#if TR_ROUND_TIMES
    asm volatile("" :: "d"(v));
#endif
    DBG_T(d2);
    if (TABS && T->tf) tf_sample<true>(T->tf, E.n_tf, E.tf_lo, E.tf_hi, v, c);
    else tf_sample(E.tf, E.n_tf, E.tf_lo, E.tf_hi, v, c);
    const double x = 1.0 - c[3];
#if TR_ROUND_TIMES
    asm volatile("" :: "d"(x));
#endif
    DBG_T(d3);
    // K:27; glibc's pow(x, 1) and pow(1, y) are exactly x and 1
    const bool need_pow = e != 1.0 && x != 1.0;
    sh.x = 1.0 - (need_pow ? ref_pow(x, e) : x);
#if TR_ROUND_TIMES
    asm volatile("" :: "d"(sh.x));
    DBG_T(d4);
    dbg_add(0, d1 - d0); dbg_add(1, d2 - d1); dbg_add(2, d3 - d2); dbg_add(3, d4 - d3);
    dbg_add(7, 1);
#endif
    if (stats) {
        atomicAdd(&g_stats[ST_FOUND], 1ull);
        if (need_pow) atomicAdd(&g_stats[ST_POW], 1ull);
    }
    sh.y = c[0]; sh.z = c[1]; sh.w = c[2];
    found = true;
    return sh;
}

// Phase 2: G lanes march one ray together.  Per round lane j of the group
// takes the ray's next-but-j sample: its interval is found from the stored
// prefix counts, its position is t = a + (k + phase) * step (K:278), and it
// is located, interpolated, classified and opacity-corrected independently;
// the group then composites the round's samples in order with the exact
// early-termination rule (K:285-295).  Groups without a ray take part in
// the warp collectives with no sample.
template <int G, int MINB, bool STATS>
__global__ void __launch_bounds__(MARCH_BLOCK, MINB)
march_kernel(SceneK S, EpochK E, FrameK F, IvBuf iv, TrOutputs O) {
    static_assert(G >= 2 && G <= 32 && (32 % G) == 0, "group size");
    __shared__ unsigned long long red[2][MARCH_BLOCK / 32];
    // per-lane sample result (ca, r, g, b) as [lane in group][group]: the G
    // reads of a composite step hit consecutive entries across the warp's
    // groups (no bank conflicts; [group][lane] was an 8-way conflict)
    __shared__ double4 shade[G][MARCH_BLOCK / G];
    __shared__ Inline inl[MARCH_BLOCK / G];             // per-group inline state (rare path)
    const TrFrame &fr = F.f;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane % G;                   // lane in group
    const int gbase = lane - j;               // first lane of my group
    Inline &L = inl[threadIdx.x / G];
    const bool track = fr.track_ppart && fr.mode != 0;
    const bool use_grid = !(fr.flags & TR_FLAG_NO_GRID);
    const bool use_cells = S.cell_off != nullptr && !(fr.flags & TR_FLAG_NO_CELLS);
    // TR_FLAG_STATS event counters.  Kept a runtime test even in the STATS =
    // false instance: measured 25% faster than a compile-time false (the
    // atomics' guards change how the hot loop is scheduled; build/ab A/B).
    const bool stats = STATS || (fr.flags & TR_FLAG_STATS) != 0;
    const bool pair_scan = (fr.flags & TR_FLAG_PAIR_SCAN) != 0;
    const unsigned gmask = (G == 32) ? FULL : (((1u << G) - 1u) << gbase);
    uint32_t n_queue = 0;
    for (int b = 1; b < N_BUCKETS; ++b) n_queue += iv.hist[b];
    unsigned long long my_samples = 0, my_visited = 0;

    // group-uniform ray state
    bool active = false, exhausted = false, inline_mode = false;
    int64_t rr = 0, out = 0;
    int32_t pix = 0, piy = 0;
    double ox = 0, oy = 0, oz = 0, dx = 0, dy = 0, dz = 0, phase = 0.5;
    Acc acc = {0.0, 0.0, 0.0, 0.0};
    int64_t samples = 0;
    uint32_t taken = 0, c_tot = 0, c_before = 0;
    int32_t i_cur = 0, n_iv = 0;
    bool more = false;
    const IvRec *rec = nullptr;

    while (true) {
        // ---- refill: one queue slot per group that needs a ray
        const bool want = !active && !exhausted;
        const unsigned lm = __ballot_sync(FULL, want && j == 0);
        if (lm) {
            const int leader = __ffs(lm) - 1;
            unsigned base = 0;
            if (lane == leader) base = atomicAdd(O.work, (unsigned)__popc(lm));
            base = __shfl_sync(FULL, base, leader);
            const unsigned qpos = base + __popc(lm & ((1u << gbase) - 1u));
            if (want) {
                if (qpos >= n_queue) {
                    exhausted = true;
                } else {
                    rr = (int64_t)iv.order[qpos];
                    const Pixel px = ray_pixel(F, rr);
                    out = px.out;
                    pix = (int32_t)px.ix;
                    piy = (int32_t)px.iy;
                    const RayD ray = make_ray(fr, px.ix, px.iy);
                    ox = ray.ox; oy = ray.oy; oz = ray.oz;
                    dx = ray.dx; dy = ray.dy; dz = ray.dz;
                    phase = fr.jitter ? hash01(px.ix, px.iy) : 0.5;
                    acc.r = acc.g = acc.b = acc.a = 0.0;
                    samples = 0;
                    taken = 0;
                    i_cur = 0;
                    c_before = 0;
                    const uint32_t c = iv.cnt[rr];
                    n_iv = (int32_t)(c & 0xffffu);
                    more = (c & CNT_MORE) != 0;
                    rec = iv.rec + rr * IV_CAP;
                    c_tot = n_iv > 0 ? load_rec(rec + (n_iv - 1)).cum : 0u;
                    inline_mode = false;
                    if (c_tot == 0) {  // only inline intervals (the trace ran out of room)
                        inline_mode = true;
                        if (j == 0) {
                            L.t_min = iv.tail[rr];
                            L.last = n_iv > 0 ? load_rec(rec + (n_iv - 1)).pid : -1;
                            L.visited = 0;
                            L.started = 0;
                            L.n = 0; L.k = 0;
                        }
                    }
                    active = true;
                }
            }
        }
        if (__all_sync(FULL, exhausted)) break;

        // ---- inline mode: lane 0 fetches the next interval with samples when needed
        bool idle = false;
        if (active && inline_mode && j == 0 && L.k >= L.n)
            idle = !inline_next(S, E, fr, pix, piy, phase, L);
        __syncwarp();
        idle = __shfl_sync(FULL, idle, gbase);

        // ---- my sample
        bool has = false;
        double a = 0.0;
        int32_t pid = -1, i_mine = 0;
        uint32_t c0_mine = 0;
        int64_t k = 0, remaining = 0;
        if (active && !idle) {
            if (!inline_mode) {
                const uint32_t s = taken + (uint32_t)j;
                remaining = (int64_t)(c_tot - taken);
                if (s < c_tot) {
                    int32_t i = i_cur;
                    uint32_t c0 = c_before;
                    IvRec r = load_rec(rec + i);
                    while (r.cum <= s) { c0 = r.cum; ++i; r = load_rec(rec + i); }
                    a = r.a;
                    pid = r.pid;
                    k = (int64_t)(s - c0);
                    i_mine = i;
                    c0_mine = c0;
                    has = true;
                }
            } else {
                remaining = L.n - L.k;
                if ((int64_t)j < remaining) {
                    a = L.a;
                    pid = L.pid;
                    k = L.k + j;
                    has = true;
                }
            }
        }

        // ---- shade my sample (K:277-290)
        double4 sh = make_double4(0.0, 0.0, 0.0, 0.0);
        bool found = false;
        if (has)
            sh = shade_sample(S, E, fr, ox, oy, oz, dx, dy, dz, a, k, phase, pid, stats, pair_scan,
                              use_grid, use_cells, found);
        shade[j][threadIdx.x / G] = sh;
        const unsigned fbits = __ballot_sync(FULL, found) >> gbase;
        __syncwarp();

        // ---- composite the round in sample order (K:285-295).  A sample
        // outside every tet has ca = c = 0, which leaves acc bit-unchanged;
        // termination is only tested after a found sample.
        const int cnt = (int)((remaining < G) ? remaining : G);
        int taken_r = cnt;
        bool term = false;
        if (active && !idle) {
            for (int m = 0; m < cnt; ++m) {
                const double4 g = shade[m][threadIdx.x / G];
                const double w = (1.0 - acc.a) * g.x;
                acc.r += w * g.y;
                acc.g += w * g.z;
                acc.b += w * g.w;
                acc.a += w;
                if (((fbits >> m) & 1u) && acc.a >= fr.term) { taken_r = m + 1; term = true; break; }
            }
            if (stats && j == 0) {
                atomicAdd(&g_stats[ST_ROUNDS], 1ull);
                if (cnt < G) atomicAdd(&g_stats[ST_PARTIAL], 1ull);
            }
        }
        __syncwarp();

        // ---- advance the group's cursor (all shuffles before any divergence)
        const int src = gbase + ((taken_r > 0) ? taken_r - 1 : 0);
        const int32_t i_last = __shfl_sync(FULL, i_mine, src);
        const uint32_t c0_last = __shfl_sync(FULL, c0_mine, src);
        bool done = false, flush = false;
        int32_t flush_n = 0;
        if (active) {
            if (idle) {  // inline intervals exhausted
                done = true;
            } else if (!inline_mode) {
                samples += taken_r;
                taken += (uint32_t)taken_r;
                i_cur = i_last;
                c_before = c0_last;
                if (term) {                       // K:388-389: the last interval visited
                    flush = true; flush_n = i_last + 1;
                    done = true;
                } else if (taken == c_tot) {      // stored list consumed
                    flush = true; flush_n = n_iv;
                    if (more) {
                        inline_mode = true;
                        if (j == 0) {
                            L.t_min = iv.tail[rr];
                            L.last = n_iv > 0 ? rec[n_iv - 1].pid : -1;
                            L.visited = 0;
                            L.started = 1;       // mode 0 has one interval, stored
                            L.n = 0; L.k = 0;
                        }
                    } else {
                        done = true;
                    }
                }
            } else {
                samples += taken_r;
                if (j == 0) {
                    L.k += taken_r;
                    if (track && L.pid >= 0)
                        atomicAdd((unsigned long long *)O.ppart + L.pid, (unsigned long long)taken_r);
                }
                if (term) done = true;
            }
        }
        // per-partition samples of the stored intervals (K:386-387): the
        // group's lanes add the intervals' counts, the last one clipped
        if (flush && track) {
            for (int32_t i = j; i < flush_n; i += G) {
                const IvRec r = load_rec(rec + i);
                const uint32_t lo = (i > 0) ? load_rec(rec + (i - 1)).cum : 0u;
                const uint32_t hi = (r.cum < taken) ? r.cum : taken;
                if (hi > lo) atomicAdd((unsigned long long *)O.ppart + r.pid, (unsigned long long)(hi - lo));
            }
        }
        if (done) {
            if (j == 0) {
                int32_t visited = 0;
                if (fr.mode != 0) {
                    if (!inline_mode) visited = term ? i_last + 1 : n_iv;
                    else visited = n_iv + L.visited;
                }
                write_pixel(fr, O, out, acc, samples, visited);
                my_samples += (unsigned long long)samples;
                my_visited += (unsigned long long)visited;
            }
            active = false;
        }
        __syncwarp();
    }
    // block reduction of the frame totals (R:198-201)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        my_samples += __shfl_xor_sync(FULL, my_samples, off);
        my_visited += __shfl_xor_sync(FULL, my_visited, off);
    }
    if (lane == 0) { red[0][warp] = my_samples; red[1][warp] = my_visited; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0, v = 0;
        for (int w = 0; w < MARCH_BLOCK / 32; ++w) { s += red[0][w]; v += red[1][w]; }
        if (s) atomicAdd((unsigned long long *)O.totals, s);
        if (v) atomicAdd((unsigned long long *)O.totals + 1, v);
    }
    (void)gmask;
}

// Variant of march_kernel with the group-uniform ray state in shared memory
// (SoA, one slot per group) instead of registers: the registers then hold a
// sample's working set only, so more warps fit per SM.  Same
// rounds, same exact compositing; lane 0 of a group writes the state.
template <int G, int MINB, bool BRICK = false, bool STATS = false, int BLK = MARCH_BLOCK>
__global__ void __launch_bounds__(BLK, MINB)
march_sm_kernel(SceneK S, EpochK E, FrameK F, IvBuf iv, TrOutputs O) {
    static_assert(G >= 2 && G <= 32 && (32 % G) == 0, "group size");
    if (F.auto_g && *(volatile const uint32_t *)iv.gsel != (uint32_t)G) return;   // not the chosen width
    constexpr int NG = BLK / G;
    __shared__ unsigned long long red[2][BLK / 32];
    __shared__ double4 shade[G][BLK / G];   // [lane in group][group]: conflict free
    __shared__ Inline inl[NG];
    __shared__ double s_d[3][NG], s_acc[4][NG], s_phase[NG];   // origin: the camera (make_ray)
    __shared__ long long s_out[NG], s_samples[NG];
    __shared__ uint32_t s_rr[NG], s_taken[NG], s_ctot[NG], s_cbefore[NG];
    __shared__ int32_t s_icur[NG], s_niv[NG], s_pix[NG], s_piy[NG];
    __shared__ double s_ra[NG];                         // the cursor interval's record
    __shared__ int32_t s_rpid[NG];                      // (rec[s_icur]: entry, partition,
    __shared__ uint32_t s_rcum[NG];                     //  running sample count)
    __shared__ uint32_t s_cfull[BRICK ? NG : 1], s_tbegin[BRICK ? NG : 1];   // brick runs
#if TR_RAY_TIMES   // diagnostics build: each ray's (start, end) globaltimer in rgba.r / .g
    __shared__ unsigned long long s_tstart[NG];
#endif
    const TrFrame &fr = F.f;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane % G;
    const int gbase = lane - j;
    const int g = threadIdx.x / G;
    Inline &L = inl[g];
    const bool track = fr.track_ppart && fr.mode != 0;
    const bool use_grid = !(fr.flags & TR_FLAG_NO_GRID);
    const bool use_cells = S.cell_off != nullptr && !(fr.flags & TR_FLAG_NO_CELLS);
    constexpr bool stats = STATS;   // TR_FLAG_STATS selects the counting instantiation
    const bool pair_scan = (fr.flags & TR_FLAG_PAIR_SCAN) != 0;
    const bool timing = (fr.flags & TR_FLAG_TILE_TIMING) != 0;
    if (timing && threadIdx.x == 0) atomicMin(&g_stats[ST_MARCH_T0], globaltimer_ns());
    // the TF table into shared memory (MarchTabs)
    extern __shared__ __align__(16) unsigned char s_tabs[];
    MarchTabs tabs;
    tabs.tf = nullptr;
    if (march_tabs_bytes(BLK, E.n_tf)) {   // compile-time false unless BLK == 128
        double *tf = reinterpret_cast<double *>(s_tabs);
        for (int k2 = threadIdx.x; k2 < 4 * E.n_tf; k2 += BLK) tf[k2] = E.tf[k2];
        tabs.tf = tf;
        __syncthreads();
    }
    uint32_t n_queue = 0;
    if (BRICK) n_queue = *(volatile const uint32_t *)F.B_ctr;
    else
        for (int b = 1; b < N_BUCKETS; ++b) n_queue += iv.hist[b];
    unsigned long long my_samples = 0, my_visited = 0;
    bool active = false, exhausted = false, inline_mode = false, more = false;

    while (true) {
        DBG_T(r0);
        // ---- refill: one queue slot per group that needs a ray
        const bool want = !active && !exhausted;
        const unsigned lm = __ballot_sync(FULL, want && j == 0);
        if (lm) {
            const int leader = __ffs(lm) - 1;
            unsigned base = 0;
            if (lane == leader) base = atomicAdd(O.work, (unsigned)__popc(lm));
            base = __shfl_sync(FULL, base, leader);
            const unsigned qpos = base + __popc(lm & ((1u << gbase) - 1u));
            if (want) {
                if (qpos >= n_queue) {
                    exhausted = true;
                    if (timing && j == 0) atomicMin(&g_stats[ST_MARCH_TQ], globaltimer_ns());
                } else {
                    const uint32_t rr = BRICK ? F.B_queue[qpos] : iv.order[qpos];
                    const uint32_t c = iv.cnt[rr];
                    const int32_t n_iv = (int32_t)(c & 0xffffu);
                    more = (c & CNT_MORE) != 0;
                    const IvRec *rec = iv.rec + (int64_t)rr * IV_CAP;
                    const uint32_t c_tot = n_iv > 0 ? load_rec(rec + (n_iv - 1)).cum : 0u;
                    inline_mode = c_tot == 0;   // only inline intervals (the trace ran out of room)
                    if (j == 0) {
                        const Pixel px = ray_pixel(F, rr);
                        const RayD ray = make_ray(fr, px.ix, px.iy);
                        s_rr[g] = rr; s_out[g] = px.out;
#if TR_RAY_TIMES
                        s_tstart[g] = globaltimer_ns();
#endif
                        s_pix[g] = (int32_t)px.ix; s_piy[g] = (int32_t)px.iy;
                        s_d[0][g] = ray.dx; s_d[1][g] = ray.dy; s_d[2][g] = ray.dz;
                        s_phase[g] = fr.jitter ? hash01(px.ix, px.iy) : 0.5;
                        s_acc[0][g] = s_acc[1][g] = s_acc[2][g] = s_acc[3][g] = 0.0;
                        s_samples[g] = 0;
                        s_taken[g] = 0; s_icur[g] = 0; s_cbefore[g] = 0;
                        s_niv[g] = n_iv; s_ctot[g] = c_tot;
                        if (BRICK) {   // resume the ray where its previous run stopped
                            const TrRayState st = F.B_state[rr];
                            s_acc[0][g] = st.acc[0]; s_acc[1][g] = st.acc[1];
                            s_acc[2][g] = st.acc[2]; s_acc[3][g] = st.acc[3];
                            s_samples[g] = st.samples;
                            s_taken[g] = st.taken; s_icur[g] = st.icur; s_cbefore[g] = st.cbefore;
                            s_ctot[g] = st.stop;        // this brick's run ends here
                            s_cfull[g] = c_tot;
                            s_tbegin[g] = st.taken;
                        }
                        if (inline_mode) {
                            L.t_min = iv.tail[rr];
                            L.last = n_iv > 0 ? load_rec(rec + (n_iv - 1)).pid : -1;
                            L.visited = 0; L.started = 0; L.n = 0; L.k = 0;
                        } else {
                            const IvRec r0 = load_rec(rec + s_icur[g]);
                            s_ra[g] = r0.a; s_rpid[g] = r0.pid; s_rcum[g] = r0.cum;
                        }
                    }
                    active = true;
                }
            }
        }
        if (__all_sync(FULL, exhausted)) break;
        __syncwarp();

        // ---- inline mode: lane 0 fetches the next interval with samples when needed
        bool idle = false;
        if (__any_sync(FULL, active && inline_mode)) {   // rare: skip the sync otherwise
            if (active && inline_mode && j == 0 && L.k >= L.n)
                idle = !inline_next(S, E, fr, s_pix[g], s_piy[g], s_phase[g], L);
            __syncwarp();
            idle = __shfl_sync(FULL, idle, gbase);
        }

        // ---- my sample
        bool has = false;
        double a = 0.0;
        int32_t pid = -1, i_mine = 0;
        uint32_t c0_mine = 0;
        IvRec r_mine = {0.0, 0, 0u};
        int64_t k = 0, remaining = 0;
        if (active && !idle) {
            if (!inline_mode) {
                const uint32_t taken = s_taken[g], c_tot = s_ctot[g];
                const uint32_t s = taken + (uint32_t)j;
                remaining = (int64_t)(c_tot - taken);
                if (s < c_tot) {
                    const IvRec *rec = iv.rec + (int64_t)s_rr[g] * IV_CAP;
                    int32_t i = s_icur[g];
                    uint32_t c0 = s_cbefore[g];
                    IvRec r;   // the cursor's record from shared memory, later ones from L2
                    r.a = s_ra[g]; r.pid = s_rpid[g]; r.cum = s_rcum[g];
                    while (r.cum <= s) { c0 = r.cum; ++i; r = load_rec(rec + i); }
                    r_mine = r;
                    a = r.a;
                    pid = r.pid;
                    // mode 0: one interval, or (bricks) its cuts, all from the entry
                    k = (int64_t)(BRICK && fr.mode == 0 ? s : s - c0);
                    i_mine = i;
                    c0_mine = c0;
                    has = true;
                }
            } else {
                remaining = L.n - L.k;
                if ((int64_t)j < remaining) {
                    a = L.a;
                    pid = L.pid;
                    k = L.k + j;
                    has = true;
                }
            }
        }

        // ---- shade my sample (K:277-290)
        DBG_T(r1);
        double4 sh = make_double4(0.0, 0.0, 0.0, 0.0);
        bool found = false;
        if (has)
            sh = shade_sample<BLK == 128 && TR_TABS_TF>(
                S, E, fr, fr.cam_pos[0], fr.cam_pos[1], fr.cam_pos[2], s_d[0][g], s_d[1][g],
                s_d[2][g], a, k, s_phase[g], pid, stats, pair_scan, use_grid, use_cells, found,
                &tabs);
        shade[j][threadIdx.x / G] = sh;
        const unsigned fbits = __ballot_sync(FULL, found) >> gbase;
        __syncwarp();
        DBG_T(r2);

        // ---- composite the round in sample order (K:285-295)
        const int cnt = (int)((remaining < G) ? remaining : G);
        int taken_r = cnt;
        bool term = false;
        Acc acc = {0.0, 0.0, 0.0, 0.0};
        if (active && !idle) {
            acc.r = s_acc[0][g]; acc.g = s_acc[1][g]; acc.b = s_acc[2][g]; acc.a = s_acc[3][g];
#if TR_UNROLL_COMPOSITE
            // unrolled and predicated: no loop counter or exit branch per sample
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m < cnt && !term) {
                    const double4 gg = shade[m][g];
                    const double w = (1.0 - acc.a) * gg.x;
                    acc.r += w * gg.y;
                    acc.g += w * gg.z;
                    acc.b += w * gg.w;
                    acc.a += w;
                    if (((fbits >> m) & 1u) && acc.a >= fr.term) { taken_r = m + 1; term = true; }
                }
            }
#else
            for (int m = 0; m < cnt; ++m) {
                const double4 gg = shade[m][g];
                const double w = (1.0 - acc.a) * gg.x;
                acc.r += w * gg.y;
                acc.g += w * gg.z;
                acc.b += w * gg.w;
                acc.a += w;
                if (((fbits >> m) & 1u) && acc.a >= fr.term) { taken_r = m + 1; term = true; break; }
            }
#endif
            if (stats && j == 0) {
                atomicAdd(&g_stats[ST_ROUNDS], 1ull);
                if (cnt < G) atomicAdd(&g_stats[ST_PARTIAL], 1ull);
            }
        }
        __syncwarp();   // every lane has read s_acc
        if (active && !idle && j == 0) {
            s_acc[0][g] = acc.r; s_acc[1][g] = acc.g; s_acc[2][g] = acc.b; s_acc[3][g] = acc.a;
        }

        // ---- advance the group's cursor (all shuffles before any divergence)
        const int src = gbase + ((taken_r > 0) ? taken_r - 1 : 0);
        const int32_t i_last = __shfl_sync(FULL, i_mine, src);
        const uint32_t c0_last = __shfl_sync(FULL, c0_mine, src);
        const double ra_last = __shfl_sync(FULL, r_mine.a, src);
        const int32_t rpid_last = __shfl_sync(FULL, r_mine.pid, src);
        const uint32_t rcum_last = __shfl_sync(FULL, r_mine.cum, src);
        bool done = false, flush = false, suspend = false;
        int32_t flush_n = 0;
        uint32_t taken_now = 0;
        if (active) {
            if (idle) {  // inline intervals exhausted
                done = true;
            } else if (!inline_mode) {
                const uint32_t c_tot = s_ctot[g];
                taken_now = s_taken[g] + (uint32_t)taken_r;
                const int32_t n_iv = s_niv[g];
                if (term) {                       // K:388-389: the last interval visited
                    flush = true; flush_n = i_last + 1;
                    done = true;
                } else if (BRICK && taken_now == c_tot && c_tot != s_cfull[g]) {
                    flush = true; flush_n = n_iv;   // run done: the next brick continues
                    suspend = true;
                } else if (taken_now == c_tot) {  // stored list consumed
                    flush = true; flush_n = n_iv;
                    if (more) {
                        inline_mode = true;
                        if (j == 0) {
                            const IvRec *rec = iv.rec + (int64_t)s_rr[g] * IV_CAP;
                            L.t_min = iv.tail[s_rr[g]];
                            L.last = n_iv > 0 ? rec[n_iv - 1].pid : -1;
                            L.visited = 0; L.started = 1; L.n = 0; L.k = 0;
                        }
                    } else {
                        done = true;
                    }
                }
            } else {
                if (j == 0) {
                    L.k += taken_r;
                    if (track && L.pid >= 0)
                        atomicAdd((unsigned long long *)O.ppart + L.pid, (unsigned long long)taken_r);
                }
                if (term) done = true;
            }
        }
        // per-partition samples of the stored intervals (K:386-387)
        if (flush && track) {
            const IvRec *rec = iv.rec + (int64_t)s_rr[g] * IV_CAP;
            for (int32_t i = j; i < flush_n; i += G) {
                const IvRec r = load_rec(rec + i);
                uint32_t lo = (i > 0) ? load_rec(rec + (i - 1)).cum : 0u;
                if (BRICK && lo < s_tbegin[g]) lo = s_tbegin[g];   // this run's samples only
                const uint32_t hi = (r.cum < taken_now) ? r.cum : taken_now;
                if (hi > lo) atomicAdd((unsigned long long *)O.ppart + r.pid, (unsigned long long)(hi - lo));
            }
        }
        __syncwarp();
        if (active && j == 0) {
            const long long samples = s_samples[g] + taken_r;
            s_samples[g] = samples;
            if (!idle && taken_now) {
                s_taken[g] = taken_now;
                s_icur[g] = i_last;
                s_cbefore[g] = c0_last;
                s_ra[g] = ra_last; s_rpid[g] = rpid_last; s_rcum[g] = rcum_last;
            }
            if (done) {
                int32_t visited = 0;
                if (fr.mode != 0) {
                    if (!inline_mode) visited = term ? i_last + 1 : s_niv[g];
                    else visited = s_niv[g] + L.visited;
                }
#if TR_RAY_TIMES
                const Acc acc = {(double)s_tstart[g], (double)globaltimer_ns(), 0.0, 1.0};
#else
                const Acc acc = {s_acc[0][g], s_acc[1][g], s_acc[2][g], s_acc[3][g]};
#endif
                write_pixel(fr, O, s_out[g], acc, samples, visited);
                my_samples += (unsigned long long)samples;
                my_visited += (unsigned long long)visited;
                if (BRICK) {
                    TrRayState st = {};
                    st.flags = 2u;
                    F.B_state[s_rr[g]] = st;
                }
            } else if (BRICK && suspend) {
                TrRayState st = {};
                st.acc[0] = s_acc[0][g]; st.acc[1] = s_acc[1][g];
                st.acc[2] = s_acc[2][g]; st.acc[3] = s_acc[3][g];
                st.samples = samples;
                st.taken = s_taken[g]; st.icur = s_icur[g]; st.cbefore = s_cbefore[g];
                st.flags = 1u;
                F.B_state[s_rr[g]] = st;
                if (F.B_npeers) push_state(F, iv, s_rr[g], st);
            }
        }
        if (done || suspend) active = false;
        __syncwarp();
#if TR_ROUND_TIMES
        if (lane == 0) {
            DBG_T(r3);
            dbg_add(4, r1 - r0); dbg_add(5, r2 - r1); dbg_add(6, r3 - r2);
        }
#endif
    }
    if (timing && threadIdx.x == 0) atomicMax(&g_stats[ST_MARCH_T1], globaltimer_ns());
    // block reduction of the frame totals (R:198-201)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        my_samples += __shfl_xor_sync(FULL, my_samples, off);
        my_visited += __shfl_xor_sync(FULL, my_visited, off);
    }
    if (lane == 0) { red[0][warp] = my_samples; red[1][warp] = my_visited; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0, v = 0;
        for (int w = 0; w < BLK / 32; ++w) { s += red[0][w]; v += red[1][w]; }
        if (s) atomicAdd((unsigned long long *)O.totals, s);
        if (v) atomicAdd((unsigned long long *)O.totals + 1, v);
    }
}

__global__ void field_at_many_kernel(SceneK S, int64_t n, const double *__restrict__ pts,
                                     uint8_t *found, double *vals, int64_t *tet) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const PQuery q = make_query(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        LeafHint h;
        h.valid = false;
        double v;
        const uint32_t pos = field_at(S, q, h, false, true, v);
        found[i] = pos != UINT32_MAX ? 1 : 0;
        vals[i] = v;
        if (tet) tet[i] = pos == UINT32_MAX ? -1 : (S.pleaf_ids ? (int64_t)__ldg(S.pleaf_ids + pos) : (int64_t)pos);
    }
}

__global__ void pow_batch_kernel(int64_t n, const double *__restrict__ x,
                                 const double *__restrict__ y, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = ref_pow(x[i], y[i]);
}

__global__ void scatter_tiles_kernel(int64_t width, int64_t height, int64_t tiles_x,
                                     int64_t n_tiles, int32_t count, int64_t slots,
                                     const double *__restrict__ src_rgba,
                                     const int64_t *__restrict__ src_samples,
                                     const int32_t *__restrict__ src_visited, double *rgba,
                                     int64_t *samples, int32_t *visited) {
    const int64_t total = (int64_t)count * slots * (TILE_W * TILE_H);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lane = i % (TILE_W * TILE_H);
        const int64_t slot = (i / (TILE_W * TILE_H)) % slots;
        const int64_t rank = i / (TILE_W * TILE_H * slots);
        const int64_t tile = rank + (int64_t)count * slot;
        if (tile >= n_tiles) continue;
        const int64_t ix = (tile % tiles_x) * TILE_W + lane % TILE_W;
        const int64_t iy = (tile / tiles_x) * TILE_H + lane / TILE_W;
        if (ix >= width || iy >= height) continue;
        const int64_t o = iy * width + ix;
        const double2 *s = reinterpret_cast<const double2 *>(src_rgba + 4 * i);
        double2 *d = reinterpret_cast<double2 *>(rgba + 4 * o);
        d[0] = s[0];
        d[1] = s[1];
        samples[o] = src_samples[i];
        visited[o] = src_visited[i];
    }
}

thread_local int64_t g_last_launch[3] = {0, 0, 0};

int cuda_fail(cudaError_t e, const char *where) {
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    return tr_fail(TR_ECUDA, m.c_str());
}

SceneK make_scene(const TrDeviceScene *s) {
    SceneK S;
    S.tets = s->tets;
    S.pnodes = s->pnodes;
    S.pleaves = s->pleaves;
    S.pleaf_ids = s->pleaf_ids;
    S.bnodes = s->bnodes;
    S.pgrid = s->pgrid;
    S.pgrid_leaf = s->pgrid_leaf;
    S.part_lo = s->part_lo;
    S.part_hi = s->part_hi;
    S.knodes = s->knodes;
    S.kleaf_pids = s->kleaf_pids;
    for (int a = 0; a < 3; ++a) { S.kroot_lo[a] = s->kroot[a]; S.kroot_hi[a] = s->kroot[3 + a]; }
    S.centering = s->centering;
    for (int a = 0; a < 3; ++a) {
        S.gdim[a] = s->gdim[a];
        S.gorg[a] = s->gorg[a];
        S.gscale[a] = s->gscale[a];
    }
    for (int a = 0; a < 3; ++a) { S.mesh_lo[a] = s->mesh_lo[a]; S.mesh_hi[a] = s->mesh_hi[a]; }
    S.cell_off = s->cell_off;
    S.cell_recs = s->cell_recs;
    S.tbox = reinterpret_cast<const float4 *>(s->tbox);
    for (int a = 0; a < 3; ++a) { S.cdim[a] = s->cdim[a]; S.corg[a] = s->corg[a]; S.cscale[a] = s->cscale[a]; }
    S.cells_first = s->cells_first;
    if (!s->cell_recs || !s->tbox) S.cell_off = nullptr;
    S.pgrid_pred = reinterpret_cast<const float4 *>(s->pgrid_pred);
    S.pred_classes = s->pred_classes;
    for (int c = 0; c < 2; ++c)
        for (int k = 0; k < 12; ++k) S.pred_class[c][k] = (&s->pred_class[c].row[0][0])[k];
    S.grid_n = s->class_walk ? s->grid_n : 0;
    S.grid_pad = s->grid_pad;
    S.grid_brick = s->grid_brick;
    S.class_walk = s->class_walk;
    return S;
}

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Resident CTAs per SM of a kernel, cached per (device, kernel): the query
// costs several microseconds of host time on every frame otherwise.
static cudaError_t occupancy(int *out, const void *fn, int block, int smem = 0) {
    struct Ent { int dev; const void *fn; int block, smem, n; };
    static Ent cache[64];
    static int n_cache = 0;
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < n_cache; ++i)
        if (cache[i].dev == dev && cache[i].fn == fn && cache[i].block == block &&
            cache[i].smem == smem) {
            *out = cache[i].n;
            return cudaSuccess;
        }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, block, (size_t)smem);
    if (e == cudaSuccess && n_cache < 64) cache[n_cache++] = {dev, fn, block, smem, *out};
    return e;
}

// Side stream + events of background_kernel, per device (created on first use).
struct BgAux {
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_trace = nullptr, ev_bg = nullptr;
};
static std::mutex g_bg_mutex;

static int bg_aux(BgAux **out) {
    static BgAux aux[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= 64) return tr_fail(TR_EINVAL, "tr_render_frame: device index out of range");
    BgAux &a = aux[dev];
    if (!a.stream) {
        if ((e = cudaStreamCreateWithFlags(&a.stream, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&a.ev_trace, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&a.ev_bg, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "background stream setup");
    }
    *out = &a;
    return TR_OK;
}

constexpr int64_t IV_BYTES_PER_RAY = IV_CAP * 16 + 8 + 4 + 4 + 4 + 24 + CAND_CAP * 24;  // rec + tail + cnt + order + ccount + rinv + cand
constexpr int64_t IV_FIXED_BYTES = 1024;

// ---- brick-sharded frames (tr_brick_*)

// PEER exchange: a suspended ray's state goes to the inbox of the ONE rank
// that owns its next run (the brick of the interval holding sample `taken`,
// found as the plan finds it), in this round's parity slot, tagged so that
// the next round's plan takes exactly this round's entries.  Finished rays
// are not sent: their pixel is written here and no other rank plans a ray
// it was not sent.
__device__ __forceinline__ int brick_of(const FrameK &F, int32_t pid);
__device__ __noinline__ void push_state(const FrameK &F, const IvBuf &iv, int64_t rr, TrRayState st) {
    st.tag = F.B_tag + 1u;
    const int par = (int)(F.B_tag & 1u);
    const uint32_t n_iv = iv.cnt[rr] & 0xffffu;
    const IvRec *rec = iv.rec + rr * IV_CAP;
    int32_t i = st.icur;
    int nb = F.B_rank;   // no further interval (not expected): keep it here
    while (i < (int32_t)n_iv) {
        const IvRec r = load_rec(rec + i);
        if (r.cum > st.taken) { nb = brick_of(F, r.pid); break; }
        ++i;
    }
    TrRayState *dst = nb == F.B_rank ? F.B_inbox + (int64_t)par * F.n_rays : F.B_peer_inbox[2 * nb + par];
    if (dst) dst[rr] = st;
    __threadfence_system();
}

__device__ __forceinline__ int brick_of(const FrameK &F, int32_t pid) {
    return pid >= 0 ? (int)__ldg(F.B_owner + pid) : (-1 - pid);
}

// Every active ray's next run: the interval holding sample `taken`, its
// brick, and the run's end (the last following interval that is the same
// brick's or holds no sample).  Runs of F.B_rank are queued; with
// B_zero_foreign every other state is zeroed for the SUM exchange.
__global__ void __launch_bounds__(256) brick_plan_kernel(FrameK F, IvBuf iv) {
    const int lane = threadIdx.x & 31;
    for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x; r0 < F.n_rays; r0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rr = r0 + threadIdx.x;
        bool act = false, mine = false;
        uint32_t bucket = 0;
        TrRayState st = {};
        if (rr < F.n_rays) {
            st = F.B_state[rr];
            if (F.B_npeers && (F.B_tag & 255u) != 0u) {
                // after round 0 a rank plans only the rays sent to it last round
                const TrRayState in = F.B_inbox[(int64_t)((F.B_tag - 1u) & 1u) * F.n_rays + rr];
                if (in.tag == F.B_tag) {
                    st = in;
                    F.B_state[rr] = in;
                } else {
                    st.flags = 0u;
                }
            }
            act = st.flags == 1u;
        }
        if (act) {
            const uint32_t n_iv = iv.cnt[rr] & 0xffffu;
            const IvRec *rec = iv.rec + rr * IV_CAP;
            int32_t i = st.icur;
            uint32_t c0 = st.cbefore;
            IvRec r = load_rec(rec + i);
            while (r.cum <= st.taken) { c0 = r.cum; ++i; r = load_rec(rec + i); }
            const int b = brick_of(F, r.pid);
            int32_t i2 = i;
            uint32_t cend = r.cum;
            while (i2 + 1 < (int32_t)n_iv) {
                const IvRec r2 = load_rec(rec + i2 + 1);
                if (r2.cum != cend && brick_of(F, r2.pid) != b) break;
                ++i2;
                cend = r2.cum;
            }
            if (b == F.B_rank) {
                mine = true;
                st.icur = i;
                st.cbefore = c0;
                st.stop = cend;
                F.B_state[rr] = st;
                bucket = cost_bucket((double)(cend - st.taken));
            }
        }
        if (rr < F.n_rays && !mine && F.B_zero_foreign) {
            const TrRayState z = {};
            F.B_state[rr] = z;
        }
        const unsigned am = __ballot_sync(FULL, act), mm = __ballot_sync(FULL, mine);
        if (lane == 0 && am) atomicAdd(F.B_ctr + 1, (unsigned)__popc(am));
        unsigned base = 0;
        if (lane == 0 && mm) base = atomicAdd(F.B_ctr, (unsigned)__popc(mm));
        base = __shfl_sync(FULL, base, 0);
        unsigned long long run = mine ? (unsigned long long)(st.stop - st.taken) : 0ull, run_max = run;
        for (int o = 16; o; o >>= 1) {
            run += __shfl_xor_sync(FULL, run, o);
            const unsigned long long m = __shfl_xor_sync(FULL, run_max, o);
            run_max = m > run_max ? m : run_max;
        }
        if (lane == 0 && mm) {   // this round's work and longest run: the lane width
            atomicAdd(iv.ray_stats, run);
            atomicMax(iv.ray_stats + 1, run_max);
        }
        if (mine) {   // unsorted; brick_order_kernel sorts the runs longest first
            iv.order[base + __popc(mm & ((1u << lane) - 1u))] = (uint32_t)rr;
            const unsigned peers = __match_any_sync(mm, bucket);
            if (lane == __ffs(peers) - 1) atomicAdd(iv.hist + bucket, (unsigned)__popc(peers));
        }
    }
}

// This round's queue in descending run-length buckets (the one-device
// march's longest-first order, order_rays_kernel, applied to the runs): a
// round ends with its longest run, so starting the long runs first shortens
// the round's tail.  Order inside a bucket is arbitrary; outputs do not
// depend on it.
__global__ void __launch_bounds__(256) brick_order_kernel(FrameK F, IvBuf iv) {
    __shared__ uint32_t start[N_BUCKETS];
    if (blockIdx.x == 0 && threadIdx.x == 0) {   // order_rays_kernel's lane-width rule on the runs
        const unsigned long long sum = iv.ray_stats[0], mx = iv.ray_stats[1];
        *iv.gsel = (mx * (unsigned long long)F.march_lanes <= 4ull * sum) ? 4u : 16u;
    }
    if (threadIdx.x < N_BUCKETS) {
        uint32_t s = 0;
        for (int b = N_BUCKETS - 1; b > (int)threadIdx.x; --b) s += iv.hist[b];
        start[threadIdx.x] = s;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t n = *F.B_ctr;
    for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x; e0 < n; e0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = e0 + threadIdx.x;
        const bool valid = e < n;
        const unsigned vm = __ballot_sync(FULL, valid);
        if (!valid) continue;
        const uint32_t rr = iv.order[e];
        const TrRayState &st = F.B_state[rr];
        const uint32_t bucket = cost_bucket((double)(st.stop - st.taken));
        const unsigned peers = __match_any_sync(vm, bucket);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(iv.cursor + bucket, (unsigned)__popc(peers));
        base = __shfl_sync(peers, base, leader);
        F.B_queue[start[bucket] + base + __popc(peers & ((1u << lane) - 1u))] = rr;
    }
}

}  // namespace

extern "C" {

int64_t tr_num_tiles(int64_t width, int64_t height) {
    return ((width + TILE_W - 1) / TILE_W) * ((height + TILE_H - 1) / TILE_H);
}

int64_t tr_slots_per_rank(int64_t width, int64_t height, int32_t count) {
    if (count < 1) return 0;
    return (tr_num_tiles(width, height) + count - 1) / count;
}

int64_t tr_scratch_bytes(int64_t n_rays) {
    return n_rays * IV_BYTES_PER_RAY + IV_FIXED_BYTES + 16;
}

// Validation and the kernel-side views shared by tr_render_frame and the
// brick-sharded calls.
// The chunk's interval lists and counters in out->scratch.
static IvBuf make_iv(const TrOutputs *out, int64_t n_rays) {
    IvBuf iv;
    char *base = reinterpret_cast<char *>(out->scratch);
    iv.hist = reinterpret_cast<uint32_t *>(base);
    iv.cursor = iv.hist + N_BUCKETS;
    iv.trace_ctr = iv.cursor + N_BUCKETS;
    iv.ray_stats = reinterpret_cast<unsigned long long *>(base + 528);
    iv.gsel = reinterpret_cast<uint32_t *>(base + 544);
    iv.n_bg = reinterpret_cast<uint32_t *>(base + 548);
    iv.totals = reinterpret_cast<unsigned long long *>(out->totals);
    iv.rec = reinterpret_cast<IvRec *>(base + IV_FIXED_BYTES);
    iv.tail = reinterpret_cast<double *>(iv.rec + (int64_t)IV_CAP * n_rays);
    iv.cnt = reinterpret_cast<uint32_t *>(iv.tail + n_rays);
    iv.order = iv.cnt + n_rays;
    iv.ccount = iv.order + n_rays;
    char *c = base + IV_FIXED_BYTES + ((n_rays * (IV_CAP * 16 + 8 + 4 + 4 + 4) + 15) / 16) * 16;
    iv.rinv = reinterpret_cast<double *>(c);
    iv.cand_pa = iv.rinv + 3 * n_rays;
    iv.cand_pb = iv.cand_pa + (int64_t)CAND_CAP * n_rays;
    iv.cand_pid = reinterpret_cast<int32_t *>(iv.cand_pb + (int64_t)CAND_CAP * n_rays);
    iv.cand_nkey = reinterpret_cast<float *>(iv.cand_pid + (int64_t)CAND_CAP * n_rays);
    return iv;
}

static cudaError_t launch_cand_raster(const SceneK &S, const EpochK &E, const FrameK &F,
                                      const IvBuf &iv, cudaStream_t st) {
    ray_table_kernel<<<(unsigned)((F.n_rays + 255) / 256), 256, 0, st>>>(F, iv);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    FrameK G = F;
    // warps per partition rectangle ~ pixels of the chunk's band / 256K (1 at
    // 512^2; rectangles grow with the frame, so large frames spread wider)
    const int64_t rows = (F.n_rays / 32 + F.tiles_x - 1) / F.tiles_x * TILE_H;
    G.raster_sub = (int32_t)std::min<int64_t>(std::max<int64_t>(F.f.width * rows / TR_RASTER_PX, 1), 64);
    int64_t grid = (F.n_parts * G.raster_sub + 7) / 8;
    if (grid > (int64_t)sm_count() * 8) grid = (int64_t)sm_count() * 8;
    if (grid < 1) grid = 1;
    cand_raster_kernel<<<(unsigned)grid, 256, 0, st>>>(S, E, G, iv);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // a CTA per 32-ray tile, no grid stride: empty tiles retire at once and
    // the scheduler refills their slots
    const int64_t sg = (F.n_rays + 31) / 32;
    cand_sort_kernel<<<(unsigned)sg, SORT_THREADS, 0, st>>>(F, iv);
    return cudaGetLastError();
}

static int prepare_frame(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                         const TrOutputs *out, SceneK &S, EpochK &E, FrameK &F) {
    if (!scene || !epoch || !frame || !out)
        return tr_fail(TR_EINVAL, "tr_render_frame: null argument");
    if (frame->width < 1 || frame->height < 1 || frame->mode < 0 || frame->mode > 2 ||
        frame->shard_count < 1 || frame->shard_rank < 0 || frame->shard_rank >= frame->shard_count)
        return tr_fail(TR_EINVAL, "tr_render_frame: invalid frame");
    if (!scene->tets || !scene->pnodes || !scene->pleaves || !out->rgba ||
        !out->samples || !out->visited || !out->totals || !out->work || !epoch->tf_table ||
        epoch->n_tf < 2)
        return tr_fail(TR_EINVAL, "tr_render_frame: missing buffer");
    if (frame->mode != 0 && (!scene->bnodes || !epoch->active || !epoch->bnode_active ||
                             (frame->mode == 2 && (!epoch->step || !epoch->step_ratio))))
        return tr_fail(TR_EINVAL, "tr_render_frame: missing partition buffers");
    if (frame->track_ppart && frame->mode != 0 && !out->ppart)
        return tr_fail(TR_EINVAL, "tr_render_frame: missing ppart buffer");
    S = make_scene(scene);
    E = EpochK{};
    E.active = epoch->active;
    E.knode_active = epoch->knode_active;
    E.bnode_active = epoch->bnode_active;
    E.step = epoch->step;
    E.step_ratio = epoch->step_ratio;
    E.tf = epoch->tf_table;
    E.n_tf = epoch->n_tf;
    E.tf_lo = epoch->tf_lo;
    E.tf_hi = epoch->tf_hi;
    F = FrameK{};
    F.f = *frame;
    F.tiles_x = (frame->width + TILE_W - 1) / TILE_W;
    F.n_tiles = tr_num_tiles(frame->width, frame->height);
    F.my_tiles = (F.n_tiles - frame->shard_rank + frame->shard_count - 1) / frame->shard_count;
    if (F.my_tiles < 0) F.my_tiles = 0;
    F.n_parts = (int32_t)scene->n_parts;
    // candidate raster up to 1M pixels; beyond, neighbouring rays are coherent
    // enough that the BSP walk is as fast (measured equal at 1024^2-2048^2,
    // 3% faster at 4096^2, while the raster wins 13% at 512^2)
    F.use_cand = (frame->mode != 0 && !(frame->flags & TR_FLAG_NO_CAND) &&
                  ((int64_t)frame->width * frame->height <= (1 << 20) ||
                   (frame->flags & TR_FLAG_FORCE_CAND))) ? 1 : 0;
    return TR_OK;
}

// render()'s synchronous frame in one call (DeviceScene.render): counter
// reset, the frame's kernels bracketed by events, the counters (and the
// epoch's inexact word) copied to page-locked memory, stream synchronize.
int tr_render_sync(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                   const TrOutputs *out, int64_t n_counters, int64_t *counters_host,
                   int32_t *inexact_host, void *stream, float *device_ms,
                   const TrEpochUpload *reupload) {
    if (!out || !out->totals || n_counters < 3 || !counters_host)
        return tr_fail(TR_EINVAL, "tr_render_sync: invalid arguments");
    struct Ev { int dev = -1; cudaEvent_t a = nullptr, b = nullptr; };
    thread_local Ev ev;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "tr_render_sync");
    if (ev.dev != dev) {
        if ((e = cudaEventCreate(&ev.a)) != cudaSuccess || (e = cudaEventCreate(&ev.b)) != cudaSuccess)
            return cuda_fail(e, "tr_render_sync events");
        ev.dev = dev;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (reupload) {   // the same buffers: `epoch` stays valid
        TrEpoch again;
        if (int rc = tr_epoch_upload_s(reupload, &again, nullptr, stream)) return rc;
    }
    if ((e = cudaMemsetAsync(out->totals, 0, 8 * n_counters, st)) != cudaSuccess ||
        (e = cudaEventRecord(ev.a, st)) != cudaSuccess)
        return cuda_fail(e, "tr_render_sync reset");
    if (int rc = tr_render_frame(scene, epoch, frame, out, stream)) return rc;
    if ((e = cudaEventRecord(ev.b, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(counters_host, out->totals, 8 * n_counters, cudaMemcpyDeviceToHost,
                             st)) != cudaSuccess)
        return cuda_fail(e, "tr_render_sync copy");
    if (inexact_host && epoch->inexact &&
        (e = cudaMemcpyAsync(inexact_host, epoch->inexact, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return cuda_fail(e, "tr_render_sync copy");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "tr_render_sync sync");
    if (device_ms && (e = cudaEventElapsedTime(device_ms, ev.a, ev.b)) != cudaSuccess)
        return cuda_fail(e, "tr_render_sync elapsed");
    return TR_OK;
}

int tr_render_frame(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                    const TrOutputs *out, void *stream) {
    SceneK S;
    EpochK E;
    FrameK F;
    if (int rc = prepare_frame(scene, epoch, frame, out, S, E, F)) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t total_rays = F.my_tiles * (TILE_W * TILE_H);
    // ray chunk = what the scratch interval lists can hold
    if (!out->scratch || out->scratch_bytes < IV_BYTES_PER_RAY * 32 + IV_FIXED_BYTES)
        return tr_fail(TR_EINVAL, "tr_render_frame: scratch buffer too small");
    int64_t chunk = (out->scratch_bytes - IV_FIXED_BYTES) / IV_BYTES_PER_RAY / 32 * 32;
    if (chunk > total_rays) chunk = total_rays;
    if (chunk < 32) chunk = 32;
    // lanes per ray: flags bits 8-11 = log2(G) (0: default 4); bits 12-13:
    // minimum resident CTAs per SM of the G = 4 kernel (register budget; 0: 2)
    const int lg = (frame->flags >> 8) & 0xf;
    const int gsize = lg ? (1 << lg) : 4;
    // bits 12-13: minimum resident CTAs per SM (register budget); 0 = 3 CTAs
    // (80 registers, 24 warps): measured best or within 3% from 1e6 to 1e9
    // tets (32 warps spill and thrash L1; 16 hide too little latency)
    int minb = (frame->flags >> 12) & 0x3;
    if (minb == 0) minb = 3;
    void (*march_fn)(SceneK, EpochK, FrameK, IvBuf, TrOutputs);
    if (frame->flags & TR_FLAG_REG_STATE) {   // ray state in registers (2 CTAs per SM)
        switch (gsize) {
            case 2: march_fn = march_kernel<2, 2, false>; break;
            case 4: march_fn = march_kernel<4, 2, false>; break;
            case 8: march_fn = march_kernel<8, 2, false>; break;
            case 16: march_fn = march_kernel<16, 2, false>; break;
            case 32: march_fn = march_kernel<32, 2, false>; break;
            default: return tr_fail(TR_EINVAL, "tr_render_frame: group size must be 2, 4, 8, 16 or 32");
        }
    } else {
        switch (gsize) {
            case 2: march_fn = march_sm_kernel<2, 3>; break;
            case 4: march_fn = minb == 2 ? march_sm_kernel<4, 2>
                             : (minb == 1 ? march_sm_kernel<4, 4>
                                : ((frame->flags & TR_FLAG_STATS) ? march_sm_kernel<4, MB, false, true>
                                                                  : march_sm_kernel<4, MB>)); break;
            case 8: march_fn = march_sm_kernel<8, 3>; break;
            case 16: march_fn = march_sm_kernel<16, MB>; break;
            default: return tr_fail(TR_EINVAL, "tr_render_frame: group size must be 2, 4, 8 or 16");
        }
    }
    // reference and skip modes never evaluate pow: 128-thread CTAs budgeted for
    // 7 per SM (72 registers, 28 warps) hide more latency there (-4%, profiles/r02)
    int march_block = MARCH_BLOCK;
    void (*march16_fn)(SceneK, EpochK, FrameK, IvBuf, TrOutputs) = march_sm_kernel<16, MB>;
    if (frame->mode != 2 && lg == 0 && minb == 3 && !(frame->flags & (TR_FLAG_REG_STATE | TR_FLAG_STATS))) {
        march_fn = march_sm_kernel<4, 7, false, false, 128>;
        march16_fn = march_sm_kernel<16, 7, false, false, 128>;
        march_block = 128;
    }
    cudaError_t e;
    int per_sm = 0;
    const int tabs_smem = march_tabs_bytes(march_block, epoch->n_tf);   // MarchTabs (dynamic smem)
    e = occupancy(&per_sm, (const void *)march_fn, march_block, tabs_smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (per_sm < 1) per_sm = 1;
    if ((frame->flags >> 14) & 0x3) per_sm = (frame->flags >> 14) & 0x3;  // tuning: CTAs per SM
    F.auto_g = (lg == 0 && !(frame->flags & TR_FLAG_REG_STATE) && minb == 3) ? 1 : 0;
    F.march_lanes = (int64_t)sm_count() * per_sm * march_block;
    int trace_per_sm = 0;
    void (*trace_fn)(SceneK, EpochK, FrameK, IvBuf, TrOutputs) =
        (frame->flags & TR_FLAG_STATS) ? trace_intervals_kernel<true> : trace_intervals_kernel<false>;
    e = occupancy(&trace_per_sm, (const void *)trace_fn, TRACE_BLOCK);
    if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor(trace)");
    if (trace_per_sm < 1) trace_per_sm = 1;
    if ((frame->flags >> 20) & 0x7) trace_per_sm = (frame->flags >> 20) & 0x7;   // tuning: trace CTAs per SM
    // a page-locked host framebuffer: the march's pixel stores go over PCIe
    // as it runs; the background pixels go to background_kernel
    F.defer_bg = 0;
    {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, out->rgba) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            !(frame->flags & TR_FLAG_NO_BG_WRITER))
            F.defer_bg = 1;
        else
            cudaGetLastError();
    }
    BgAux *aux = nullptr;
    std::unique_lock<std::mutex> bg_lock;
    if (F.defer_bg) {
        bg_lock = std::unique_lock<std::mutex>(g_bg_mutex);
        if (int rc = bg_aux(&aux)) return rc;
    }
    int64_t launches = 0, march_grid = 0;
    for (int64_t r0 = 0; r0 < total_rays; r0 += chunk) {
        F.ray_begin = r0;
        F.n_rays = (total_rays - r0 < chunk) ? total_rays - r0 : chunk;
        IvBuf iv = make_iv(out, F.n_rays);
        e = cudaMemsetAsync(out->work, 0, sizeof(uint32_t), st);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(work)");
        e = cudaMemsetAsync(iv.hist, 0, 552, st);   // hist, cursor, trace_ctr, ray_stats, gsel, n_bg
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(hist)");
        if (F.use_cand) {
            if ((e = launch_cand_raster(S, E, F, iv, st)) != cudaSuccess) return cuda_fail(e, "cand_raster_kernel");
            launches += 3;   // ray table, raster, sort
        }
        const int64_t tg = (F.n_rays + TRACE_BLOCK - 1) / TRACE_BLOCK;
        const int64_t trace_grid = (tg < (int64_t)sm_count() * trace_per_sm) ? tg : (int64_t)sm_count() * trace_per_sm;
        trace_fn<<<(unsigned)trace_grid, TRACE_BLOCK, 0, st>>>(S, E, F, iv, *out);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "trace_intervals_kernel launch");
        if (F.defer_bg) {
            if ((e = cudaEventRecord(aux->ev_trace, st)) != cudaSuccess ||
                (e = cudaStreamWaitEvent(aux->stream, aux->ev_trace, 0)) != cudaSuccess)
                return cuda_fail(e, "background stream fork");
            background_kernel<<<BG_CTAS, BG_THREADS, 0, aux->stream>>>(F, iv, *out);
            if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "background_kernel launch");
            if ((e = cudaEventRecord(aux->ev_bg, aux->stream)) != cudaSuccess)
                return cuda_fail(e, "background stream record");
            ++launches;
        }
        order_rays_kernel<<<(unsigned)tg, TRACE_BLOCK, 0, st>>>(F, iv);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "order_rays_kernel launch");
        launches += 2;
        if (out->ev_march_begin && r0 == 0) {
            e = cudaEventRecord((cudaEvent_t)out->ev_march_begin, st);
            if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord(begin)");
        }
        // auto width: the G = 4 and 16 kernels are both launched and the one
        // order_rays_kernel did not choose returns at once
        void (*fns[2])(SceneK, EpochK, FrameK, IvBuf, TrOutputs) = {march_fn, nullptr};
        int gs[2] = {gsize, 0};
        int nf = 1;
        if (F.auto_g) {
            fns[1] = march16_fn;
            gs[1] = 16;
            nf = 2;
        }
        for (int q = 0; q < nf; ++q) {
            int64_t grid = (int64_t)sm_count() * per_sm;
            const int64_t need = (F.n_rays * gs[q] + march_block - 1) / march_block;
            if (grid > need) grid = need;
            if (grid < 1) grid = 1;
            fns[q]<<<(unsigned)grid, march_block, tabs_smem, st>>>(S, E, F, iv, *out);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "march_kernel launch");
            ++launches;
            if (q == 0) march_grid = grid;
        }
        if (F.defer_bg) {   // join: the next chunk reuses the list; the frame ends after it
            e = cudaStreamWaitEvent(st, aux->ev_bg, 0);
            if (e != cudaSuccess) return cuda_fail(e, "background stream join");
        }
        if (out->ev_march_end && r0 + chunk >= total_rays) {
            e = cudaEventRecord((cudaEvent_t)out->ev_march_end, st);
            if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord(end)");
        }
    }
    g_last_launch[0] = launches;
    g_last_launch[1] = march_grid;
    g_last_launch[2] = march_block;
    return TR_OK;
}

int tr_field_at_many(const TrDeviceScene *scene, int64_t n, const double *pts, uint8_t *found,
                     double *vals, int64_t *tet, void *stream) {
    if (!scene || n < 0 || (n > 0 && (!pts || !found || !vals)))
        return tr_fail(TR_EINVAL, "tr_field_at_many: invalid arguments");
    if (n == 0) return TR_OK;
    SceneK S = make_scene(scene);
    int64_t grid = (n + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    field_at_many_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(S, n, pts, found, vals, tet);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "field_at_many_kernel launch");
    return TR_OK;
}

int tr_scatter_tiles(int64_t width, int64_t height, int32_t count, const double *src_rgba,
                     const int64_t *src_samples, const int32_t *src_visited,
                     int64_t slots_per_rank, double *rgba, int64_t *samples, int32_t *visited,
                     void *stream) {
    if (width < 1 || height < 1 || count < 1 || slots_per_rank < 0 || !src_rgba || !src_samples ||
        !src_visited || !rgba || !samples || !visited)
        return tr_fail(TR_EINVAL, "tr_scatter_tiles: invalid arguments");
    const int64_t total = (int64_t)count * slots_per_rank * TILE_W * TILE_H;
    if (total == 0) return TR_OK;
    int64_t grid = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (grid > cap) grid = cap;
    scatter_tiles_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
        width, height, (width + TILE_W - 1) / TILE_W, tr_num_tiles(width, height), count,
        slots_per_rank, src_rgba, src_samples, src_visited, rgba, samples, visited);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "scatter_tiles_kernel launch");
    return TR_OK;
}

int tr_kernel_stats(int64_t *out, int32_t n, int32_t reset) {
    unsigned long long h[32];
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "tr_kernel_stats sync");
    e = cudaMemcpyFromSymbol(h, g_stats, sizeof h);
    if (e != cudaSuccess) return cuda_fail(e, "tr_kernel_stats copy");
    for (int i = 0; i < n && i < 32; ++i) out[i] = (int64_t)h[i];
#if TR_ROUND_TIMES   // slots 24-31: the phase sums over every thread
    {
        static unsigned long long dbg[DBG_THREADS * DBG_PH];
        if ((e = cudaMemcpyFromSymbol(dbg, g_dbg, sizeof dbg)) != cudaSuccess)
            return cuda_fail(e, "tr_kernel_stats dbg");
        for (int ph = 0; ph < DBG_PH && 24 + ph < n; ++ph) {
            unsigned long long t = 0;
            for (int i = 0; i < DBG_THREADS; ++i) t += dbg[i * DBG_PH + ph];
            out[24 + ph] = (int64_t)t;
        }
        if (reset) {
            for (int i = 0; i < DBG_THREADS * DBG_PH; ++i) dbg[i] = 0;
            if ((e = cudaMemcpyToSymbol(g_dbg, dbg, sizeof dbg)) != cudaSuccess)
                return cuda_fail(e, "tr_kernel_stats dbg reset");
        }
    }
#endif
    if (reset) {
        for (int i = 0; i < 32; ++i) h[i] = 0;
        h[ST_MARCH_T0] = h[ST_MARCH_TQ] = ~0ull;   // atomicMin slots
        e = cudaMemcpyToSymbol(g_stats, h, sizeof h);
        if (e != cudaSuccess) return cuda_fail(e, "tr_kernel_stats reset");
    }
    return TR_OK;
}

int tr_pow_glibc_batch(int64_t n, const double *x, const double *y, double *out, void *stream) {
    if (n < 0 || (n > 0 && (!x || !y || !out)))
        return tr_fail(TR_EINVAL, "tr_pow_glibc_batch: invalid arguments");
    if (n == 0) return TR_OK;
    int64_t grid = (n + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    pow_batch_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(n, x, y, out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pow_batch_kernel launch");
    return TR_OK;
}

int tr_memset_async(void *dst, int32_t value, int64_t bytes, void *stream) {
    if (!dst || bytes < 0) return tr_fail(TR_EINVAL, "tr_memset_async: invalid arguments");
    cudaError_t e = cudaMemsetAsync(dst, value, (size_t)bytes, (cudaStream_t)stream);
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "cudaMemsetAsync");
}

int tr_copy_async(void *dst, const void *src, int64_t bytes, void *stream) {
    if (!dst || !src || bytes < 0) return tr_fail(TR_EINVAL, "tr_copy_async: invalid arguments");
    cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream);
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "cudaMemcpyAsync");
}

int tr_host_device_pointer(void *host, void **dev) {
    if (!host || !dev) return tr_fail(TR_EINVAL, "tr_host_device_pointer: null");
    cudaError_t e = cudaHostGetDevicePointer(dev, host, 0);
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostGetDevicePointer");
    return TR_OK;
}

int tr_host_register(void *host, int64_t bytes, void **dev) {
    if (!host || bytes <= 0 || !dev) return tr_fail(TR_EINVAL, "tr_host_register: invalid arguments");
    cudaError_t e = cudaHostRegister(host, (size_t)bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostRegister");
    e = cudaHostGetDevicePointer(dev, host, 0);
    if (e != cudaSuccess) {
        cudaHostUnregister(host);
        return cuda_fail(e, "cudaHostGetDevicePointer");
    }
    return TR_OK;
}

int tr_host_unregister(void *host) {
    if (!host) return tr_fail(TR_EINVAL, "tr_host_unregister: null");
    cudaError_t e = cudaHostUnregister(host);
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "cudaHostUnregister");
}

int tr_last_launch(int64_t *out3) {
    if (!out3) return tr_fail(TR_EINVAL, "tr_last_launch: null");
    for (int i = 0; i < 3; ++i) out3[i] = g_last_launch[i];
    return TR_OK;
}

static int brick_setup(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                       const TrBricks *bricks, const TrOutputs *out, SceneK &S, EpochK &E,
                       FrameK &F, IvBuf &iv) {
    if (int rc = prepare_frame(scene, epoch, frame, out, S, E, F)) return rc;
    if (!bricks || bricks->n_bricks < 1 || bricks->n_bricks > 64 || bricks->rank < 0 ||
        bricks->rank >= bricks->n_bricks || !bricks->owner || !bricks->brick_lo ||
        !bricks->brick_hi || !bricks->state || !bricks->queue || !bricks->counters)
        return tr_fail(TR_EINVAL, "tr_brick: invalid TrBricks");
    if (frame->flags & TR_FLAG_REG_STATE)
        return tr_fail(TR_EINVAL, "tr_brick: TR_FLAG_REG_STATE is not supported");
    const int64_t total_rays = F.my_tiles * (TILE_W * TILE_H);
    if (!out->scratch || out->scratch_bytes < tr_scratch_bytes(total_rays))
        return tr_fail(TR_EINVAL, "tr_brick: the frame must fit one ray chunk (scratch too small)");
    F.ray_begin = 0;
    F.n_rays = total_rays;
    F.B_on = 1;
    F.B_rank = bricks->rank;
    F.B_n = bricks->n_bricks;
    F.B_write_bg = bricks->write_background;
    F.B_zero_foreign = bricks->zero_foreign;
    F.B_owner = bricks->owner;
    F.B_lo = bricks->brick_lo;
    F.B_hi = bricks->brick_hi;
    F.B_state = bricks->state;
    F.B_queue = bricks->queue;
    F.B_ctr = bricks->counters;
    F.B_tag = bricks->exchange_tag;
    F.B_npeers = bricks->n_peers;
    F.B_peer_inbox = bricks->peer_inbox;
    F.B_inbox = bricks->inbox;
    if (F.B_npeers && (!F.B_peer_inbox || !F.B_inbox || F.B_zero_foreign || bricks->exchange_tag < 256))
        return tr_fail(TR_EINVAL, "tr_brick: PEER exchange needs peer_inbox, inbox, zero_foreign = 0 "
                                  "and exchange_tag >= 256");
    iv = make_iv(out, F.n_rays);
    return TR_OK;
}

int tr_brick_trace(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                   const TrBricks *bricks, const TrOutputs *out, void *stream) {
    SceneK S;
    EpochK E;
    FrameK F;
    IvBuf iv;
    if (int rc = brick_setup(scene, epoch, frame, bricks, out, S, E, F, iv)) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if ((e = cudaMemsetAsync(iv.hist, 0, 552, st)) != cudaSuccess ||
        (e = cudaMemsetAsync(bricks->counters, 0, 16, st)) != cudaSuccess ||
        (e = cudaMemsetAsync(bricks->state, 0, sizeof(TrRayState) * F.n_rays, st)) != cudaSuccess)
        return cuda_fail(e, "tr_brick_trace memset");
    if (F.n_rays == 0) return TR_OK;
    if (F.use_cand && (e = launch_cand_raster(S, E, F, iv, st)) != cudaSuccess)
        return cuda_fail(e, "cand_raster_kernel (bricks)");
    void (*trace_fn)(SceneK, EpochK, FrameK, IvBuf, TrOutputs) =
        (frame->flags & TR_FLAG_STATS) ? trace_intervals_kernel<true> : trace_intervals_kernel<false>;
    int trace_per_sm = 0;
    if ((e = occupancy(&trace_per_sm, (const void *)trace_fn, TRACE_BLOCK)) != cudaSuccess)
        return cuda_fail(e, "occupancy(trace)");
    if (trace_per_sm < 1) trace_per_sm = 1;
    const int64_t tg = (F.n_rays + TRACE_BLOCK - 1) / TRACE_BLOCK;
    const int64_t cap = (int64_t)sm_count() * trace_per_sm;
    trace_fn<<<(unsigned)(tg < cap ? tg : cap), TRACE_BLOCK, 0, st>>>(S, E, F, iv, *out);
    e = cudaGetLastError();
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "trace_intervals_kernel launch (bricks)");
}

int tr_brick_round(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                   const TrBricks *bricks, const TrOutputs *out, void *stream) {
    SceneK S;
    EpochK E;
    FrameK F;
    IvBuf iv;
    if (int rc = brick_setup(scene, epoch, frame, bricks, out, S, E, F, iv)) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if ((e = cudaMemsetAsync(bricks->counters, 0, 8, st)) != cudaSuccess ||
        (e = cudaMemsetAsync(iv.hist, 0, 552, st)) != cudaSuccess ||   // hist .. gsel
        (e = cudaMemsetAsync(out->work, 0, sizeof(uint32_t), st)) != cudaSuccess)
        return cuda_fail(e, "tr_brick_round memset");
    if (F.n_rays == 0) return TR_OK;
    int64_t pg = (F.n_rays + 255) / 256;
    if (pg > (int64_t)sm_count() * 8) pg = (int64_t)sm_count() * 8;
    brick_plan_kernel<<<(unsigned)pg, 256, 0, st>>>(F, iv);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "brick_plan_kernel launch");
    // lanes per ray as in tr_render_frame (4, or 16 when the round's
    // longest run would set its time): both widths launch, one returns
    void (*fns[2])(SceneK, EpochK, FrameK, IvBuf, TrOutputs) = {march_sm_kernel<4, 3, true>,
                                                                march_sm_kernel<16, 3, true>};
    const int gs[2] = {4, 16};
    int per_sm = 0;
    const int tabs_smem = march_tabs_bytes(MARCH_BLOCK, epoch->n_tf);
    if ((e = occupancy(&per_sm, (const void *)fns[0], MARCH_BLOCK, tabs_smem)) != cudaSuccess)
        return cuda_fail(e, "occupancy(march)");
    if (per_sm < 1) per_sm = 1;
    F.auto_g = 1;
    F.march_lanes = (int64_t)sm_count() * per_sm * MARCH_BLOCK;
    brick_order_kernel<<<(unsigned)pg, 256, 0, st>>>(F, iv);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "brick_order_kernel launch");
    for (int q = 0; q < 2; ++q) {
        int64_t grid = (int64_t)sm_count() * per_sm;
        const int64_t need = (F.n_rays * gs[q] + MARCH_BLOCK - 1) / MARCH_BLOCK;
        if (grid > need) grid = need;
        if (grid < 1) grid = 1;
        fns[q]<<<(unsigned)grid, MARCH_BLOCK, tabs_smem, st>>>(S, E, F, iv, *out);
        if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "march_sm_kernel launch (bricks)");
    }
    return TR_OK;
}

}  // extern "C"
