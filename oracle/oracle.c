/*
 * oracle.c -- CPU restatement of the tetray hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity ORACLE, not the product.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product path (paper_1908_01906_b200.render) never calls
 * into it and fails loudly when its CUDA library is missing.
 *
 * It restates, in plain C99 with OpenMP over image rows, the numba kernels of
 * the reference renderer:
 *
 *   reference  pkg/src/tetray/_kernels.py  (abbreviated K below)
 *              pkg/src/tetray/bvh.py       (median-split flat BVH builder)
 *
 * Arithmetic contract: every expression is evaluated
 * in Python's left-to-right order, in IEEE binary64, with NO contraction
 * (build with -ffp-contract=off, no -ffast-math).  `x ** y` is glibc pow(),
 * exactly what numba lowers llvm.pow.f64 to, so results are bit-identical to
 * the reference; this is pinned against fixtures produced by running the
 * reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BARY_TOL 1e-9 /* K:15 */
#define STACK 128     /* K:17 */

/* ---------------------------------------------------------------- scalars */

/* K:20-22  max(s1 + (s2-s1)*abs(min(sigma,1)-1)**p, s1) with Python min/max. */
double orc_step_size(double s1, double s2, double p, double sigma) {
    double m = (1.0 < sigma) ? 1.0 : sigma;        /* min(sigma, 1.0) */
    double v = s1 + (s2 - s1) * pow(fabs(m - 1.0), p);
    return (s1 > v) ? s1 : v;                      /* max(v, s1) */
}

/* K:25-27 */
double orc_opacity_correction(double alpha, double s, double s1) {
    return 1.0 - pow(1.0 - alpha, s / s1);
}

/* K:30-71  ray/box interval; a miss returns t0 > t1 (1, 0 for a parallel miss). */
static inline void slab(double ox, double oy, double oz, double dx, double dy, double dz,
                        double lx, double ly, double lz, double hx, double hy, double hz,
                        double *r0, double *r1) {
    double t0 = -INFINITY, t1 = INFINITY;
    const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
    const double lo[3] = {lx, ly, lz}, hi[3] = {hx, hy, hz};
    for (int ax = 0; ax < 3; ++ax) {
        if (d[ax] != 0.0) {
            double inv = 1.0 / d[ax];
            double a = (lo[ax] - o[ax]) * inv;
            double b = (hi[ax] - o[ax]) * inv;
            if (a > b) { double t = a; a = b; b = t; }
            if (a > t0) t0 = a;
            if (b < t1) t1 = b;
        } else if (o[ax] < lo[ax] || o[ax] > hi[ax]) {
            *r0 = 1.0; *r1 = 0.0;
            return;
        }
    }
    *r0 = t0; *r1 = t1;
}

void orc_slab(const double *o, const double *d, const double *lo, const double *hi,
              double *out2) {
    slab(o[0], o[1], o[2], d[0], d[1], d[2], lo[0], lo[1], lo[2], hi[0], hi[1], hi[2],
         &out2[0], &out2[1]);
}

/* K:74-90  piecewise-linear RGBA lookup clamped at the ends. */
static inline void tf_sample(const double *table, long n, double lo, double hi, double v,
                             double *rgba) {
    double u = (v - lo) / (hi - lo) * (double)(n - 1);
    if (u <= 0.0) { memcpy(rgba, table, 4 * sizeof(double)); return; }
    if (u >= (double)(n - 1)) { memcpy(rgba, table + 4 * (n - 1), 4 * sizeof(double)); return; }
    long j = (long)floor(u);
    double f = u - (double)j;
    const double *a = table + 4 * j, *b = table + 4 * (j + 1);
    for (int c = 0; c < 4; ++c) rgba[c] = a[c] + f * (b[c] - a[c]);
}

void orc_tf_sample(const double *table, long n, double lo, double hi, double v, double *rgba) {
    tf_sample(table, n, lo, hi, v, rgba);
}

/* ------------------------------------------------------------ point location */

typedef struct {
    const double *nlo, *nhi;               /* (M,3) */
    const int64_t *left, *right, *start, *count, *prim;
} FlatBVH;

typedef struct {
    FlatBVH bvh;
    const int64_t *tets;                   /* (T,4) */
    const double *tet_orig;                /* (T,3) */
    const double *tet_inv;                 /* (T,3,3) */
    const double *field;                   /* (V,) or (T,) */
    int64_t centering;                     /* 0 vertex, 1 cell */
} MeshArgs;

/* K:93-136  lowest-index tet containing p via stack DFS of the tet BVH. */
static int64_t locate_point(double px, double py, double pz, const MeshArgs *m, double *bary) {
    const FlatBVH *B = &m->bvh;
    int64_t best = -1;
    double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
    int64_t stack[STACK];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        int64_t ni = stack[--sp];
        const double *lo = B->nlo + 3 * ni, *hi = B->nhi + 3 * ni;
        if (px < lo[0] || px > hi[0] || py < lo[1] || py > hi[1] || pz < lo[2] || pz > hi[2])
            continue;
        if (B->left[ni] < 0) {
            int64_t s = B->start[ni], e = s + B->count[ni];
            for (int64_t k = s; k < e; ++k) {
                int64_t t = B->prim[k];
                if (best >= 0 && t >= best) continue;
                const double *o = m->tet_orig + 3 * t, *A = m->tet_inv + 9 * t;
                double qx = px - o[0], qy = py - o[1], qz = pz - o[2];
                double l1 = A[0] * qx + A[1] * qy + A[2] * qz;
                double l2 = A[3] * qx + A[4] * qy + A[5] * qz;
                double l3 = A[6] * qx + A[7] * qy + A[8] * qz;
                double l0 = 1.0 - l1 - l2 - l3;
                if (l0 >= -BARY_TOL && l1 >= -BARY_TOL && l2 >= -BARY_TOL && l3 >= -BARY_TOL) {
                    best = t;
                    b0 = l0; b1 = l1; b2 = l2; b3 = l3;
                }
            }
        } else {
            stack[sp++] = B->left[ni];
            stack[sp++] = B->right[ni];
        }
    }
    bary[0] = b0; bary[1] = b1; bary[2] = b2; bary[3] = b3;
    return best;
}

/* K:139-154 */
static inline int field_at(double px, double py, double pz, const MeshArgs *m, double *val,
                           int64_t *tet_out) {
    double l[4];
    int64_t t = locate_point(px, py, pz, m, l);
    if (tet_out) *tet_out = t;
    if (t < 0) { *val = 0.0; return 0; }
    if (m->centering == 0) {
        const int64_t *tv = m->tets + 4 * t;
        *val = l[0] * m->field[tv[0]] + l[1] * m->field[tv[1]] + l[2] * m->field[tv[2]] +
               l[3] * m->field[tv[3]];
    } else {
        *val = m->field[t];
    }
    return 1;
}

#define MESH_PARAMS                                                                       \
    const double *m_nlo, const double *m_nhi, const int64_t *m_left, const int64_t *m_right, \
        const int64_t *m_start, const int64_t *m_count, const int64_t *m_prim,               \
        const int64_t *tets, const double *tet_orig, const double *tet_inv,                  \
        const double *field_vals, int64_t centering

#define MESH_INIT                                                                        \
    MeshArgs M = {{m_nlo, m_nhi, m_left, m_right, m_start, m_count, m_prim}, tets, tet_orig, \
                  tet_inv, field_vals, centering}

/* K:157-170 (batched point query); also reports the located tet id. */
void orc_field_at_many(int64_t n, const double *pts, MESH_PARAMS, uint8_t *found, double *vals,
                       int64_t *tet_ids, int threads) {
    MESH_INIT;
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads > 0 ? threads : 1)
    for (int64_t i = 0; i < n; ++i) {
        double v;
        int64_t t;
        int f = field_at(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], &M, &v, &t);
        found[i] = (uint8_t)f;
        vals[i] = v;
        if (tet_ids) tet_ids[i] = t;
    }
}

/* ----------------------------------------------------- partition traversal */

typedef struct {
    FlatBVH bvh;
    const double *p_lo, *p_hi;             /* (P,3) */
    const uint8_t *active;                 /* (P,) */
} PartArgs;

/* K:173-230  first active partition interval; lexicographic min (a_cl, pid). */
static int64_t next_interval(double ox, double oy, double oz, double dx, double dy, double dz,
                             double t_min, double t_max, double excl_eps, int64_t excl_id,
                             const PartArgs *P, double *ra, double *rb) {
    const FlatBVH *B = &P->bvh;
    int64_t best_id = -1;
    double best_a = INFINITY, best_b = INFINITY;
    int64_t stack[STACK];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        int64_t ni = stack[--sp];
        const double *lo = B->nlo + 3 * ni, *hi = B->nhi + 3 * ni;
        double a, b;
        slab(ox, oy, oz, dx, dy, dz, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], &a, &b);
        if (a > b) continue;
        if (b <= t_min + excl_eps) continue;
        double a_cl = (a > t_min) ? a : t_min;
        if (a_cl >= t_max) continue;
        if (a_cl > best_a) continue;
        if (B->left[ni] < 0) {
            int64_t s = B->start[ni], e = s + B->count[ni];
            for (int64_t k = s; k < e; ++k) {
                int64_t pid = B->prim[k];
                if (pid == excl_id || P->active[pid] == 0) continue;
                const double *pl = P->p_lo + 3 * pid, *ph = P->p_hi + 3 * pid;
                double pa, pb;
                slab(ox, oy, oz, dx, dy, dz, pl[0], pl[1], pl[2], ph[0], ph[1], ph[2], &pa, &pb);
                if (pa > pb) continue;
                if (pb <= t_min + excl_eps) continue;
                double pa_cl = (pa > t_min) ? pa : t_min;
                if (pa_cl >= t_max) continue;
                if (pa_cl < best_a || (pa_cl == best_a && pid < best_id)) {
                    best_id = pid;
                    best_a = pa_cl;
                    best_b = pb;
                }
            }
        } else {
            stack[sp++] = B->left[ni];
            stack[sp++] = B->right[ni];
        }
    }
    *ra = best_a; *rb = best_b;
    return best_id;
}

#define PART_PARAMS                                                                       \
    const double *b_nlo, const double *b_nhi, const int64_t *b_left, const int64_t *b_right, \
        const int64_t *b_start, const int64_t *b_count, const int64_t *b_prim,               \
        const double *p_lo, const double *p_hi, const uint8_t *active

#define PART_INIT \
    PartArgs PA = {{b_nlo, b_nhi, b_left, b_right, b_start, b_count, b_prim}, p_lo, p_hi, active}

int64_t orc_next_interval(const double *o, const double *d, double t_min, double t_max,
                          double excl_eps, int64_t excl_id, PART_PARAMS, double *out_ab) {
    PART_INIT;
    return next_interval(o[0], o[1], o[2], d[0], d[1], d[2], t_min, t_max, excl_eps, excl_id,
                         &PA, &out_ab[0], &out_ab[1]);
}

/* K:233-259 */
int64_t orc_trace_intervals(const double *o, const double *d, double t_min0, double t_max,
                            double eps, PART_PARAMS, int64_t max_out, int64_t *out_ids,
                            double *out_enter, double *out_exit) {
    PART_INIT;
    double t_min = t_min0;
    int64_t last = -1, n = 0;
    while (n < max_out) {
        double excl = (last < 0) ? 0.0 : eps;
        double a, b;
        int64_t pid = next_interval(o[0], o[1], o[2], d[0], d[1], d[2], t_min, t_max, excl,
                                    last, &PA, &a, &b);
        if (pid < 0) break;
        out_ids[n] = pid; out_enter[n] = a; out_exit[n] = b;
        ++n;
        t_min = b - eps;
        last = pid;
    }
    return n;
}

/* ------------------------------------------------------------------ march */

typedef struct {
    double r, g, b, a;
} Acc;

/* K:262-297  front-to-back compositing on [t0, t1) at t0 + (k + phase)*step. */
static int64_t march_range(double ox, double oy, double oz, double dx, double dy, double dz,
                           double t0, double t1, double step, double s1, double term,
                           double phase, const double *tf, long n_tf, double tf_lo,
                           double tf_hi, const MeshArgs *m, Acc *acc, int *terminated) {
    int64_t samples = 0;
    *terminated = 0;
    for (int64_t k = 0;; ++k) {
        double t = t0 + ((double)k + phase) * step;
        if (k > 0 && t >= t1) break;
        samples += 1;
        double v;
        if (field_at(ox + t * dx, oy + t * dy, oz + t * dz, m, &v, NULL)) {
            double c[4];
            tf_sample(tf, n_tf, tf_lo, tf_hi, v, c);
            double ca = orc_opacity_correction(c[3], step, s1);
            double w = (1.0 - acc->a) * ca;
            acc->r += w * c[0];
            acc->g += w * c[1];
            acc->b += w * c[2];
            acc->a += w;
            if (acc->a >= term) { *terminated = 1; break; }
        }
    }
    return samples;
}

int64_t orc_march_range(const double *o, const double *d, double t0, double t1, double step,
                        double s1, double term, double phase, const double *tf, long n_tf,
                        double tf_lo, double tf_hi, MESH_PARAMS, double *acc4,
                        int32_t *terminated) {
    MESH_INIT;
    Acc acc = {acc4[0], acc4[1], acc4[2], acc4[3]};
    int term_flag;
    int64_t n = march_range(o[0], o[1], o[2], d[0], d[1], d[2], t0, t1, step, s1, term, phase,
                            tf, n_tf, tf_lo, tf_hi, &M, &acc, &term_flag);
    acc4[0] = acc.r; acc4[1] = acc.g; acc4[2] = acc.b; acc4[3] = acc.a;
    *terminated = term_flag;
    return n;
}

/* K:300-309  numba types ix, iy as int64 and promotes every uint32 op to a
 * 64-bit integer, so the "uint32 wrap" of the comment never happens: the
 * arithmetic below is mod 2**64 (SURVEY.md section 7 "Hard parts"). */
double orc_hash01(int64_t ix, int64_t iy) {
    uint64_t h = ((uint64_t)(uint32_t)ix * 73856093ull) ^ ((uint64_t)(uint32_t)iy * 19349663ull);
    h = (h ^ 61ull) ^ (h >> 16);
    h = h * 9ull;
    h = h ^ (h >> 4);
    h = h * 0x27D4EB2Dull;
    h = h ^ (h >> 15);
    return (double)h / 4294967296.0;
}

/* ------------------------------------------------------------ render_frame */

/* K:312-398.  Rows [row_begin, row_end) only (row_end <= 0 means all rows),
 * so the CPU baseline can time a bounded row sample.  out_ppart is either
 * (H, P) per-row as in the reference or, when ppart_rows == 1, a single
 * (1, P) row accumulated with one private row per thread. */
void orc_render_frame(const double *cam_pos, const double *cam_right, const double *cam_up,
                      const double *cam_fwd, double tan_half, double aspect, int64_t width,
                      int64_t height, int32_t jitter, int32_t mode, double s1, double s2,
                      double p_pow, double term, double eps, const double *bg,
                      const double *tf_table, int64_t n_tf, double tf_lo, double tf_hi,
                      const double *mesh_lo, const double *mesh_hi, PART_PARAMS,
                      const double *sigma, MESH_PARAMS, double *out_rgba, int64_t *out_samples,
                      int32_t *out_visited, int64_t *out_ppart, int64_t n_parts,
                      int32_t track_ppart, int32_t ppart_rows, int64_t row_begin,
                      int64_t row_end, int threads) {
    MESH_INIT;
    PART_INIT;
    if (row_end <= 0 || row_end > height) row_end = height;
    if (row_begin < 0) row_begin = 0;
    int nthr = threads > 0 ? threads : 1;
    int64_t *priv = NULL;
    if (track_ppart && ppart_rows == 1) priv = calloc((size_t)nthr * (size_t)n_parts, 8);

#pragma omp parallel num_threads(nthr)
    {
#ifdef _OPENMP
        int tid = omp_get_thread_num();
#else
        int tid = 0;
#endif
#pragma omp for schedule(dynamic, 1)
        for (int64_t iy = row_begin; iy < row_end; ++iy) {
            int64_t *prow = NULL;
            if (track_ppart) prow = priv ? priv + (size_t)tid * n_parts : out_ppart + iy * n_parts;
            for (int64_t ix = 0; ix < width; ++ix) {
                double sx = (((double)ix + 0.5) / (double)width) * 2.0 - 1.0;
                double sy = 1.0 - (((double)iy + 0.5) / (double)height) * 2.0;
                double dx = cam_fwd[0] + sx * aspect * tan_half * cam_right[0] + sy * tan_half * cam_up[0];
                double dy = cam_fwd[1] + sx * aspect * tan_half * cam_right[1] + sy * tan_half * cam_up[1];
                double dz = cam_fwd[2] + sx * aspect * tan_half * cam_right[2] + sy * tan_half * cam_up[2];
                double dn = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
                dx *= dn; dy *= dn; dz *= dn;
                double ox = cam_pos[0], oy = cam_pos[1], oz = cam_pos[2];
                double phase = jitter ? orc_hash01(ix, iy) : 0.5;
                Acc acc = {0.0, 0.0, 0.0, 0.0};
                int64_t samples = 0;
                int32_t visited = 0;
                int term_flag;
                if (mode == 0) {
                    double a, b;
                    slab(ox, oy, oz, dx, dy, dz, mesh_lo[0], mesh_lo[1], mesh_lo[2], mesh_hi[0],
                         mesh_hi[1], mesh_hi[2], &a, &b);
                    double t0 = (a > 0.0) ? a : 0.0;
                    if (a <= b && b - t0 >= eps)
                        samples = march_range(ox, oy, oz, dx, dy, dz, t0, b, s1, s1, term, phase,
                                              tf_table, n_tf, tf_lo, tf_hi, &M, &acc, &term_flag);
                } else {
                    double t_min = 0.0;
                    int64_t last = -1;
                    for (;;) {
                        double excl = (last < 0) ? 0.0 : eps;
                        double a, b;
                        int64_t pid = next_interval(ox, oy, oz, dx, dy, dz, t_min, INFINITY, excl,
                                                    last, &PA, &a, &b);
                        if (pid < 0) break;
                        visited += 1;
                        term_flag = 0;
                        if (b - a >= eps) {
                            double s = (mode == 2) ? orc_step_size(s1, s2, p_pow, sigma[pid]) : s1;
                            int64_t ns = march_range(ox, oy, oz, dx, dy, dz, a, b, s, s1, term,
                                                     phase, tf_table, n_tf, tf_lo, tf_hi, &M, &acc,
                                                     &term_flag);
                            samples += ns;
                            if (track_ppart) prow[pid] += ns;
                        }
                        if (term_flag) break;
                        t_min = b - eps;
                        last = pid;
                    }
                }
                double *px = out_rgba + 4 * (iy * width + ix);
                px[0] = acc.r + (1.0 - acc.a) * bg[0];
                px[1] = acc.g + (1.0 - acc.a) * bg[1];
                px[2] = acc.b + (1.0 - acc.a) * bg[2];
                px[3] = acc.a + (1.0 - acc.a) * bg[3];
                out_samples[iy * width + ix] = samples;
                out_visited[iy * width + ix] = visited;
            }
        }
    }
    if (priv) {
        for (int t = 0; t < nthr; ++t)
            for (int64_t p = 0; p < n_parts; ++p) out_ppart[p] += priv[(size_t)t * n_parts + p];
        free(priv);
    }
}

/* -------------------------------------------------------------- BVH build */

/* Stable merge sort of idx[0..n) by key[idx] (numpy argsort kind="stable"). */
static void stable_sort_by_key(int64_t *idx, int64_t n, const double *key, int64_t *tmp) {
    if (n < 2) return;
    if (n <= 16) { /* insertion sort is stable */
        for (int64_t i = 1; i < n; ++i) {
            int64_t v = idx[i];
            double kv = key[v];
            int64_t j = i - 1;
            while (j >= 0 && key[idx[j]] > kv) { idx[j + 1] = idx[j]; --j; }
            idx[j + 1] = v;
        }
        return;
    }
    int64_t h = n / 2;
    stable_sort_by_key(idx, h, key, tmp);
    stable_sort_by_key(idx + h, n - h, key, tmp);
    int64_t i = 0, j = h, k = 0;
    while (i < h && j < n) tmp[k++] = (key[idx[j]] < key[idx[i]]) ? idx[j++] : idx[i++];
    while (i < h) tmp[k++] = idx[i++];
    while (j < n) tmp[k++] = idx[j++];
    memcpy(idx, tmp, (size_t)n * sizeof(int64_t));
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* bvh.py:41-98  median split on the longest node axis by stable centroid
 * order; leaves of <= leaf_size primitives sorted by id; nodes numbered in
 * the reference's order (children allocated left, right; DFS pops left
 * first).  Returns the node count (<= 2n).  Output arrays must hold 2n
 * nodes; prim must hold n. */
int64_t orc_build_bvh(int64_t n, const double *box_lo, const double *box_hi, int64_t leaf_size,
                      double *nlo, double *nhi, int64_t *left, int64_t *right, int64_t *start,
                      int64_t *count, int64_t *prim) {
    if (n <= 0) return 0;
    double *cen = malloc((size_t)n * 3 * sizeof(double));
    double *key = malloc((size_t)n * sizeof(double));
    int64_t *tmp = malloc((size_t)n * sizeof(int64_t));
    int64_t *stk = malloc((size_t)(2 * n + 8) * 3 * sizeof(int64_t));
    for (int64_t i = 0; i < 3 * n; ++i) cen[i] = 0.5 * (box_lo[i] + box_hi[i]);
    for (int64_t i = 0; i < n; ++i) prim[i] = i;
    int64_t n_nodes = 1, sp = 0;
    left[0] = right[0] = -1; start[0] = count[0] = 0;
    stk[0] = 0; stk[1] = 0; stk[2] = n; sp = 1;
    while (sp > 0) {
        --sp;
        int64_t ni = stk[3 * sp], lo_i = stk[3 * sp + 1], hi_i = stk[3 * sp + 2];
        double bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t k = lo_i; k < hi_i; ++k) {
            int64_t id = prim[k];
            for (int a = 0; a < 3; ++a) {
                double l = box_lo[3 * id + a], h = box_hi[3 * id + a];
                if (l < bl[a]) bl[a] = l;
                if (h > bh[a]) bh[a] = h;
            }
        }
        memcpy(nlo + 3 * ni, bl, sizeof bl);
        memcpy(nhi + 3 * ni, bh, sizeof bh);
        int64_t m = hi_i - lo_i;
        if (m <= leaf_size) {
            start[ni] = lo_i; count[ni] = m;
            qsort(prim + lo_i, (size_t)m, sizeof(int64_t), cmp_i64);
            continue;
        }
        /* np.argmax: first maximal extent */
        double ext0 = bh[0] - bl[0], ext1 = bh[1] - bl[1], ext2 = bh[2] - bl[2];
        int axis = 0;
        double best = ext0;
        if (ext1 > best) { axis = 1; best = ext1; }
        if (ext2 > best) { axis = 2; }
        for (int64_t k = lo_i; k < hi_i; ++k) key[prim[k]] = cen[3 * prim[k] + axis];
        stable_sort_by_key(prim + lo_i, m, key, tmp);
        int64_t mid = lo_i + m / 2;
        int64_t li = n_nodes++, ri = n_nodes++;
        left[li] = right[li] = -1; start[li] = count[li] = 0;
        left[ri] = right[ri] = -1; start[ri] = count[ri] = 0;
        left[ni] = li; right[ni] = ri;
        stk[3 * sp] = ri; stk[3 * sp + 1] = mid; stk[3 * sp + 2] = hi_i; ++sp;
        stk[3 * sp] = li; stk[3 * sp + 1] = lo_i; stk[3 * sp + 2] = mid; ++sp;
    }
    free(cen); free(key); free(tmp); free(stk);
    return n_nodes;
}
