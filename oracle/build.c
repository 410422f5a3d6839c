/*
 * build.c -- CPU restatement of the reference's SCENE BUILD (TEST INFRASTRUCTURE).
 *
 * Like oracle.c this is the parity oracle, not the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * load it.  It exists so that the oracle and the reference arm can construct
 * BASELINE config 3-4 scenes (1e8 tets) in seconds without the product
 * library (libtetray_b200.so) and without the reference's Python builders,
 * which need ~40 min for radial272.
 *
 * Restated, with the reference lines they follow:
 *   orc_gen_grid       mesh.py:198-231  generate_synthetic (radial / ramp, vertex-centered),
 *                      plus the per-tet (parity, pattern) index the Python side
 *                      uses to invert the 10 distinct edge matrices (mesh.py:251-254)
 *   orc_tet_boxes      mesh.py:104-106  tet_aabbs, mesh.py:248-250 padding
 *   orc_kd_build       partitions.py:47-128  build_partitions (median-of-centroids
 *                      KD split, straddlers duplicated, flat elements to the right,
 *                      no-progress / empty-side leaves, refined bounds, value ranges)
 *   orc_build_bvh_fast bvh.py:41-98  build_bvh, the same tree as oracle.c's
 *                      orc_build_bvh (node ids, prim order) built with OpenMP tasks
 *
 * Arithmetic follows numpy exactly: centroids (((v0+v1)+v2)+v3)/4 (mean over
 * axis 1, sequential), np.median = the middle element or fl(fl(a+b)/2), the
 * radial field = f32(sqrt((dx*dx + dy*dy) + dz*dz)).  Pinned against the
 * reference's own scene-array hashes (tests/golden/reference_frames.json,
 * reference_big.json; tests/test_oracle_build.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------ generator */

/* mesh.py:163-173: corner index = 4x + 2y + z; the 5-tet patterns of an even
 * cube and their x-mirror for odd cubes. */
static const int PATTERN_EVEN[5][4] = {
    {0, 4, 2, 1}, {6, 2, 4, 7}, {5, 1, 7, 4}, {3, 7, 1, 2}, {4, 2, 1, 7}};

static int flip_x(int c) { return c ^ 4; }

/* mesh.py:198-231 for field kind 0 = ramp (x), 1 = radial (|p - n/2|),
 * vertex-centered.  verts (g^3, 3), tets (5 n^3, 4), field (g^3),
 * pattern (5 n^3): parity * 5 + k. */
int orc_gen_grid(int64_t n, int field_kind, double *verts, int64_t *tets, double *field,
                 uint8_t *pattern) {
    if (n < 1 || (field_kind != 0 && field_kind != 1)) return -1;
    const int64_t g = n + 1;
    const double half = (double)n / 2.0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g; ++i)
        for (int64_t j = 0; j < g; ++j)
            for (int64_t k = 0; k < g; ++k) {
                int64_t v = (i * g + j) * g + k;
                double x = (double)i, y = (double)j, z = (double)k;
                verts[3 * v] = x; verts[3 * v + 1] = y; verts[3 * v + 2] = z;
                double f;
                if (field_kind == 0) {
                    f = x;
                } else {
                    double dx = x - half, dy = y - half, dz = z - half;
                    f = sqrt((dx * dx + dy * dy) + dz * dz);
                }
                field[v] = (double)(float)f;
            }
#pragma omp parallel for schedule(static)
    for (int64_t ci = 0; ci < n; ++ci)
        for (int64_t cj = 0; cj < n; ++cj)
            for (int64_t ck = 0; ck < n; ++ck) {
                int64_t cell = (ci * n + cj) * n + ck;
                int parity = (int)((ci + cj + ck) % 2);
                int64_t corner[8];
                for (int x = 0; x < 2; ++x)
                    for (int y = 0; y < 2; ++y)
                        for (int z = 0; z < 2; ++z)
                            corner[4 * x + 2 * y + z] = ((ci + x) * g + (cj + y)) * g + (ck + z);
                for (int t = 0; t < 5; ++t) {
                    int64_t tid = cell * 5 + t;
                    for (int q = 0; q < 4; ++q) {
                        int c = PATTERN_EVEN[t][q];
                        tets[4 * tid + q] = corner[parity ? flip_x(c) : c];
                    }
                    pattern[tid] = (uint8_t)(parity * 5 + t);
                }
            }
    return 0;
}

/* mesh.py:104-106 tet_aabbs (min/max over the 4 vertices); pad > 0 adds
 * mesh.py:249-250's padding (lo - pad, hi + pad). */
void orc_tet_boxes(int64_t n_tets, const double *verts, const int64_t *tets, double pad,
                   double *lo, double *hi) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_tets; ++t)
        for (int a = 0; a < 3; ++a) {
            double l = verts[3 * tets[4 * t] + a], h = l;
            for (int q = 1; q < 4; ++q) {
                double v = verts[3 * tets[4 * t + q] + a];
                if (v < l) l = v;
                if (v > h) h = v;
            }
            if (pad > 0.0) { l = l - pad; h = h + pad; }
            lo[3 * t + a] = l;
            hi[3 * t + a] = h;
        }
}

/* ----------------------------------------------------------- KD build */

typedef struct {
    const double *verts;
    const int64_t *tets;
    const double *field;
    int centering; /* 0 vertex, 1 cell */
    const double *box_lo, *box_hi;
    double *cen; /* (T,3) */
    int64_t max_leaf, max_depth;
} KdCtx;

typedef struct KdNode {
    struct KdNode *left, *right;   /* NULL for a leaf */
    int64_t *ids;                  /* leaf: sorted element ids */
    int64_t n;
    double lo[3], hi[3];           /* leaf: refined bounds */
    double vmin, vmax;
} KdNode;

static void swapd(double *a, double *b) { double t = *a; *a = *b; *b = t; }

/* k-th smallest of v[0..n) (v is permuted); 3-way partition quickselect. */
static double select_kth(double *v, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n - 1;
    uint64_t seed = 0x9e3779b97f4a7c15ull ^ (uint64_t)n;
    while (lo < hi) {
        seed = seed * 6364136223846793005ull + 1442695040888963407ull;
        double p = v[lo + (int64_t)((seed >> 33) % (uint64_t)(hi - lo + 1))];
        int64_t lt = lo, i = lo, gt = hi;
        while (i <= gt) {
            if (v[i] < p) swapd(&v[lt++], &v[i++]);
            else if (v[i] > p) swapd(&v[i], &v[gt--]);
            else ++i;
        }
        if (k < lt) hi = lt - 1;
        else if (k > gt) lo = gt + 1;
        else return p;
    }
    return v[k];
}

/* np.median (numpy/lib/_function_base_impl.py _median): odd n -> the middle
 * element; even n -> mean of the two middle elements = fl(fl(a+b)/2). */
static double np_median(double *v, int64_t n) {
    int64_t h = n / 2;
    if (n % 2 == 1) return select_kth(v, n, h);
    double b = select_kth(v, n, h);
    /* after selecting h, v[0..h) holds the h smallest; their max is a */
    double a = v[0];
    for (int64_t i = 1; i < h; ++i)
        if (v[i] > a) a = v[i];
    return (a + b) / 2.0;
}

static int cmp_i64k(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* partitions.py:82-93 emit + refine_partition_bounds (partitions.py:60-70). */
static void kd_emit(const KdCtx *c, KdNode *nd, int64_t *ids, int64_t n, const double *nlo,
                    const double *nhi) {
    int sorted = 1;
    for (int64_t i = 1; i < n && sorted; ++i) sorted = ids[i - 1] < ids[i];
    if (!sorted) qsort(ids, (size_t)n, sizeof(int64_t), cmp_i64k);
    double vmin = INFINITY, vmax = -INFINITY;
    double plo[3] = {INFINITY, INFINITY, INFINITY}, phi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = ids[i];
        double emin, emax;
        if (c->centering == 0) { /* element_value_ranges: min/max of the 4 vertex values */
            emin = emax = c->field[c->tets[4 * t]];
            for (int q = 1; q < 4; ++q) {
                double f = c->field[c->tets[4 * t + q]];
                if (f < emin) emin = f;
                if (f > emax) emax = f;
            }
        } else {
            emin = emax = c->field[t];
        }
        if (emin < vmin) vmin = emin;
        if (emax > vmax) vmax = emax;
        for (int q = 0; q < 4; ++q)
            for (int a = 0; a < 3; ++a) {
                double x = c->verts[3 * c->tets[4 * t + q] + a];
                if (x < plo[a]) plo[a] = x;
                if (x > phi[a]) phi[a] = x;
            }
    }
    for (int a = 0; a < 3; ++a) { /* AABB.intersection: max of lows, min of highs */
        nd->lo[a] = plo[a] > nlo[a] ? plo[a] : nlo[a];
        nd->hi[a] = phi[a] < nhi[a] ? phi[a] : nhi[a];
    }
    nd->vmin = vmin;
    nd->vmax = vmax;
    nd->ids = ids;
    nd->n = n;
    nd->left = nd->right = NULL;
}

/* partitions.py:95-121 split(ids, node_lo, node_hi, depth).  Takes ownership
 * of `ids` (malloc'ed). */
static void kd_split(const KdCtx *c, KdNode *nd, int64_t *ids, int64_t n, const double *nlo,
                     const double *nhi, int64_t depth) {
    if (n <= c->max_leaf || depth >= c->max_depth) {
        kd_emit(c, nd, ids, n, nlo, nhi);
        return;
    }
    double ext0 = nhi[0] - nlo[0], ext1 = nhi[1] - nlo[1], ext2 = nhi[2] - nlo[2];
    int axis = 0; /* np.argmax: first maximum */
    double best = ext0;
    if (ext1 > best) { axis = 1; best = ext1; }
    if (ext2 > best) axis = 2;
    double *vals = malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) vals[i] = c->cen[3 * ids[i] + axis];
    double m = np_median(vals, n);
    free(vals);
    int64_t nl = 0, nr = 0, ne = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = ids[i];
        int l = c->box_lo[3 * t + axis] < m, r = c->box_hi[3 * t + axis] > m;
        nl += l;
        nr += r;
        ne += (!l && !r);
    }
    /* right = ids[hi > m] then the uncovered (flat-on-plane) ids, sorted
     * (np.setdiff1d); the order inside a side never matters: medians are
     * order-free and leaves are sorted */
    if ((nl == n && nr + ne == n) || nl == 0 || nr + ne == 0) {
        kd_emit(c, nd, ids, n, nlo, nhi);
        return;
    }
    int64_t *L = malloc((size_t)(nl > 0 ? nl : 1) * sizeof(int64_t));
    int64_t *R = malloc((size_t)(nr + ne > 0 ? nr + ne : 1) * sizeof(int64_t));
    int64_t il = 0, ir = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = ids[i];
        int l = c->box_lo[3 * t + axis] < m, r = c->box_hi[3 * t + axis] > m;
        if (l) L[il++] = t;
        if (r || !l) R[ir++] = t;
    }
    free(ids);
    double lhi[3] = {nhi[0], nhi[1], nhi[2]}, rlo[3] = {nlo[0], nlo[1], nlo[2]};
    lhi[axis] = m;
    rlo[axis] = m;
    nd->left = calloc(1, sizeof(KdNode));
    nd->right = calloc(1, sizeof(KdNode));
    nd->ids = NULL;
    nd->n = 0;
    KdNode *ln = nd->left, *rn = nd->right;
#pragma omp task if (nl > 200000) firstprivate(ln, L, nl, depth)
    kd_split(c, ln, L, nl, nlo, lhi, depth + 1);
#pragma omp task if (ir > 200000) firstprivate(rn, R, ir, depth)
    kd_split(c, rn, R, ir, rlo, nhi, depth + 1);
#pragma omp taskwait
}

typedef struct {
    int64_t n_parts, n_ids;
    KdNode *root;
} KdResult;

static void kd_count(KdNode *nd, int64_t *np, int64_t *ni) {
    if (!nd->left) { ++*np; *ni += nd->n; return; }
    kd_count(nd->left, np, ni);
    kd_count(nd->right, np, ni);
}

static void kd_collect(KdNode *nd, int64_t *p, int64_t *off, int64_t *offsets, int64_t *ids,
                       double *lo, double *hi, double *vrange) {
    if (nd->left) {
        kd_collect(nd->left, p, off, offsets, ids, lo, hi, vrange);
        kd_collect(nd->right, p, off, offsets, ids, lo, hi, vrange);
        free(nd->left);
        free(nd->right);
        return;
    }
    int64_t k = (*p)++;
    offsets[k] = *off;
    memcpy(ids + *off, nd->ids, (size_t)nd->n * sizeof(int64_t));
    *off += nd->n;
    offsets[k + 1] = *off;
    memcpy(lo + 3 * k, nd->lo, sizeof nd->lo);
    memcpy(hi + 3 * k, nd->hi, sizeof nd->hi);
    vrange[2 * k] = nd->vmin;
    vrange[2 * k + 1] = nd->vmax;
    free(nd->ids);
}

/* Phase 1: build the KD tree; returns an opaque handle and the partition /
 * id counts.  Phase 2 (orc_kd_take) copies the leaves out in left-first DFS
 * order (partitions.py:82-84, ids = len(partitions) at emit) and frees it. */
void *orc_kd_build(int64_t n_tets, const double *verts, const int64_t *tets, const double *field,
                   int centering, int64_t max_leaf, int64_t max_depth, const double *mesh_lo,
                   const double *mesh_hi, int64_t *n_parts, int64_t *n_ids) {
    KdCtx *c = calloc(1, sizeof(KdCtx));
    c->verts = verts; c->tets = tets; c->field = field; c->centering = centering;
    c->max_leaf = max_leaf; c->max_depth = max_depth;
    double *blo = malloc((size_t)n_tets * 3 * sizeof(double));
    double *bhi = malloc((size_t)n_tets * 3 * sizeof(double));
    orc_tet_boxes(n_tets, verts, tets, 0.0, blo, bhi);
    c->box_lo = blo; c->box_hi = bhi;
    c->cen = malloc((size_t)n_tets * 3 * sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_tets; ++t)
        for (int a = 0; a < 3; ++a) {
            double s = verts[3 * tets[4 * t] + a];
            for (int q = 1; q < 4; ++q) s = s + verts[3 * tets[4 * t + q] + a];
            c->cen[3 * t + a] = s / 4.0;
        }
    int64_t *ids = malloc((size_t)n_tets * sizeof(int64_t));
    for (int64_t i = 0; i < n_tets; ++i) ids[i] = i;
    KdResult *res = calloc(1, sizeof(KdResult));
    res->root = calloc(1, sizeof(KdNode));
#pragma omp parallel
#pragma omp single
    kd_split(c, res->root, ids, n_tets, mesh_lo, mesh_hi, 0);
    free(blo); free(bhi); free(c->cen); free(c);
    kd_count(res->root, &res->n_parts, &res->n_ids);
    *n_parts = res->n_parts;
    *n_ids = res->n_ids;
    return res;
}

void orc_kd_take(void *h, int64_t *offsets, int64_t *ids, double *lo, double *hi,
                 double *vrange) {
    KdResult *res = h;
    int64_t p = 0, off = 0;
    kd_collect(res->root, &p, &off, offsets, ids, lo, hi, vrange);
    free(res->root);
    free(res);
}

/* ---------------------------------------------------------- BVH build */

/* Order-preserving map of a double to u64 (no NaNs in box centroids). */
static inline uint64_t dkey(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

/* Stable LSD radix sort of idx[0..n) by key[idx]: the order of
 * np.argsort(kind="stable") (bvh.py:87).  Passes whose digit is constant
 * over the range are skipped. */
static void radix_stable(int64_t *idx, int64_t n, const uint64_t *key, int64_t *tmp) {
    if (n < 2) return;
    if (n <= 32) {
        for (int64_t i = 1; i < n; ++i) {
            int64_t v = idx[i];
            uint64_t kv = key[v];
            int64_t j = i - 1;
            while (j >= 0 && key[idx[j]] > kv) { idx[j + 1] = idx[j]; --j; }
            idx[j + 1] = v;
        }
        return;
    }
    uint64_t kmin = UINT64_MAX, kmax = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t k = key[idx[i]];
        if (k < kmin) kmin = k;
        if (k > kmax) kmax = k;
    }
    uint64_t range = kmax - kmin;
    int64_t *src = idx, *dst = tmp;
    enum { B = 11 };
    int64_t cnt[1 << B];
    for (int shift = 0; shift < 64 && (range >> shift) != 0; shift += B) {
        memset(cnt, 0, sizeof cnt);
        for (int64_t i = 0; i < n; ++i) cnt[((key[src[i]] - kmin) >> shift) & ((1 << B) - 1)]++;
        int single = 0;
        for (int d = 0; d < (1 << B); ++d) single |= (cnt[d] == n);
        if (single) continue; /* constant digit: the pass would not move anything */
        int64_t s = 0;
        for (int d = 0; d < (1 << B); ++d) { int64_t c = cnt[d]; cnt[d] = s; s += c; }
        for (int64_t i = 0; i < n; ++i)
            dst[cnt[((key[src[i]] - kmin) >> shift) & ((1 << B) - 1)]++] = src[i];
        int64_t *t = src; src = dst; dst = t;
    }
    if (src != idx) memcpy(idx, src, (size_t)n * sizeof(int64_t));
}


/* Nodes of the subtree over m primitives: the tree shape depends only on m
 * (split at m // 2, leaf iff m <= leaf_size).  Every size in the tree is
 * floor or ceil of n / 2^d, so the table holds at most 2 per level. */
#define NODE_TAB 160
typedef struct { int64_t m[NODE_TAB], nodes[NODE_TAB]; int k; } NodeTab;

static int64_t tab_get(const NodeTab *t, int64_t m) {
    for (int i = 0; i < t->k; ++i)
        if (t->m[i] == m) return t->nodes[i];
    abort();
}

static int64_t tab_fill(NodeTab *t, int64_t m, int64_t leaf) {
    for (int i = 0; i < t->k; ++i)
        if (t->m[i] == m) return t->nodes[i];
    int64_t r = (m <= leaf) ? 1 : 1 + tab_fill(t, m / 2, leaf) + tab_fill(t, m - m / 2, leaf);
    if (t->k >= NODE_TAB) abort();
    t->m[t->k] = m;
    t->nodes[t->k++] = r;
    return r;
}

typedef struct {
    const double *box_lo, *box_hi;
    uint64_t *key[3];
    int64_t leaf;
    double *nlo, *nhi;
    int64_t *left, *right, *start, *count, *prim, *tmp;
    const NodeTab *tab;
} BvhCtx;

static int cmp_i64b(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* bvh.py:72-93 for node ni over prim[lo_i, hi_i); `next` is the id the
 * reference's counter holds when ni is popped (children get next, next+1;
 * the left subtree is finished before the right one is popped). */
static void bvh_node(const BvhCtx *c, int64_t ni, int64_t lo_i, int64_t hi_i, int64_t next) {
    double bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t k = lo_i; k < hi_i; ++k) {
        int64_t id = c->prim[k];
        for (int a = 0; a < 3; ++a) {
            double l = c->box_lo[3 * id + a], h = c->box_hi[3 * id + a];
            if (l < bl[a]) bl[a] = l;
            if (h > bh[a]) bh[a] = h;
        }
    }
    memcpy(c->nlo + 3 * ni, bl, sizeof bl);
    memcpy(c->nhi + 3 * ni, bh, sizeof bh);
    int64_t m = hi_i - lo_i;
    c->left[ni] = c->right[ni] = -1;
    if (m <= c->leaf) {
        c->start[ni] = lo_i;
        c->count[ni] = m;
        qsort(c->prim + lo_i, (size_t)m, sizeof(int64_t), cmp_i64b);
        return;
    }
    c->start[ni] = c->count[ni] = 0;
    double ext0 = bh[0] - bl[0], ext1 = bh[1] - bl[1], ext2 = bh[2] - bl[2];
    int axis = 0;
    double best = ext0;
    if (ext1 > best) { axis = 1; best = ext1; }
    if (ext2 > best) axis = 2;
    radix_stable(c->prim + lo_i, m, c->key[axis], c->tmp + lo_i);
    int64_t mid = lo_i + m / 2;
    int64_t li = next, ri = next + 1;
    c->left[ni] = li;
    c->right[ni] = ri;
    int64_t rnext = next + 2 + tab_get(c->tab, mid - lo_i) - 1;
#pragma omp task if (m > 100000) firstprivate(li, lo_i, mid, next)
    bvh_node(c, li, lo_i, mid, next + 2);
#pragma omp task if (m > 100000) firstprivate(ri, mid, hi_i, rnext)
    bvh_node(c, ri, mid, hi_i, rnext);
#pragma omp taskwait
}

/* bvh.py:41-98, same outputs as orc_build_bvh (oracle.c). */
int64_t orc_build_bvh_fast(int64_t n, const double *box_lo, const double *box_hi,
                           int64_t leaf_size, double *nlo, double *nhi, int64_t *left,
                           int64_t *right, int64_t *start, int64_t *count, int64_t *prim) {
    if (n <= 0) return 0;
    NodeTab tab = {{0}, {0}, 0};
    int64_t total = tab_fill(&tab, n, leaf_size);
    BvhCtx c = {box_lo, box_hi, {NULL, NULL, NULL}, leaf_size, nlo, nhi, left, right, start,
                count, prim, NULL, &tab};
    for (int a = 0; a < 3; ++a) c.key[a] = malloc((size_t)n * sizeof(uint64_t));
    c.tmp = malloc((size_t)n * sizeof(int64_t));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a)
            c.key[a][i] = dkey(0.5 * (box_lo[3 * i + a] + box_hi[3 * i + a])); /* bvh.py:70 */
        prim[i] = i;
    }
#pragma omp parallel
#pragma omp single
    bvh_node(&c, 0, 0, n, 1);
    for (int a = 0; a < 3; ++a) free(c.key[a]);
    free(c.tmp);
    return total;
}
