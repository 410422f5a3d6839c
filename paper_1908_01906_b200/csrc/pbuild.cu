// pbuild.cu -- device build of the point-location structures of an ARBITRARY
// mesh ("Morton/LBVH point-location tree").
//
// The reference builds MeshSampler's tet BVH on the host (mesh.py:246-254,
// bvh.py:41-98: median split, padded boxes) and locates points with a
// lowest-index DFS (K:93-136).  Any conservative structure gives the same
// answer, so the device builds the same STRUCTURE TYPES the host
// builder (host_build.cpp tr_pbvh_build / tr_cells_build) writes and the march
// consumes, in HBM, from the mesh arrays uploaded once:
//   1. padded tet boxes (mesh.py:248-250: min/max of the 4 vertices -/+ pad);
//   2. 60-bit Morton codes of the box centres (20 bits per axis over the
//      centres' bounding box) and a radix sort of (code, tet id) -- stable,
//      so equal codes keep ascending ids; equal codes form one cluster (the
//      5 tets of a generator cube share their box, so they never split);
//   3. Karras' binary radix tree over the unique codes (one thread per
//      internal node: direction, range and split from common-prefix lengths);
//   4. every radix-tree node holding more than leaf_max tets is kept as a BVH2
//      node; its children with at most leaf_max tets (or a single cluster)
//      are leaves.  Nodes and leaves are renumbered by prefix sums (root = 0;
//      leaves in code order, so a leaf's tets are consecutive records); ids
//      inside a leaf are sorted ascending (the lowest-index-first scan);
//   5. bottom-up refit (one thread per leaf, the second arrival at a node
//      continues): exact f64 unions, child boxes rounded outward to f32,
//      subtree minimum ids (descent pruning, K:119);
//   6. exclusive box per leaf: its box minus greedy axis cuts against every
//      other leaf box that meets it (host p_exclusive_boxes), rounded inward;
//   7. the uniform leaf grid (host p_build_grid: dims, origin, scale by the
//      same expressions; each cell names the leaf whose exclusive box covers
//      most of it -- a 64-bit atomicMax of (f32 overlap, leaf)) and coverage;
//   8. when coverage is low (unstructured meshes), the cell candidate lists
//      (host tr_cells_build): counts, prefix sum, fill, per-cell sort by tet id,
//      overflow bit, f32 record boxes.
//   9. (tr_dpb_walk, below) the leaf walk tables: neighbours, start,
//      predictors and certificates proved with orientation-determinant error
//      bounds.  Without it leaves carry walk = 0, which the march reads as
//      "scan the leaf in id order".
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "tetray_b200.h"
#include "tr_internal.h"

struct TrDevPointBuild {
    cudaStream_t st = nullptr;
    int64_t n_tets = 0, n_nodes = 0, n_leaves = 0, n_grid = 0, n_ccells = 0, n_crecs = 0;
    int32_t gdim[3] = {1, 1, 1}, cdim[3] = {1, 1, 1};
    double gorg[3] = {0, 0, 0}, gscale[3] = {1, 1, 1}, corg[3] = {0, 0, 0}, cscale[3] = {1, 1, 1};
    double coverage = 0.0;
    TrPNode *nodes = nullptr;
    TrPLeaf *leaves = nullptr;
    uint32_t *ids = nullptr;
    int32_t *grid = nullptr;
    uint32_t *coff = nullptr, *crecs = nullptr;
    float *tbox = nullptr;
    TrLeafPred *pred = nullptr;   // tr_dpb_walk: walk-start predictor per leaf
};

namespace {

__device__ __forceinline__ int64_t clampi(int64_t v, int64_t hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

constexpr int32_t CHILD_NONE = INT32_MIN;
constexpr int EX_STACK = 64;
constexpr int MORTON_BITS = 20;   // per axis: 60-bit codes, radix-tree depth <= 60 < PSTACK

int cuda_fail(cudaError_t e, const char *where) {
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    return tr_fail(TR_ECUDA, m.c_str());
}

unsigned grid_for(int64_t items) {
    int64_t g = (items + 255) / 256;
    if (g > 148 * 64) g = 148 * 64;
    return (unsigned)(g < 1 ? 1 : g);
}

#define GRID_STRIDE(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
                               i += (int64_t)gridDim.x * blockDim.x)

// order-preserving u64 image of a double (atomic min/max of doubles)
__device__ __forceinline__ unsigned long long ord(double x) {
    unsigned long long u = (unsigned long long)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double unord(unsigned long long u) {
    u = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double d;
    memcpy(&d, &u, 8);
    return d;
#endif
}

// Block-wide min/max of 6 values (lo x,y,z as min, hi x,y,z as max) folded
// into bounds[6] (ordered u64) with one atomic per block.
__device__ void bounds_fold(double v[6], unsigned long long *bounds) {
    __shared__ unsigned long long sh[8][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < 6; ++a) {
        double x = v[a];
        for (int o = 16; o > 0; o >>= 1) {
            double y = __shfl_xor_sync(0xffffffffu, x, o);
            x = a < 3 ? fmin(x, y) : fmax(x, y);
        }
        if (lane == 0) sh[w][a] = ord(x);
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        const int a = threadIdx.x;
        unsigned long long r = sh[0][a];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = a < 3 ? min(r, sh[k][a]) : max(r, sh[k][a]);
        if (a < 3) atomicMin(bounds + a, r); else atomicMax(bounds + a, r);
    }
}

// 1. padded boxes (tr_tet_boxes' expressions) and the bounds of their centres
__global__ void __launch_bounds__(256) boxes_kernel(int64_t T, const double *__restrict__ V,
                                                    const int64_t *__restrict__ tets, double pad,
                                                    double *__restrict__ box,
                                                    unsigned long long *cbounds) {
    double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    GRID_STRIDE(t, T) {
        const int64_t *tv = tets + 4 * t;
        const int64_t i0 = tv[0], i1 = tv[1], i2 = tv[2], i3 = tv[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double v0 = V[3 * i0 + a], v1 = V[3 * i1 + a], v2 = V[3 * i2 + a], v3 = V[3 * i3 + a];
            const double lo = fmin(fmin(v0, v1), fmin(v2, v3)) - pad;
            const double hi = fmax(fmax(v0, v1), fmax(v2, v3)) + pad;
            box[6 * t + a] = lo;
            box[6 * t + 3 + a] = hi;
            const double c = 0.5 * (lo + hi);
            v[a] = fmin(v[a], c);
            v[3 + a] = fmax(v[3 + a], c);
        }
    }
    bounds_fold(v, cbounds);
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {   // 21 bits -> every third bit
    x &= 0x1fffffull;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

// 2. Morton codes of the box centres
__global__ void __launch_bounds__(256) morton_kernel(int64_t T, const double *__restrict__ box,
                                                     const unsigned long long *cbounds,
                                                     uint64_t *__restrict__ code, uint32_t *__restrict__ id) {
    double lo[3], inv[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = unord(cbounds[a]);
        const double ext = unord(cbounds[3 + a]) - lo[a];
        inv[a] = ext > 0.0 ? (double)(1 << MORTON_BITS) / ext : 0.0;
    }
    GRID_STRIDE(t, T) {
        uint64_t c = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double cen = 0.5 * (box[6 * t + a] + box[6 * t + 3 + a]);
            double q = (cen - lo[a]) * inv[a];
            q = fmin(fmax(q, 0.0), (double)((1 << MORTON_BITS) - 1));
            c |= spread3((uint64_t)q) << (2 - a);
        }
        code[t] = c;
        id[t] = (uint32_t)t;
    }
}

// cluster heads: flag[i] = code[i] != code[i - 1]
__global__ void heads_kernel(int64_t T, const uint64_t *__restrict__ code, uint32_t *__restrict__ flag) {
    GRID_STRIDE(i, T) flag[i] = (i == 0 || code[i] != code[i - 1]) ? 1u : 0u;
}

// cstart[cluster] = first sorted position, ucode[cluster] = its code
__global__ void clusters_kernel(int64_t T, const uint64_t *__restrict__ code,
                                const uint32_t *__restrict__ flag, const uint32_t *__restrict__ cidx,
                                uint32_t *__restrict__ cstart, uint64_t *__restrict__ ucode, int64_t n_u) {
    GRID_STRIDE(i, T) {
        if (flag[i]) {
            cstart[cidx[i]] = (uint32_t)i;
            ucode[cidx[i]] = code[i];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) cstart[n_u] = (uint32_t)T;
}

__device__ __forceinline__ int delta(const uint64_t *k, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    return __clzll((long long)(k[i] ^ k[j]));
}

// 3. Karras (2012) radix tree over n unique codes: internal node i covers
// clusters [first, last]; children are internal (>= 0) or cluster ~j.
__global__ void karras_kernel(int64_t n, const uint64_t *__restrict__ k, int32_t *__restrict__ first,
                              int32_t *__restrict__ last, int32_t *__restrict__ left,
                              int32_t *__restrict__ right) {
    GRID_STRIDE(i, n - 1) {
        const int d = delta(k, n, i, i + 1) > delta(k, n, i, i - 1) ? 1 : -1;
        const int dmin = delta(k, n, i, i - d);
        int64_t lmax = 2;
        while (delta(k, n, i, i + lmax * d) > dmin) lmax *= 2;
        int64_t l = 0;
        for (int64_t t = lmax / 2; t >= 1; t /= 2)
            if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
        const int64_t j = i + l * d;
        const int dnode = delta(k, n, i, j);
        int64_t s = 0;
        for (int64_t div = 2;; div *= 2) {
            const int64_t t = (l + div - 1) / div;
            if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
            if (t <= 1) break;
        }
        const int64_t gamma = i + s * d + (d < 0 ? -1 : 0);
        const int64_t f = i < j ? i : j, g = i < j ? j : i;
        first[i] = (int32_t)f;
        last[i] = (int32_t)g;
        left[i] = f == gamma ? ~(int32_t)gamma : (int32_t)gamma;
        right[i] = g == gamma + 1 ? ~(int32_t)(gamma + 1) : (int32_t)(gamma + 1);
    }
}

struct Tree {
    const int32_t *first, *last, *left, *right;
    const uint32_t *cstart;
    int32_t leaf_max;
    __device__ __forceinline__ void range(int32_t c, int32_t &f, int32_t &l) const {
        if (c < 0) { f = l = ~c; } else { f = first[c]; l = last[c]; }
    }
    __device__ __forceinline__ int64_t count(int32_t c) const {
        int32_t f, l;
        range(c, f, l);
        return (int64_t)cstart[l + 1] - (int64_t)cstart[f];
    }
    __device__ __forceinline__ bool kept(int32_t c) const { return c >= 0 && count(c) > leaf_max; }
};

// 4a. keep flags of internal nodes and leaf heads over clusters
__global__ void keep_kernel(int64_t n_int, Tree Tr, uint32_t *__restrict__ keep,
                            uint32_t *__restrict__ leafhead, int32_t *__restrict__ err) {
    GRID_STRIDE(i, n_int) {
        const bool k = Tr.kept((int32_t)i);
        keep[i] = k ? 1u : 0u;
        if (!k) continue;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int32_t c = s == 0 ? Tr.left[i] : Tr.right[i];
            if (Tr.kept(c)) continue;
            int32_t f, l;
            Tr.range(c, f, l);
            leafhead[f] = 1u;
            if (Tr.count(c) > 64) atomicExch(err, 1);   // one cluster of > 64 equal codes
        }
    }
}

// 4b. renumbered links: TrPNode.child, leaf ranges, parents
__global__ void link_kernel(int64_t n_int, Tree Tr, const uint32_t *__restrict__ keep,
                            const uint32_t *__restrict__ nidx, const uint32_t *__restrict__ lidx,
                            TrPNode *__restrict__ nodes, int32_t *__restrict__ node_parent,
                            uint8_t *__restrict__ node_slot, uint32_t *__restrict__ leaf_b,
                            uint32_t *__restrict__ leaf_e, int32_t *__restrict__ leaf_parent,
                            uint8_t *__restrict__ leaf_slot) {
    GRID_STRIDE(i, n_int) {
        if (!keep[i]) continue;
        const int32_t p = (int32_t)nidx[i];
        if (i == 0) { node_parent[0] = -1; node_slot[0] = 0; }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int32_t c = s == 0 ? Tr.left[i] : Tr.right[i];
            if (Tr.kept(c)) {
                const int32_t q = (int32_t)nidx[c];
                nodes[p].child[s] = q;
                node_parent[q] = p;
                node_slot[q] = (uint8_t)s;
            } else {
                int32_t f, l;
                Tr.range(c, f, l);
                const int32_t L = (int32_t)lidx[f];
                nodes[p].child[s] = ~L;
                leaf_b[L] = Tr.cstart[f];
                leaf_e[L] = Tr.cstart[l + 1];
                leaf_parent[L] = p;
                leaf_slot[L] = (uint8_t)s;
            }
        }
    }
}

__device__ __forceinline__ void set_child(TrPNode &N, int s, const double b[6], uint32_t minid) {
    float *lo = s == 0 ? N.lo0 : N.lo1, *hi = s == 0 ? N.hi0 : N.hi1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = __double2float_rd(b[a]);
        hi[a] = __double2float_ru(b[3 + a]);
    }
    N.minid[s] = minid;
}

// 4c + 5. sort each leaf's ids, its exact box, TrPLeaf header; then climb and
// refit (the second child to arrive at a node computes the node's union).
__global__ void __launch_bounds__(256) leaves_refit_kernel(
    int64_t n_leaves, uint32_t *__restrict__ ids, const double *__restrict__ box,
    const uint32_t *__restrict__ leaf_b, const uint32_t *__restrict__ leaf_e,
    const int32_t *__restrict__ leaf_parent, const uint8_t *__restrict__ leaf_slot,
    const int32_t *__restrict__ node_parent, const uint8_t *__restrict__ node_slot,
    TrPLeaf *__restrict__ leaves, double *__restrict__ leafbox, TrPNode *nodes, double *cbox,
    uint32_t *cmin, uint32_t *visit) {
    GRID_STRIDE(L, n_leaves) {
        const uint32_t b = leaf_b[L], e = leaf_e[L];
        for (uint32_t x = b + 1; x < e; ++x) {   // insertion sort (<= 64 ids, mostly sorted)
            const uint32_t v = ids[x];
            uint32_t y = x;
            while (y > b && ids[y - 1] > v) { ids[y] = ids[y - 1]; --y; }
            ids[y] = v;
        }
        double bx[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (uint32_t x = b; x < e; ++x) {
            const double *tb = box + 6 * (size_t)ids[x];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                bx[a] = fmin(bx[a], tb[a]);
                bx[3 + a] = fmax(bx[3 + a], tb[3 + a]);
            }
        }
        TrPLeaf lf;
#pragma unroll
        for (int a = 0; a < 3; ++a) { lf.ex_lo[a] = 1.0f; lf.ex_hi[a] = 0.0f; }
        lf.start = b;
        lf.count = e - b;
#pragma unroll
        for (int w = 0; w < 8; ++w) lf.walk[w] = 0u;
        leaves[L] = lf;
#pragma unroll
        for (int a = 0; a < 6; ++a) leafbox[6 * L + a] = bx[a];
        uint32_t mid = ids[b];
        int32_t p = leaf_parent[L];
        int s = leaf_slot[L];
        while (p >= 0) {
            set_child(nodes[p], s, bx, mid);
            volatile double *cb = cbox + 12 * (size_t)p + 6 * s;
#pragma unroll
            for (int a = 0; a < 6; ++a) cb[a] = bx[a];
            ((volatile uint32_t *)cmin)[2 * p + s] = mid;
            __threadfence();
            if (atomicAdd(visit + p, 1u) == 0u) break;   // the sibling finishes this node
            __threadfence();
            const volatile double *ob = cbox + 12 * (size_t)p + 6 * (1 - s);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                bx[a] = fmin(bx[a], ob[a]);
                bx[3 + a] = fmax(bx[3 + a], ob[3 + a]);
            }
            mid = min(mid, ((volatile uint32_t *)cmin)[2 * p + 1 - s]);
            s = node_slot[p];
            p = node_parent[p];
        }
    }
}

__device__ __forceinline__ bool boxes_meet(const double *a, const double *b) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (a[k] > b[3 + k] || b[k] > a[3 + k]) return false;
    return true;
}

// 6. exclusive boxes (host p_exclusive_boxes, same greedy cut rule)
__global__ void __launch_bounds__(128) exclusive_kernel(int64_t n_leaves, const TrPNode *__restrict__ nodes,
                                                        const double *__restrict__ leafbox,
                                                        TrPLeaf *__restrict__ leaves) {
    GRID_STRIDE(L, n_leaves) {
        double B[6], E[6];
#pragma unroll
        for (int a = 0; a < 6; ++a) B[a] = E[a] = leafbox[6 * L + a];
        int32_t stack[EX_STACK];
        int sp = 0;
        stack[sp++] = 0;
        bool dead = false;
        while (sp > 0 && !dead) {
            const TrPNode &N = nodes[stack[--sp]];
            for (int c = 0; c < 2; ++c) {
                const int32_t ch = N.child[c];
                if (ch == CHILD_NONE) continue;
                const float *lo = c == 0 ? N.lo0 : N.lo1, *hi = c == 0 ? N.hi0 : N.hi1;
                const double cb[6] = {lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]};
                if (!boxes_meet(cb, B)) continue;
                if (ch >= 0) {
                    if (sp == EX_STACK) { dead = true; break; }   // never for <= 60-bit codes
                    stack[sp++] = ch;
                    continue;
                }
                const int64_t M = ~ch;
                if (M == L) continue;
                double Mb[6];
#pragma unroll
                for (int a = 0; a < 6; ++a) Mb[a] = leafbox[6 * M + a];
                if (!boxes_meet(Mb, E)) continue;
                double best_vol = -1.0, cut_val = 0.0;
                int cut_axis = -1, cut_side = 0;
                for (int a = 0; a < 3; ++a) {
                    for (int side = 0; side < 2; ++side) {
                        double nlo = E[a], nhi = E[3 + a];
                        if (side == 0) { if (!(Mb[a] > E[a])) continue; nhi = Mb[a]; }
                        else { if (!(Mb[3 + a] < E[3 + a])) continue; nlo = Mb[3 + a]; }
                        double vol = 1.0;
                        for (int q = 0; q < 3; ++q) {
                            const double lo_q = q == a ? nlo : E[q], hi_q = q == a ? nhi : E[3 + q];
                            vol *= fmax(0.0, hi_q - lo_q);
                        }
                        if (vol > best_vol) {
                            best_vol = vol;
                            cut_axis = a;
                            cut_side = side;
                            cut_val = side == 0 ? nhi : nlo;
                        }
                    }
                }
                if (cut_axis < 0) { dead = true; break; }   // M covers E
                if (cut_side == 0) E[3 + cut_axis] = cut_val; else E[cut_axis] = cut_val;
            }
        }
        TrPLeaf &LF = leaves[L];
        if (dead || !(E[0] <= E[3])) {
            LF.ex_lo[0] = 1.0f;
            LF.ex_hi[0] = 0.0f;
            LF.ex_lo[1] = LF.ex_lo[2] = 1.0f;
            LF.ex_hi[1] = LF.ex_hi[2] = 0.0f;
        } else {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                LF.ex_lo[a] = __double2float_ru(E[a]);
                LF.ex_hi[a] = __double2float_rd(E[3 + a]);
            }
        }
    }
}

__global__ void __launch_bounds__(256) leaf_bounds_kernel(int64_t n_leaves, const double *__restrict__ leafbox,
                                                          unsigned long long *bounds) {
    double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    GRID_STRIDE(L, n_leaves) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            v[a] = fmin(v[a], leafbox[6 * L + a]);
            v[3 + a] = fmax(v[3 + a], leafbox[6 * L + 3 + a]);
        }
    }
    bounds_fold(v, bounds);
}

struct GridP {
    int32_t dim[3];
    double org[3], scale[3];
};

// 7. grid candidates: per leaf, every cell its exclusive box meets
__global__ void __launch_bounds__(256) grid_vote_kernel(int64_t n_leaves, const TrPLeaf *__restrict__ leaves,
                                                        GridP G, unsigned long long *__restrict__ vote) {
    GRID_STRIDE(L, n_leaves) {
        const TrPLeaf lf = leaves[L];
        double e0[3], e1[3];
        bool ok = true;
        int64_t c0[3], c1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            e0[a] = lf.ex_lo[a];
            e1[a] = lf.ex_hi[a];
            ok = ok && e0[a] < e1[a];
            const int64_t f0 = (int64_t)floor((e0[a] - G.org[a]) * G.scale[a]);
            const int64_t f1 = (int64_t)floor((e1[a] - G.org[a]) * G.scale[a]);
            c0[a] = clampi(f0, G.dim[a] - 1);
            c1[a] = clampi(f1, G.dim[a] - 1);
        }
        if (!ok) continue;
        for (int64_t x = c0[0]; x <= c1[0]; ++x)
            for (int64_t y = c0[1]; y <= c1[1]; ++y)
                for (int64_t z = c0[2]; z <= c1[2]; ++z) {
                    const int64_t c[3] = {x, y, z};
                    double ov = 1.0;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const double cl = G.org[a] + (double)c[a] / G.scale[a];
                        const double ch = G.org[a] + (double)(c[a] + 1) / G.scale[a];
                        ov *= fmax(0.0, fmin(e1[a], ch) - fmax(e0[a], cl));
                    }
                    const float ovf = (float)ov;
                    if (!(ovf > 0.0f)) continue;
                    const unsigned long long key = ((unsigned long long)__float_as_uint(ovf) << 32) |
                                                   (unsigned long long)(0xffffffffu - (uint32_t)L);
                    atomicMax(vote + (x * G.dim[1] + y) * G.dim[2] + z, key);
                }
    }
}

__global__ void __launch_bounds__(256) grid_final_kernel(int64_t n_cells, const unsigned long long *__restrict__ vote,
                                                         double cell_vol, int32_t *__restrict__ grid,
                                                         double *cov) {
    double acc = 0.0;
    GRID_STRIDE(c, n_cells) {
        const unsigned long long k = vote[c];
        if (k == 0ull) { grid[c] = -1; continue; }
        grid[c] = (int32_t)(0xffffffffu - (uint32_t)(k & 0xffffffffull));
        acc += fmin((double)__uint_as_float((uint32_t)(k >> 32)) / cell_vol, 1.0);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(cov, acc);
}

// 8. cell candidate lists (host tr_cells_build)
struct CellP {
    int32_t dim[3];
    double org[3], scale[3];
};

__device__ __forceinline__ void crange(const CellP &Cp, const double *b, int64_t c0[3], int64_t c1[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double f0 = (b[a] - Cp.org[a]) * Cp.scale[a], f1 = (b[3 + a] - Cp.org[a]) * Cp.scale[a];
        c0[a] = clampi((int64_t)floor(f0), Cp.dim[a] - 1);
        c1[a] = clampi((int64_t)floor(f1), Cp.dim[a] - 1);
    }
}

__global__ void __launch_bounds__(256) cells_count_kernel(int64_t nrec, const uint32_t *__restrict__ ids,
                                                          const double *__restrict__ box, CellP Cp,
                                                          uint32_t *__restrict__ cnt) {
    GRID_STRIDE(k, nrec) {
        int64_t c0[3], c1[3];
        crange(Cp, box + 6 * (size_t)ids[k], c0, c1);
        for (int64_t x = c0[0]; x <= c1[0]; ++x)
            for (int64_t y = c0[1]; y <= c1[1]; ++y)
                for (int64_t z = c0[2]; z <= c1[2]; ++z)
                    atomicAdd(cnt + (x * Cp.dim[1] + y) * Cp.dim[2] + z, 1u);
    }
}

__global__ void cells_eff_kernel(int64_t n, const uint32_t *__restrict__ cnt, uint32_t max_list,
                                 uint64_t *__restrict__ eff) {
    GRID_STRIDE(c, n) eff[c] = cnt[c] <= max_list ? cnt[c] : 0u;
}

__global__ void __launch_bounds__(256) cells_fill_kernel(int64_t nrec, const uint32_t *__restrict__ ids,
                                                         const double *__restrict__ box, CellP Cp,
                                                         const uint32_t *__restrict__ cnt, uint32_t max_list,
                                                         const uint64_t *__restrict__ off,
                                                         uint32_t *__restrict__ fill, uint32_t *__restrict__ recs) {
    GRID_STRIDE(k, nrec) {
        int64_t c0[3], c1[3];
        crange(Cp, box + 6 * (size_t)ids[k], c0, c1);
        for (int64_t x = c0[0]; x <= c1[0]; ++x)
            for (int64_t y = c0[1]; y <= c1[1]; ++y)
                for (int64_t z = c0[2]; z <= c1[2]; ++z) {
                    const int64_t c = (x * Cp.dim[1] + y) * Cp.dim[2] + z;
                    if (cnt[c] > max_list) continue;
                    recs[off[c] + atomicAdd(fill + c, 1u)] = (uint32_t)k;
                }
    }
}

__global__ void cells_sort_kernel(int64_t n, const uint32_t *__restrict__ cnt, uint32_t max_list,
                                  const uint64_t *__restrict__ off, const uint32_t *__restrict__ ids,
                                  uint32_t *__restrict__ recs, uint32_t *__restrict__ off32) {
    GRID_STRIDE(c, n) {
        const uint32_t m = cnt[c];
        const uint64_t o = off[c];
        off32[c] = (uint32_t)o | (m > max_list ? 0x80000000u : 0u);
        if (c == n - 1) off32[n] = (uint32_t)off[n];
        if (m > max_list) continue;
        uint32_t *r = recs + o;
        for (uint32_t x = 1; x < m; ++x) {   // ascending tet id
            const uint32_t v = r[x], kv = ids[v];
            uint32_t y = x;
            while (y > 0 && ids[r[y - 1]] > kv) { r[y] = r[y - 1]; --y; }
            r[y] = v;
        }
    }
}

__global__ void tbox_kernel(int64_t nrec, const uint32_t *__restrict__ ids, const double *__restrict__ box,
                            float *__restrict__ tbox) {
    GRID_STRIDE(k, nrec) {
        const double *b = box + 6 * (size_t)ids[k];
        float4 lo, hi;
        lo.x = __double2float_rd(b[0]);
        lo.y = __double2float_rd(b[1]);
        lo.z = __double2float_rd(b[2]);
        lo.w = __double2float_ru(b[3]);
        hi.x = __double2float_ru(b[4]);
        hi.y = __double2float_ru(b[5]);
        hi.z = 0.0f;
        hi.w = 0.0f;
        reinterpret_cast<float4 *>(tbox)[2 * k] = lo;
        reinterpret_cast<float4 *>(tbox)[2 * k + 1] = hi;
    }
}

__global__ void grid_leaf_kernel(int64_t n, const int32_t *__restrict__ grid, const TrPLeaf *__restrict__ leaves,
                                 TrPLeaf *__restrict__ out, const TrLeafPred *__restrict__ pred,
                                 TrLeafPred *__restrict__ pred_out) {
    GRID_STRIDE(c, n) {
        const int32_t L = grid[c];
        if (pred_out) {
            TrLeafPred p = {};
            if (L >= 0 && pred) p = pred[L];
            pred_out[c] = p;
        }
        TrPLeaf lf;
        if (L >= 0) {
            lf = leaves[L];
        } else {
#pragma unroll
            for (int a = 0; a < 3; ++a) { lf.ex_lo[a] = 1.0f; lf.ex_hi[a] = 0.0f; }
            lf.start = lf.count = 0u;
#pragma unroll
            for (int w = 0; w < 8; ++w) lf.walk[w] = 0u;
        }
        out[c] = lf;
    }
}

__global__ void pack_kernel(int64_t n, const int64_t *__restrict__ tets, const double *__restrict__ orig,
                            const double *__restrict__ inv, const double *__restrict__ field, int32_t centering,
                            const uint32_t *__restrict__ order, TrTetRecord *__restrict__ out) {
    GRID_STRIDE(k, n) {
        const int64_t t = order ? (int64_t)order[k] : k;
        TrTetRecord R;
#pragma unroll
        for (int q = 0; q < 9; ++q) R.inv[q] = inv[9 * t + q];
#pragma unroll
        for (int q = 0; q < 3; ++q) R.orig[q] = orig[3 * t + q];
        if (centering == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) R.f[q] = field[tets[4 * t + q]];
        } else {
            R.f[0] = field[t];
            R.f[1] = R.f[2] = R.f[3] = 0.0;
        }
        out[k] = R;
    }
}

// Scratch of one build (freed on every exit path).
struct Scratch {
    cudaStream_t st;
    void *p[64] = {};
    int n = 0;
    cudaError_t err = cudaSuccess;
    template <class T>
    T *get(size_t count) {
        void *q = nullptr;
        if (n == (int)(sizeof p / sizeof p[0])) err = cudaErrorMemoryAllocation;   // table full
        if (err == cudaSuccess) err = cudaMallocAsync(&q, count * sizeof(T) + 16, st);
        if (err != cudaSuccess) return nullptr;
        p[n++] = q;
        return static_cast<T *>(q);
    }
    ~Scratch() {
        for (int i = 0; i < n; ++i) cudaFreeAsync(p[i], st);
    }
};

void free_build(TrDevPointBuild *B) {
    if (!B) return;
    void *ps[] = {B->nodes, B->leaves, B->ids, B->grid, B->coff, B->crecs, B->tbox, B->pred};
    for (void *q : ps)
        if (q) cudaFreeAsync(q, B->st);
    cudaStreamSynchronize(B->st);
    delete B;
}

}  // namespace

extern "C" {

int tr_pbvh_build_device(int64_t n_vertices, const double *vertices, int64_t n_tets, const int64_t *tets,
                         double pad, int32_t leaf_max, double cells_below, int32_t refine, int32_t max_list,
                         void *stream, TrDevPointBuild **out) {
    if (!out || !vertices || !tets || n_vertices < 4 || n_tets <= leaf_max || n_tets >= (int64_t)INT32_MAX ||
        leaf_max < 1 || leaf_max > 64 || refine < 1 || refine > 8 || max_list < 1 || !(pad >= 0.0))
        return tr_fail(TR_EINVAL, "tr_pbvh_build_device: invalid arguments");
    *out = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t T = n_tets;
    TrDevPointBuild *B = new TrDevPointBuild();
    B->st = st;
    B->n_tets = T;
    cudaError_t e = cudaSuccess, ce = cudaSuccess;   // ce: first CUB error
    auto ck = [&ce](cudaError_t x) { if (x != cudaSuccess && ce == cudaSuccess) ce = x; };
    int rc = TR_OK;
    {
        Scratch S{st};
        double *box = S.get<double>(6 * (size_t)T);
        unsigned long long *bnd = S.get<unsigned long long>(12);
        uint64_t *code = S.get<uint64_t>(T), *code2 = S.get<uint64_t>(T);
        uint32_t *id = S.get<uint32_t>(T);
        uint32_t *flag = S.get<uint32_t>(T), *cidx = S.get<uint32_t>(T);
        int32_t *err = S.get<int32_t>(1);
        double *cov = S.get<double>(1);
        e = S.err;
        if (e == cudaSuccess) e = cudaMallocAsync(&B->ids, T * sizeof(uint32_t), st);
        if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: allocation"); }
        unsigned long long h_init[12];
        for (int a = 0; a < 12; ++a) h_init[a] = (a % 6) < 3 ? ~0ull : 0ull;
        cudaMemcpyAsync(bnd, h_init, sizeof h_init, cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(err, 0, sizeof(int32_t), st);
        cudaMemsetAsync(cov, 0, sizeof(double), st);
        boxes_kernel<<<grid_for(T), 256, 0, st>>>(T, vertices, tets, pad, box, bnd);
        morton_kernel<<<grid_for(T), 256, 0, st>>>(T, box, bnd, code, id);
        // radix sort (code, id): stable, ids ascending within equal codes
        size_t tmp_bytes = 0, tb2 = 0;
        ck(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, code, code2, id, B->ids, (int)T, 0,
                                        3 * MORTON_BITS, st));
        ck(cub::DeviceScan::ExclusiveSum(nullptr, tb2, flag, cidx, (int)T, st));
        if (tb2 > tmp_bytes) tmp_bytes = tb2;
        void *tmp = S.get<uint8_t>(tmp_bytes + 1024);
        if ((e = S.err) != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: allocation"); }
        size_t tsz = tmp_bytes;
        ck(cub::DeviceRadixSort::SortPairs(tmp, tsz, code, code2, id, B->ids, (int)T, 0, 3 * MORTON_BITS, st));
        heads_kernel<<<grid_for(T), 256, 0, st>>>(T, code2, flag);
        tsz = tmp_bytes;
        ck(cub::DeviceScan::ExclusiveSum(tmp, tsz, flag, cidx, (int)T, st));
        uint32_t last_c = 0, last_f = 0;
        cudaMemcpyAsync(&last_c, cidx + T - 1, 4, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&last_f, flag + T - 1, 4, cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st)) == cudaSuccess) e = ce;
        if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: sort"); }
        const int64_t n_u = (int64_t)last_c + last_f;
        if (n_u < 2) { free_build(B); return tr_fail(TR_EINVAL, "tr_pbvh_build_device: every tet box has the same centre"); }
        uint32_t *cstart = S.get<uint32_t>(n_u + 1);
        uint64_t *ucode = S.get<uint64_t>(n_u);
        const int64_t n_int = n_u - 1;
        int32_t *first = S.get<int32_t>(n_int), *last = S.get<int32_t>(n_int);
        int32_t *left = S.get<int32_t>(n_int), *right = S.get<int32_t>(n_int);
        uint32_t *keep = S.get<uint32_t>(n_int), *nidx = S.get<uint32_t>(n_int);
        uint32_t *lhead = S.get<uint32_t>(n_u), *lidx = S.get<uint32_t>(n_u);
        if ((e = S.err) != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: allocation"); }
        clusters_kernel<<<grid_for(T), 256, 0, st>>>(T, code2, flag, cidx, cstart, ucode, n_u);
        karras_kernel<<<grid_for(n_int), 256, 0, st>>>(n_u, ucode, first, last, left, right);
        cudaMemsetAsync(lhead, 0, n_u * sizeof(uint32_t), st);
        Tree Tr{first, last, left, right, cstart, leaf_max};
        keep_kernel<<<grid_for(n_int), 256, 0, st>>>(n_int, Tr, keep, lhead, err);
        tsz = tmp_bytes;
        ck(cub::DeviceScan::ExclusiveSum(tmp, tsz, keep, nidx, (int)n_int, st));
        tsz = tmp_bytes;
        ck(cub::DeviceScan::ExclusiveSum(tmp, tsz, lhead, lidx, (int)n_u, st));
        uint32_t h4[5] = {0, 0, 0, 0, 0};
        cudaMemcpyAsync(h4 + 0, nidx + n_int - 1, 4, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(h4 + 1, keep + n_int - 1, 4, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(h4 + 2, lidx + n_u - 1, 4, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(h4 + 3, lhead + n_u - 1, 4, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(h4 + 4, err, 4, cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st)) == cudaSuccess) e = ce;
        if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: tree"); }
        if (h4[4]) { free_build(B); return tr_fail(TR_EINVAL, "tr_pbvh_build_device: more than 64 tets share a Morton cell"); }
        B->n_nodes = (int64_t)h4[0] + h4[1];
        B->n_leaves = (int64_t)h4[2] + h4[3];
        const int64_t NN = B->n_nodes, NL = B->n_leaves;
        int32_t *node_parent = S.get<int32_t>(NN), *leaf_parent = S.get<int32_t>(NL);
        uint8_t *node_slot = S.get<uint8_t>(NN), *leaf_slot = S.get<uint8_t>(NL);
        uint32_t *leaf_b = S.get<uint32_t>(NL), *leaf_e = S.get<uint32_t>(NL);
        double *leafbox = S.get<double>(6 * (size_t)NL), *cbox = S.get<double>(12 * (size_t)NN);
        uint32_t *cmin = S.get<uint32_t>(2 * (size_t)NN), *visit = S.get<uint32_t>(NN);
        if ((e = S.err) == cudaSuccess) e = cudaMallocAsync(&B->nodes, NN * sizeof(TrPNode), st);
        if (e == cudaSuccess) e = cudaMallocAsync(&B->leaves, NL * sizeof(TrPLeaf), st);
        if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: allocation"); }
        cudaMemsetAsync(visit, 0, NN * sizeof(uint32_t), st);
        link_kernel<<<grid_for(n_int), 256, 0, st>>>(n_int, Tr, keep, nidx, lidx, B->nodes, node_parent,
                                                      node_slot, leaf_b, leaf_e, leaf_parent, leaf_slot);
        leaves_refit_kernel<<<grid_for(NL), 256, 0, st>>>(NL, B->ids, box, leaf_b, leaf_e, leaf_parent,
                                                           leaf_slot, node_parent, node_slot, B->leaves,
                                                           leafbox, B->nodes, cbox, cmin, visit);
        exclusive_kernel<<<grid_for(NL) * 2, 128, 0, st>>>(NL, B->nodes, leafbox, B->leaves);
        leaf_bounds_kernel<<<grid_for(NL), 256, 0, st>>>(NL, leafbox, bnd + 6);
        unsigned long long hb[6];
        cudaMemcpyAsync(hb, bnd + 6, sizeof hb, cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: refit"); }
        // grid dims: host p_build_grid's expressions
        double lo[3], hi[3], ext[3], vol = 1.0;
        for (int a = 0; a < 3; ++a) {
            lo[a] = unord(hb[a]);
            hi[a] = unord(hb[3 + a]);
            ext[a] = std::max(hi[a] - lo[a], 1e-300);
            vol *= ext[a];
        }
        const double side = std::cbrt(vol / (double)std::max<int64_t>(NL, 1));
        int64_t cells = 1;
        GridP G;
        for (int a = 0; a < 3; ++a) {
            const double d = std::round(ext[a] / side);
            B->gdim[a] = G.dim[a] = (int32_t)std::min(std::max(d, 1.0), 2048.0);
            cells *= B->gdim[a];
            B->gorg[a] = G.org[a] = lo[a];
            B->gscale[a] = G.scale[a] = (double)B->gdim[a] / ext[a];
        }
        B->n_grid = cells;
        unsigned long long *vote = S.get<unsigned long long>(cells);
        if ((e = S.err) == cudaSuccess) e = cudaMallocAsync(&B->grid, cells * sizeof(int32_t), st);
        if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: allocation"); }
        cudaMemsetAsync(vote, 0, cells * sizeof(unsigned long long), st);
        grid_vote_kernel<<<grid_for(NL), 256, 0, st>>>(NL, B->leaves, G, vote);
        double cell_vol = 1.0;
        for (int a = 0; a < 3; ++a) cell_vol /= B->gscale[a];
        grid_final_kernel<<<grid_for(cells), 256, 0, st>>>(cells, vote, cell_vol, B->grid, cov);
        double hcov = 0.0;
        cudaMemcpyAsync(&hcov, cov, sizeof(double), cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: grid"); }
        B->coverage = cells > 0 ? hcov / (double)cells : 0.0;
        if (B->coverage < cells_below) {
            CellP Cp;
            int64_t nc = 1;
            for (int a = 0; a < 3; ++a) {
                B->cdim[a] = Cp.dim[a] = (int32_t)std::min<int64_t>((int64_t)B->gdim[a] * refine, 4096);
                B->corg[a] = Cp.org[a] = B->gorg[a];
                B->cscale[a] = Cp.scale[a] = B->gscale[a] * (double)B->cdim[a] / (double)B->gdim[a];
                nc *= B->cdim[a];
            }
            B->n_ccells = nc;
            uint32_t *cnt = S.get<uint32_t>(nc), *fill = S.get<uint32_t>(nc);
            uint64_t *eff = S.get<uint64_t>(nc + 1), *off = S.get<uint64_t>(nc + 1);
            size_t tb3 = 0;
            ck(cub::DeviceScan::ExclusiveSum(nullptr, tb3, eff, off, (int)(nc + 1), st));
            void *tmp3 = S.get<uint8_t>(tb3 + 16);
            if ((e = S.err) == cudaSuccess) e = cudaMallocAsync(&B->coff, (nc + 1) * sizeof(uint32_t), st);
            if (e == cudaSuccess) e = cudaMallocAsync(&B->tbox, T * 8 * sizeof(float), st);
            if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: allocation"); }
            cudaMemsetAsync(cnt, 0, nc * sizeof(uint32_t), st);
            cudaMemsetAsync(fill, 0, nc * sizeof(uint32_t), st);
            cudaMemsetAsync(eff + nc, 0, sizeof(uint64_t), st);
            cells_count_kernel<<<grid_for(T), 256, 0, st>>>(T, B->ids, box, Cp, cnt);
            cells_eff_kernel<<<grid_for(nc), 256, 0, st>>>(nc, cnt, (uint32_t)max_list, eff);
            ck(cub::DeviceScan::ExclusiveSum(tmp3, tb3, eff, off, (int)(nc + 1), st));
            uint64_t total = 0;
            cudaMemcpyAsync(&total, off + nc, 8, cudaMemcpyDeviceToHost, st);
            if ((e = cudaStreamSynchronize(st)) == cudaSuccess) e = ce;
            if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: cells"); }
            if (total >= 0x7fffffffull) { free_build(B); return tr_fail(TR_ENOMEM, "tr_pbvh_build_device: cell lists too large"); }
            B->n_crecs = (int64_t)total;
            e = cudaMallocAsync(&B->crecs, std::max<uint64_t>(total, 1) * sizeof(uint32_t), st);
            if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: allocation"); }
            cells_fill_kernel<<<grid_for(T), 256, 0, st>>>(T, B->ids, box, Cp, cnt, (uint32_t)max_list, off,
                                                           fill, B->crecs);
            cells_sort_kernel<<<grid_for(nc), 256, 0, st>>>(nc, cnt, (uint32_t)max_list, off, B->ids, B->crecs,
                                                            B->coff);
            tbox_kernel<<<grid_for(T), 256, 0, st>>>(T, B->ids, box, B->tbox);
        }
        if ((e = cudaGetLastError()) == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device"); }
    }   // scratch freed (stream-ordered)
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { free_build(B); return cuda_fail(e, "tr_pbvh_build_device: free"); }
    *out = B;
    return rc;
}

int tr_dpb_sizes(const TrDevPointBuild *b, int64_t *sizes6) {
    if (!b || !sizes6) return tr_fail(TR_EINVAL, "tr_dpb_sizes: invalid arguments");
    sizes6[0] = b->n_nodes;
    sizes6[1] = b->n_leaves;
    sizes6[2] = b->n_tets;
    sizes6[3] = b->n_grid;
    sizes6[4] = b->n_ccells;
    sizes6[5] = b->n_crecs;
    return TR_OK;
}

int tr_dpb_grid(const TrDevPointBuild *b, int32_t *gdim3, double *gorg3, double *gscale3, double *coverage,
                int32_t *cdim3, double *corg3, double *cscale3) {
    if (!b) return tr_fail(TR_EINVAL, "tr_dpb_grid: invalid arguments");
    for (int a = 0; a < 3; ++a) {
        if (gdim3) gdim3[a] = b->gdim[a];
        if (gorg3) gorg3[a] = b->gorg[a];
        if (gscale3) gscale3[a] = b->gscale[a];
        if (cdim3) cdim3[a] = b->cdim[a];
        if (corg3) corg3[a] = b->corg[a];
        if (cscale3) cscale3[a] = b->cscale[a];
    }
    if (coverage) *coverage = b->coverage;
    return TR_OK;
}

int tr_dpb_copy(const TrDevPointBuild *b, TrPNode *nodes, TrPLeaf *leaves, uint32_t *ids, int32_t *grid,
                TrPLeaf *grid_leaf, TrLeafPred *grid_pred, uint32_t *cell_off, uint32_t *cell_recs, float *tbox,
                void *stream) {
    if (!b) return tr_fail(TR_EINVAL, "tr_dpb_copy: invalid arguments");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    auto cp = [&](void *dst, const void *src, size_t n) {
        if (dst && src && n && e == cudaSuccess) e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, st);
    };
    cp(nodes, b->nodes, b->n_nodes * sizeof(TrPNode));
    cp(leaves, b->leaves, b->n_leaves * sizeof(TrPLeaf));
    cp(ids, b->ids, b->n_tets * sizeof(uint32_t));
    cp(grid, b->grid, b->n_grid * sizeof(int32_t));
    if (b->n_ccells) {
        cp(cell_off, b->coff, (b->n_ccells + 1) * sizeof(uint32_t));
        cp(cell_recs, b->crecs, b->n_crecs * sizeof(uint32_t));
        cp(tbox, b->tbox, b->n_tets * 8 * sizeof(float));
    }
    if (e == cudaSuccess && grid_leaf)
        grid_leaf_kernel<<<grid_for(b->n_grid), 256, 0, st>>>(b->n_grid, b->grid, b->leaves, grid_leaf, b->pred,
                                                              grid_pred);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "tr_dpb_copy");
}

void tr_dpb_free(TrDevPointBuild *b) { free_build(b); }

int tr_pack_tets_device(int64_t n, const int64_t *tets, const double *tet_orig, const double *tet_inv,
                        const double *field, int32_t centering, const uint32_t *order, TrTetRecord *out,
                        void *stream) {
    if (n <= 0 || !tets || !tet_orig || !tet_inv || !field || !out || (centering != 0 && centering != 1))
        return tr_fail(TR_EINVAL, "tr_pack_tets_device: invalid arguments");
    cudaStream_t st = (cudaStream_t)stream;
    pack_kernel<<<grid_for(n), 256, 0, st>>>(n, tets, tet_orig, tet_inv, field, centering, order, out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "pack_kernel");
}

}  // extern "C"

// Host -> device copy of a large pageable host array through two page-locked
// staging chunks: host threads (OpenMP) fill one chunk while the copy engine
// drains the other (a pageable cudaMemcpy of a fresh numpy array runs at a
// fraction of PCIe speed).  Synchronous on return.
extern "C" int tr_upload(void *dst, const void *src, int64_t bytes, void *stream) {
    if (bytes < 0 || (bytes > 0 && (!dst || !src))) return tr_fail(TR_EINVAL, "tr_upload: invalid arguments");
    if (bytes == 0) return TR_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (bytes <= ((int64_t)1 << 20)) {   // small: the driver's own staging
        cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return e == cudaSuccess ? TR_OK : cuda_fail(e, "tr_upload");
    }
    const int64_t CH = (int64_t)64 << 20;
    const int nbuf = bytes > CH ? 2 : 1;
    void *stage[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < nbuf && e == cudaSuccess; ++i) {
        e = cudaHostAlloc(&stage[i], (size_t)std::min(CH, bytes), cudaHostAllocDefault);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    }
    bool used[2] = {false, false};
    for (int64_t off = 0, k = 0; off < bytes && e == cudaSuccess; off += CH, ++k) {
        const int b = (int)(k % nbuf);
        const int64_t n = std::min(CH, bytes - off);
        if (used[b] && (e = cudaEventSynchronize(ev[b])) != cudaSuccess) break;
        const char *s = static_cast<const char *>(src) + off;
        char *d = static_cast<char *>(stage[b]);
        const int64_t piece = (int64_t)1 << 20;
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < n; p += piece) memcpy(d + p, s + p, (size_t)std::min(piece, n - p));
        e = cudaMemcpyAsync(static_cast<char *>(dst) + off, d, (size_t)n, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev[b], st);
        used[b] = true;
    }
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
    for (int i = 0; i < 2; ++i) {
        if (ev[i]) cudaEventDestroy(ev[i]);
        if (stage[i]) cudaFreeHost(stage[i]);
    }
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "tr_upload");
}

// ---------------------------------------------------------------- walk tables
// tr_leaf_walk's tables (host_build.cpp walk_table) on the device: face
// neighbours by shared vertex ids, the walk's first tet (largest volume),
// the walk-start predictor, and the CERTIFIED bit of tet i when every
// lower-id tet j of the leaf is separated from it (host `separated`: a face
// plane of j has i shrunk to barycentrics >= TAU / 2 beyond -(1e-9 + 1e-8),
// or a face plane of i has j inflated by that slack below TAU / 2).  The host
// evaluates the barycentrics in long double; here each one is a ratio of
// orientation determinants, and a face test passes only if it passes with
// the determinants' forward error bound (Shewchuk's orient3d bound, taken as
// 1e-15 x the permanent) added against it -- so a device certificate implies
// the exact one (tests compare the device tables with tr_leaf_walk's).
namespace {

constexpr double W_TOL = 1e-9, W_M1 = 1e-8, W_TAU = TR_WALK_TAU;

__device__ __forceinline__ double orient_eb(const double *a, const double *b, const double *c, const double *x,
                                            double &eb) {
    const double ad0 = a[0] - x[0], ad1 = a[1] - x[1], ad2 = a[2] - x[2];
    const double bd0 = b[0] - x[0], bd1 = b[1] - x[1], bd2 = b[2] - x[2];
    const double cd0 = c[0] - x[0], cd1 = c[1] - x[1], cd2 = c[2] - x[2];
    const double det = ad0 * (bd1 * cd2 - bd2 * cd1) + ad1 * (bd2 * cd0 - bd0 * cd2) + ad2 * (bd0 * cd1 - bd1 * cd0);
    const double perm = fabs(ad0) * (fabs(bd1 * cd2) + fabs(bd2 * cd1)) +
                        fabs(ad1) * (fabs(bd2 * cd0) + fabs(bd0 * cd2)) +
                        fabs(ad2) * (fabs(bd0 * cd1) + fabs(bd1 * cd0));
    eb = 1e-15 * perm;
    return det;
}

__device__ __forceinline__ void face_of(int f, int o[3]) {
    int m = 0;
    for (int q = 0; q < 4; ++q)
        if (q != f) o[m++] = q;
}

// For every point x in pts[4]: sign(D) O_f(x) + off |D| <= 0 with the error
// bounds against it, where l_f(x) = O_f(x) / D (tet T's barycentric of f).
__device__ bool face_rejects(const double (*T)[3], int f, const double (*pts)[3], double off) {
    int o[3];
    face_of(f, o);
    double eD;
    const double D = orient_eb(T[o[0]], T[o[1]], T[o[2]], T[f], eD);
    if (!(fabs(D) > eD)) return false;
    const double sg = D > 0.0 ? 1.0 : -1.0;
    for (int i = 0; i < 4; ++i) {
        double eO;
        const double O = orient_eb(T[o[0]], T[o[1]], T[o[2]], pts[i], eO);
        if (!(sg * O + off * fabs(D) + eO + fabs(off) * eD <= 0.0)) return false;
    }
    return true;
}

__device__ bool separated_dev(const double (*J)[3], const double (*K)[3]) {
    double sk[3] = {0, 0, 0}, sj[3] = {0, 0, 0};
    for (int i = 0; i < 4; ++i)
        for (int a = 0; a < 3; ++a) { sk[a] += K[i][a]; sj[a] += J[i][a]; }
    const double s = W_TOL + W_M1;
    double w[4][3], u[4][3];
    for (int i = 0; i < 4; ++i)
        for (int a = 0; a < 3; ++a) {
            w[i][a] = (1.0 - 2.0 * W_TAU) * K[i][a] + 0.5 * W_TAU * sk[a];
            u[i][a] = (1.0 + 4.0 * s) * J[i][a] - s * sj[a];
        }
    for (int f = 0; f < 4; ++f) {
        if (face_rejects(J, f, w, s)) return true;              // l_f^J(w) <= -(slack + margin)
        if (face_rejects(K, f, u, -0.5 * W_TAU)) return true;   // l_f^K(u) <= TAU / 2
    }
    return false;
}

__global__ void __launch_bounds__(128) walk_kernel(int64_t n_leaves, TrPLeaf *__restrict__ leaves,
                                                   const uint32_t *__restrict__ ids, const double *__restrict__ V,
                                                   const int64_t *__restrict__ tets, TrLeafPred *__restrict__ pred) {
    GRID_STRIDE(L, n_leaves) {
        TrPLeaf &lf = leaves[L];
        uint32_t walk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        TrLeafPred pr = {};
        const int n = (int)min(lf.count, 9u);
        bool ok = n >= 1 && n <= 8;
        double P[8][4][3];
        int64_t vid[8][4], tid[8];
        double inv[8][3][3];
        double vmax = 0.0, imax = 0.0, vol_best = -1.0;
        int first = 0;
        for (int i = 0; ok && i < n; ++i) {
            tid[i] = ids[lf.start + i];
            for (int q = 0; q < 4; ++q) {
                vid[i][q] = tets[4 * tid[i] + q];
                for (int a = 0; a < 3; ++a) {
                    P[i][q][a] = V[3 * vid[i][q] + a];
                    vmax = fmax(vmax, fabs(P[i][q][a]));
                }
            }
            double e[3][3];   // columns v1-v0, v2-v0, v3-v0
            for (int a = 0; a < 3; ++a)
                for (int c = 0; c < 3; ++c) e[a][c] = P[i][c + 1][a] - P[i][0][a];
            const double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                               e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                               e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
            if (!(det != 0.0 && isfinite(det))) { ok = false; break; }
            double (&m)[3][3] = inv[i];
            m[0][0] = (e[1][1] * e[2][2] - e[1][2] * e[2][1]) / det;
            m[0][1] = (e[0][2] * e[2][1] - e[0][1] * e[2][2]) / det;
            m[0][2] = (e[0][1] * e[1][2] - e[0][2] * e[1][1]) / det;
            m[1][0] = (e[1][2] * e[2][0] - e[1][0] * e[2][2]) / det;
            m[1][1] = (e[0][0] * e[2][2] - e[0][2] * e[2][0]) / det;
            m[1][2] = (e[0][2] * e[1][0] - e[0][0] * e[1][2]) / det;
            m[2][0] = (e[1][0] * e[2][1] - e[1][1] * e[2][0]) / det;
            m[2][1] = (e[0][1] * e[2][0] - e[0][0] * e[2][1]) / det;
            m[2][2] = (e[0][0] * e[1][1] - e[0][1] * e[1][0]) / det;
            double isum = 0.0;
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) isum += fabs(m[r][c]);
            imax = fmax(imax, isum);
            const double vol = fabs(det);
            if (vol > vol_best) { vol_best = vol; first = i; }
        }
        if (ok) {
            const bool certifiable = imax * (vmax + 1.0) * 0x1p-51 < 1e-10;
            for (int i = 0; i < n; ++i) {
                uint32_t e = 0;
                for (int f = 0; f < 4; ++f) {
                    int64_t fa[3];
                    int m = 0;
                    for (int q = 0; q < 4; ++q)
                        if (q != f) fa[m++] = vid[i][q];
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
                    if (tid[j] < tid[i]) cert = separated_dev(P[j], P[i]);
                if (cert) e |= 1u << 12;
                walk[i >> 1] |= e << (16 * (i & 1));
            }
            walk[4] = (uint32_t)first | (1u << 31);
            for (int r = 0; r < 3; ++r) {
                double d = 0.0;
                for (int c = 0; c < 3; ++c) {
                    pr.row[r][c] = (float)inv[first][r][c];
                    d += inv[first][r][c] * ((double)lf.ex_lo[c] - P[first][0][c]);
                }
                pr.row[r][3] = (float)d;
            }
        }
        for (int k = 0; k < 8; ++k) lf.walk[k] = walk[k];
        if (pred) pred[L] = pr;
    }
}

}  // namespace

extern "C" int tr_dpb_walk(TrDevPointBuild *b, const double *vertices, const int64_t *tets, void *stream) {
    if (!b || !vertices || !tets) return tr_fail(TR_EINVAL, "tr_dpb_walk: invalid arguments");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (!b->pred) e = cudaMallocAsync(&b->pred, std::max<int64_t>(b->n_leaves, 1) * sizeof(TrLeafPred), st);
    if (e != cudaSuccess) return cuda_fail(e, "tr_dpb_walk: allocation");
    walk_kernel<<<grid_for(b->n_leaves) * 2, 128, 0, st>>>(b->n_leaves, b->leaves, b->ids, vertices, tets, b->pred);
    if ((e = cudaGetLastError()) == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "walk_kernel");
}

extern "C" int tr_ipc_alloc(int64_t bytes, void **dptr, void *handle64) {
    if (bytes <= 0 || !dptr || !handle64) return tr_fail(TR_EINVAL, "tr_ipc_alloc: invalid arguments");
    cudaError_t e = cudaMalloc(dptr, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMemset(*dptr, 0, (size_t)bytes);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, *dptr);
    if (e != cudaSuccess) return cuda_fail(e, "tr_ipc_alloc");
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle64, &h, sizeof h);
    return TR_OK;
}

extern "C" int tr_ipc_open(const void *handle64, void **dptr) {
    if (!handle64 || !dptr) return tr_fail(TR_EINVAL, "tr_ipc_open: invalid arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "tr_ipc_open");
}

extern "C" int tr_ipc_close(void *dptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dptr);
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "tr_ipc_close");
}

extern "C" int tr_dev_free(void *dptr) {
    cudaError_t e = cudaFree(dptr);
    return e == cudaSuccess ? TR_OK : cuda_fail(e, "tr_dev_free");
}
