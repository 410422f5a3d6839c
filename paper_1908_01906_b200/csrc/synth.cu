// synth.cu -- device build of the synthetic cube-grid scene.
//
// The reference builds every scene on the host in Python: generate_synthetic
// (mesh.py:147-231), MeshSampler's padded tet boxes, BVH and inverse edge
// matrices (mesh.py:246-254, bvh.py:41-98).  At 1e9 tets (BASELINE config 4)
// those host arrays alone exceed 250 GB, so for the generator's mesh the
// device-resident scene is produced here directly in HBM:
//   * tet records (128 B): vertex 0 as origin, the inverse edge matrix taken
//     from the 10 distinct ones (5 tets x 2 cube parities) that the host
//     inverts with numpy's LAPACK (bit-identical to inverting all T: the
//     integer edge matrices are translation invariant), and the f32-rounded
//     analytic field at the 4 vertices (mesh.py:170-171, 230);
//   * records in 8^3-cube brick order (ids != NULL; ids[k] = tet id of record
//     k) so that spatial neighbours share DRAM pages and L2 sets, or in id order;
//   * one leaf per cube (its 5 tets, ascending ids, consecutive records), exclusive
//     box = the cube shrunk by the box pad (no other cube's padded tet boxes
//     reach inside it), rounded inward to f32, and the walk table of its
//     parity (tr_walk_table_cube: the same builder as tr_leaf_walk's);
//   * the uniform point grid is the cube grid itself (origin 0, scale 1), so
//     a cell's candidate leaf header is the leaf array (no copy);
//   * a BVH2 over the cubes by recursive halving of the longest cube range,
//     in pre-order: node j's cube range is found by descending from the root
//     (a subtree of n cubes owns the n - 1 node indices after its root), so
//     every node is written independently; child boxes are the cube ranges
//     padded by the box pad and rounded outward, min ids = 5 x first cube.
// Every structure has the same meaning as the host builders' output, so the
// render kernels are unchanged; tests/test_grid_scene.py renders both builds
// and requires identical frames.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "grid_layout.cuh"
#include "tetray_b200.h"
#include "tr_internal.h"

namespace {

constexpr int32_t CHILD_NONE = INT32_MIN;

// mesh.py:151-163 five-tet cube pattern (corner offsets x, y, z per vertex);
// odd-parity cubes mirror x.
__constant__ int8_t c_pattern[5][4][3] = {
    {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
    {{1, 1, 0}, {0, 1, 0}, {1, 0, 0}, {1, 1, 1}},
    {{1, 0, 1}, {0, 0, 1}, {1, 1, 1}, {1, 0, 0}},
    {{0, 1, 1}, {1, 1, 1}, {0, 0, 1}, {0, 1, 0}},
    {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 1}},
};

struct GridK {
    int64_t n;
    int32_t field;  // 0 ramp, 1 radial
    int32_t brick;  // records in 8x8x8-cube brick order (else cube order)
    double pad;
};

// Record slot of cube (x, y, z): grid_layout.cuh (shared with the march).
__device__ __forceinline__ int64_t cube_slot(const GridK &G, int64_t x, int64_t y, int64_t z) {
    return tr_grid::cube_slot(G.n, G.brick != 0, x, y, z);
}

// mesh.py _ramp / _radial, then .astype(float32).astype(float64)
__device__ __forceinline__ double grid_field(const GridK &G, double x, double y, double z) {
    if (G.field == 0) return (double)__double2float_rn(x);
    const double h = (double)G.n / 2.0;
    const double d0 = x - h, d1 = y - h, d2 = z - h;
    return (double)__double2float_rn(sqrt((d0 * d0 + d1 * d1) + d2 * d2));
}

__global__ void grid_records_kernel(GridK G, const double *__restrict__ inv10, TrTetRecord *recs,
                                    uint32_t *ids) {
    __shared__ double s_inv[90];
    for (int i = threadIdx.x; i < 90; i += blockDim.x) s_inv[i] = inv10[i];
    __syncthreads();
    const int64_t n = G.n, T = 5 * n * n * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / 5;
        const int k = (int)(t - 5 * c);
        const int64_t z = c % n, y = (c / n) % n, x = c / (n * n);
        const int par = (int)((x + y + z) & 1);
        double v[4][3];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int dx = c_pattern[k][q][0];
            v[q][0] = (double)(x + (par ? 1 - dx : dx));
            v[q][1] = (double)(y + c_pattern[k][q][1]);
            v[q][2] = (double)(z + c_pattern[k][q][2]);
        }
        const double *m = s_inv + 9 * (par * 5 + k);
        const int64_t slot = 5 * cube_slot(G, x, y, z) + k;
        if (ids) ids[slot] = (uint32_t)t;
        double2 *o = reinterpret_cast<double2 *>(recs + slot);
        o[0] = make_double2(m[0], m[1]);
        o[1] = make_double2(m[2], m[3]);
        o[2] = make_double2(m[4], m[5]);
        o[3] = make_double2(m[6], m[7]);
        o[4] = make_double2(m[8], v[0][0]);
        o[5] = make_double2(v[0][1], v[0][2]);
        o[6] = make_double2(grid_field(G, v[0][0], v[0][1], v[0][2]),
                            grid_field(G, v[1][0], v[1][1], v[1][2]));
        o[7] = make_double2(grid_field(G, v[2][0], v[2][1], v[2][2]),
                            grid_field(G, v[3][0], v[3][1], v[3][2]));
    }
}

struct WalkK {
    uint32_t w[2][8];   // TrPLeaf.walk of an even / odd cube (tr_walk_table_cube)
};

__global__ void grid_leaves_kernel(GridK G, WalkK W, TrPLeaf *leaves) {
    const int64_t n = G.n, C = n * n * n;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q[3] = {c / (n * n), (c / n) % n, c % n};
        TrPLeaf L;
        for (int a = 0; a < 3; ++a) {   // inward (grid_layout.cuh, shared with the march)
            L.ex_lo[a] = __double2float_ru(tr_grid::ex_lo(q[a], n, G.pad));
            L.ex_hi[a] = __double2float_rd(tr_grid::ex_hi(q[a], n, G.pad));
        }
        L.start = (uint32_t)(5 * cube_slot(G, q[0], q[1], q[2]));
        L.count = 5u;
        const int par = (int)((q[0] + q[1] + q[2]) & 1);
        for (int k = 0; k < 8; ++k) L.walk[k] = W.w[par][k];
        leaves[c] = L;
    }
}

struct CubeBox {
    int64_t lo[3], hi[3];  // half-open cube ranges
};

__device__ __forceinline__ int64_t box_cubes(const CubeBox &b) {
    return (b.hi[0] - b.lo[0]) * (b.hi[1] - b.lo[1]) * (b.hi[2] - b.lo[2]);
}

// halve the longest cube range (first axis on ties)
__device__ __forceinline__ void split_box(const CubeBox &b, CubeBox &l, CubeBox &r) {
    int axis = 0;
    int64_t len = b.hi[0] - b.lo[0];
    for (int a = 1; a < 3; ++a)
        if (b.hi[a] - b.lo[a] > len) { len = b.hi[a] - b.lo[a]; axis = a; }
    l = b;
    r = b;
    l.hi[axis] = b.lo[axis] + len / 2;
    r.lo[axis] = l.hi[axis];
}

__global__ void grid_nodes_kernel(GridK G, int64_t n_nodes, TrPNode *nodes) {
    const int64_t n = G.n;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_nodes;
         j += (int64_t)gridDim.x * blockDim.x) {
        CubeBox b;
        for (int a = 0; a < 3; ++a) { b.lo[a] = 0; b.hi[a] = n; }
        int64_t idx = 0;
        CubeBox l, r;
        while (true) {  // the subtree rooted at idx owns node indices [idx, idx + cubes - 1)
            split_box(b, l, r);
            if (j == idx) break;
            const int64_t nl = box_cubes(l);
            if (j < idx + nl) { b = l; idx = idx + 1; }
            else { b = r; idx = idx + nl; }
        }
        TrPNode N;
        const CubeBox *ch[2] = {&l, &r};
        const int64_t nl = box_cubes(l);
        for (int c = 0; c < 2; ++c) {
            const CubeBox &cb = *ch[c];
            float *lo = c == 0 ? N.lo0 : N.lo1, *hi = c == 0 ? N.hi0 : N.hi1;
            for (int a = 0; a < 3; ++a) {   // padded tet boxes of the range, rounded outward
                lo[a] = __double2float_rd((double)cb.lo[a] - G.pad);
                hi[a] = __double2float_ru((double)cb.hi[a] + G.pad);
            }
            const int64_t first = (cb.lo[0] * n + cb.lo[1]) * n + cb.lo[2];
            N.minid[c] = (uint32_t)(5 * first);
            if (box_cubes(cb) == 1) N.child[c] = ~(int32_t)first;   // leaf = cube
            else N.child[c] = (int32_t)(c == 0 ? idx + 1 : idx + nl);
        }
        nodes[j] = N;
    }
}

// n = 1: one cube, a root node holding the single leaf
__global__ void grid_single_node_kernel(GridK G, TrPNode *nodes) {
    TrPNode N;
    for (int a = 0; a < 3; ++a) {
        N.lo0[a] = __double2float_rd(-G.pad);
        N.hi0[a] = __double2float_ru(1.0 + G.pad);
        N.lo1[a] = 1.0f;
        N.hi1[a] = 0.0f;
    }
    N.child[0] = ~0;
    N.child[1] = CHILD_NONE;
    N.minid[0] = 0;
    N.minid[1] = UINT32_MAX;
    nodes[0] = N;
}

int cuda_fail(cudaError_t e, const char *where) {
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    return tr_fail(TR_ECUDA, m.c_str());
}

unsigned grid_for(int64_t items) {
    int64_t g = (items + 255) / 256;
    if (g > 148 * 64) g = 148 * 64;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int tr_grid_scene_sizes(int64_t n, int64_t *n_tets, int64_t *n_leaves, int64_t *n_nodes) {
    if (n < 1 || n > 1024 || !n_tets || !n_leaves || !n_nodes)
        return tr_fail(TR_EINVAL, "tr_grid_scene_sizes: n must be in [1, 1024]");
    const int64_t c = n * n * n;
    if (5 * c >= (int64_t)UINT32_MAX) return tr_fail(TR_EINVAL, "tr_grid_scene_sizes: too many tets");
    *n_tets = 5 * c;
    *n_leaves = c;
    *n_nodes = c > 1 ? c - 1 : 1;
    return TR_OK;
}

int tr_grid_scene_build(int64_t n, int32_t field, double pad, const double *inv10,
                        TrTetRecord *recs, TrPLeaf *leaves, TrPNode *nodes, uint32_t *ids,
                        void *stream) {
    int64_t T, Lc, Nn;
    int rc = tr_grid_scene_sizes(n, &T, &Lc, &Nn);
    if (rc) return rc;
    if ((field != 0 && field != 1) || !(pad >= 0.0) || !inv10 || !recs || !leaves || !nodes)
        return tr_fail(TR_EINVAL, "tr_grid_scene_build: invalid arguments");
    cudaStream_t st = (cudaStream_t)stream;
    GridK G{n, field, ids != nullptr ? 1 : 0, pad};
    double *d_inv = nullptr;
    cudaError_t e = cudaMallocAsync(&d_inv, 90 * sizeof(double), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(inv10)");
    e = cudaMemcpyAsync(d_inv, inv10, 90 * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(inv10)");
    grid_records_kernel<<<grid_for(T), 256, 0, st>>>(G, d_inv, recs, ids);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "grid_records_kernel");
    WalkK W;
    tr_walk_table_cube(0, W.w[0]);
    tr_walk_table_cube(1, W.w[1]);
    grid_leaves_kernel<<<grid_for(Lc), 256, 0, st>>>(G, W, leaves);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "grid_leaves_kernel");
    if (Lc > 1) grid_nodes_kernel<<<grid_for(Nn), 256, 0, st>>>(G, Nn, nodes);
    else grid_single_node_kernel<<<1, 1, 0, st>>>(G, nodes);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "grid_nodes_kernel");
    e = cudaFreeAsync(d_inv, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync(inv10)");
    return TR_OK;
}

}  // extern "C"
