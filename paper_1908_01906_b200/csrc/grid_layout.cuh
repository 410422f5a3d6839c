// grid_layout.cuh -- the analytic layout of tr_grid_scene_build's scenes
// (csrc/synth.cu), shared by the generator and the march kernels, which
// locate a sample's leaf and records from its cube coordinates instead of
// loading a leaf header (render.cu, shade_sample).
#pragma once
#include <cstdint>

namespace tr_grid {

constexpr int64_t BRICK = 8;   // 8^3-cube bricks of records

// Record slot of cube (x, y, z) of an n^3 grid: cube-major, or brick-major
// with the cubes of a brick (8^3, clipped at the far faces) in x, y, z
// order -- dense, so the 5 records of cube c start at 5 * cube_slot(c).
__host__ __device__ __forceinline__ int64_t cube_slot(int64_t n, bool brick, int64_t x, int64_t y,
                                                      int64_t z) {
    if (!brick) return (x * n + y) * n + z;
    const int64_t bx = x / BRICK, by = y / BRICK, bz = z / BRICK;
    const int64_t sx = n - bx * BRICK < BRICK ? n - bx * BRICK : BRICK;
    const int64_t sy = n - by * BRICK < BRICK ? n - by * BRICK : BRICK;
    const int64_t sz = n - bz * BRICK < BRICK ? n - bz * BRICK : BRICK;
    const int64_t before = BRICK * bx * n * n + sx * BRICK * by * n + sx * sy * BRICK * bz;
    return before + ((x - bx * BRICK) * sy + (y - by * BRICK)) * sz + (z - bz * BRICK);
}

// 32-bit cube_slot for the march (n <= 1024 and 5 n^3 < 2^32, checked by
// tr_grid_scene_sizes, so every value fits).
__host__ __device__ __forceinline__ uint32_t cube_slot32(uint32_t n, bool brick, uint32_t x, uint32_t y,
                                                         uint32_t z) {
    if (!brick) return (x * n + y) * n + z;
    const uint32_t b = (uint32_t)BRICK;
    const uint32_t bx = x / b, by = y / b, bz = z / b;
    const uint32_t sx = n - bx * b < b ? n - bx * b : b;
    const uint32_t sy = n - by * b < b ? n - by * b : b;
    const uint32_t sz = n - bz * b < b ? n - bz * b : b;
    const uint32_t before = b * bx * n * n + sx * b * by * n + sx * sy * b * bz;
    return before + ((x - bx * b) * sy + (y - by * b)) * sz + (z - bz * b);
}

// The cube's exclusive box on one axis before f32 rounding (inward): the
// cube shrunk by the box pad, reaching out by the pad at the grid's faces.
// In f64 these are exactly the neighbouring cubes' padded tet box faces
// (fl(c + pad), fl((c + 1) - pad): mesh.py:249-250 computes them the same
// way), so the open interval between them meets no other cube's padded tet
// box -- the march tests against them directly.
__host__ __device__ __forceinline__ double ex_lo(int64_t c, int64_t n, double pad) {
    return (c == 0) ? -pad : (double)c + pad;
}
__host__ __device__ __forceinline__ double ex_hi(int64_t c, int64_t n, double pad) {
    return (c == n - 1) ? (double)n + pad : (double)(c + 1) - pad;
}

}  // namespace tr_grid
