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

// The cube's exclusive box on one axis before f32 rounding (inward): the
// cube shrunk by the box pad, reaching out by the pad at the grid's faces.
__host__ __device__ __forceinline__ double ex_lo(int64_t c, int64_t n, double pad) {
    return (c == 0) ? -pad : (double)c + pad;
}
__host__ __device__ __forceinline__ double ex_hi(int64_t c, int64_t n, double pad) {
    return (c == n - 1) ? (double)n + pad : (double)(c + 1) - pad;
}

}  // namespace tr_grid
