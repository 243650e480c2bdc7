// Shared device helpers for the vegsplat_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "vegsplat_b200.h"

#define VEGS_CHECK_LAUNCH()                                            \
    do {                                                               \
        cudaError_t e_ = cudaGetLastError();                           \
        if (e_ != cudaSuccess) return VEGS_ERR_CUDA;                   \
    } while (0)

#define VEGS_CUDA(call)                                                \
    do {                                                               \
        if ((call) != cudaSuccess) return VEGS_ERR_CUDA;               \
    } while (0)

namespace vegs {

constexpr int kTile = 16;            // pixels per tile side (RasterSettings.tile_size)
constexpr int kTileThreads = kTile * kTile;
constexpr double kBetaMin = 1.0, kBetaMax = 128.0;

__host__ __device__ inline int rec_stride(int n_ch) { return ((7 + n_ch) + 3) & ~3; }
__host__ __device__ inline int row_width(int n_ch) { return 6 + n_ch; }
constexpr int kProjStride = 8;  // float64 per Gaussian in a vegs_project table

// Class-major parameter layout (model.py FIELD_LAYOUT): element offsets for n Gaussians.
struct ParamView {
    const double *pos, *log_scale, *rot, *raw_value, *raw_weight, *normal, *raw_ka, *raw_kd,
        *raw_ks, *raw_beta;
    __host__ __device__ ParamView(const double *p, int64_t n)
        : pos(p), log_scale(p + 3 * n), rot(p + 6 * n), raw_value(p + 10 * n),
          raw_weight(p + 11 * n), normal(p + 12 * n), raw_ka(p + 15 * n), raw_kd(p + 16 * n),
          raw_ks(p + 17 * n), raw_beta(p + 18 * n) {}
};

struct GradView {
    double *pos, *log_scale, *rot, *raw_value, *raw_weight, *normal, *raw_ka, *raw_kd, *raw_ks,
        *raw_beta;
    __host__ __device__ GradView(double *p, int64_t n)
        : pos(p), log_scale(p + 3 * n), rot(p + 6 * n), raw_value(p + 10 * n),
          raw_weight(p + 11 * n), normal(p + 12 * n), raw_ka(p + 15 * n), raw_kd(p + 16 * n),
          raw_ks(p + 17 * n), raw_beta(p + 18 * n) {}
};

// Pixel owned by thread `tid` of a 256-thread tile CTA: each warp covers an 8x4 block
// (2 x 4 warps), so rect culling and early exit act on compact pixel groups.
__device__ __forceinline__ void tile_pixel(int tid, int &lx, int &ly) {
    const int warp = tid >> 5, lane = tid & 31;
    lx = (warp & 1) * 8 + (lane & 7);
    ly = (warp >> 1) * 4 + (lane >> 3);
}

// Duplicate-order index of a splat's instance in tile (tx, ty): the splat's first index
// (exclusive scan of tile counts) plus the tile's row-major position inside the splat's
// tile rectangle (pipeline.py:174-187).  rect = (x0, x1, y0, y1) in pixels, clipped.
__device__ __forceinline__ int64_t dup_index(int64_t first, int4 r, int tx, int ty) {
    const int x0 = r.x / kTile, y0 = r.z / kTile, nx = (r.y - 1) / kTile - x0 + 1;
    return first + (int64_t)(ty - y0) * nx + (tx - x0);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace vegs
