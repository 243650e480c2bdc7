// (w_l1) L1 + lam (1 - SSIM) with its analytic gradient, float32 H x W x 3 images.
//
// Reference: loss.py:48-63 (_conv_valid / _conv_adjoint: separable 11-tap Gaussian,
// sigma 1.5, valid window positions only), :80-124 (ssim, ssim_backward), :146-168
// (compute_loss; the normal / smoothness regularisers are off in every BASELINE config).
//
// Two tiled passes, each a 256-thread CTA over a 32x32 output tile with an 11-px halo
// staged in shared memory and the separable blur done as a horizontal then a vertical
// smem pass:
//   pass 1 (valid positions): blur x, y, x^2, y^2, xy -> SSIM map, its sum, and the three
//           per-position gradient maps dL/dmu_x, dL/dE[x^2], dL/dE[xy];
//   pass 2 (all pixels): adjoint blur of the three maps, combine with x, y and the L1
//           sign term into dL/dx, plus the L1 sum.

#include "vegs_common.cuh"

namespace vegs {

constexpr int kWin = 11, kHalf = 5, kLT = 32;  // window, half window, output tile
constexpr int kIn = kLT + kWin - 1;             // 42: staged input tile side

struct Taps {
    float k[kWin];
};

__device__ __forceinline__ float block_sum_f(float v, float *red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float s = 0.f;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    __syncthreads();
    return s;
}

__global__ void __launch_bounds__(256) ssim_fwd_kernel(const float *__restrict__ x, const float *__restrict__ y,
                                                       int H, int W, Taps taps, float c1, float c2, float coeff,
                                                       float *__restrict__ maps, double *sums) {
    __shared__ float sx[kIn][kIn + 1], sy[kIn][kIn + 1];
    __shared__ float hs[5][kIn][kLT + 1];
    __shared__ float red[8];
    const int Hv = H - 2 * kHalf, Wv = W - 2 * kHalf;
    const int u0 = blockIdx.y * kLT, v0 = blockIdx.x * kLT;  // valid-output tile origin
    const int64_t plane = (int64_t)Hv * Wv;
    float local = 0.f;
    for (int c = 0; c < 3; ++c) {
        __syncthreads();
        for (int i = threadIdx.x; i < kIn * kIn; i += blockDim.x) {
            const int r = i / kIn, q = i - r * kIn;
            const int gy = u0 + r, gx = v0 + q;
            const bool ok = gy < H && gx < W;
            sx[r][q] = ok ? x[((int64_t)gy * W + gx) * 3 + c] : 0.f;
            sy[r][q] = ok ? y[((int64_t)gy * W + gx) * 3 + c] : 0.f;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kIn * kLT; i += blockDim.x) {
            const int r = i / kLT, q = i - r * kLT;
            float a = 0.f, b = 0.f, aa = 0.f, bb = 0.f, ab = 0.f;
#pragma unroll
            for (int t = 0; t < kWin; ++t) {
                const float xv = sx[r][q + t], yv = sy[r][q + t], k = taps.k[t];
                a += k * xv;
                b += k * yv;
                aa += k * (xv * xv);
                bb += k * (yv * yv);
                ab += k * (xv * yv);
            }
            hs[0][r][q] = a;
            hs[1][r][q] = b;
            hs[2][r][q] = aa;
            hs[3][r][q] = bb;
            hs[4][r][q] = ab;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kLT * kLT; i += blockDim.x) {
            const int r = i / kLT, q = i - r * kLT;
            const int u = u0 + r, v = v0 + q;
            if (u >= Hv || v >= Wv) continue;
            float m[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int t = 0; t < kWin; ++t) {
                const float k = taps.k[t];
#pragma unroll
                for (int e = 0; e < 5; ++e) m[e] += k * hs[e][r + t][q];
            }
            const float mux = m[0], muy = m[1];
            const float sxx = m[2] - mux * mux, syy = m[3] - muy * muy, sxy = m[4] - mux * muy;
            const float a1 = 2.f * mux * muy + c1, b1 = mux * mux + muy * muy + c1;
            const float a2 = 2.f * sxy + c2, b2 = sxx + syy + c2;
            const float inv = 1.f / (b1 * b2);
            const float smap = (a1 * a2) * inv;
            local += smap;
            const float g_mu = coeff * (2.f * muy * a2 * inv - 2.f * mux * smap / b1 - 2.f * muy * a1 * inv +
                                        2.f * mux * smap / b2);
            const float g_xx = coeff * (-smap / b2);
            const float g_xy = coeff * (2.f * a1 * inv);
            const int64_t o = (int64_t)c * plane + (int64_t)u * Wv + v;
            maps[o] = g_mu;
            maps[3 * plane + o] = g_xx;
            maps[6 * plane + o] = g_xy;
        }
    }
    const float tot = block_sum_f(local, red);
    if (threadIdx.x == 0) atomicAdd(sums + 1, (double)tot);
}

__global__ void __launch_bounds__(256) ssim_bwd_kernel(const float *__restrict__ x, const float *__restrict__ y,
                                                       int H, int W, Taps taps, float l1_coeff,
                                                       const float *__restrict__ maps, float *__restrict__ dx,
                                                       double *sums) {
    __shared__ float sm[3][kIn][kIn + 1];
    __shared__ float hs[3][kIn][kLT + 1];
    __shared__ float red[8];
    const int Hv = H - 2 * kHalf, Wv = W - 2 * kHalf;
    const int i0 = blockIdx.y * kLT, j0 = blockIdx.x * kLT;  // full-image tile origin
    const int64_t plane = (int64_t)Hv * Wv;
    float l1 = 0.f;
    for (int c = 0; c < 3; ++c) {
        __syncthreads();
        for (int i = threadIdx.x; i < kIn * kIn; i += blockDim.x) {
            const int r = i / kIn, q = i - r * kIn;
            const int u = i0 - 2 * kHalf + r, v = j0 - 2 * kHalf + q;  // valid-map coordinates
            const bool ok = u >= 0 && v >= 0 && u < Hv && v < Wv;
            const int64_t o = (int64_t)c * plane + (int64_t)u * Wv + v;
            sm[0][r][q] = ok ? maps[o] : 0.f;
            sm[1][r][q] = ok ? maps[3 * plane + o] : 0.f;
            sm[2][r][q] = ok ? maps[6 * plane + o] : 0.f;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kIn * kLT; i += blockDim.x) {
            const int r = i / kLT, q = i - r * kLT;
            float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int t = 0; t < kWin; ++t) {
                const float k = taps.k[kWin - 1 - t];
#pragma unroll
                for (int e = 0; e < 3; ++e) acc[e] += k * sm[e][r][q + t];
            }
#pragma unroll
            for (int e = 0; e < 3; ++e) hs[e][r][q] = acc[e];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kLT * kLT; i += blockDim.x) {
            const int r = i / kLT, q = i - r * kLT;
            const int gi = i0 + r, gj = j0 + q;
            if (gi >= H || gj >= W) continue;
            float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int t = 0; t < kWin; ++t) {
                const float k = taps.k[kWin - 1 - t];
#pragma unroll
                for (int e = 0; e < 3; ++e) acc[e] += k * hs[e][r + t][q];
            }
            const int64_t p = ((int64_t)gi * W + gj) * 3 + c;
            const float xv = x[p], yv = y[p];
            const float d = xv - yv;
            l1 += fabsf(d);
            const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
            dx[p] = l1_coeff * sgn + acc[0] + 2.f * xv * acc[1] + yv * acc[2];
        }
    }
    const float tot = block_sum_f(l1, red);
    if (threadIdx.x == 0) atomicAdd(sums, (double)tot);
}

}  // namespace vegs

using namespace vegs;

extern "C" int vegs_loss_l1_ssim(const float *x, const float *y, int32_t height, int32_t width, double w_l1,
                                 double lam, float *d_x, double *sums, void *ws, size_t *ws_bytes, void *stream) {
    if (!ws_bytes || height < kWin || width < kWin) return VEGS_ERR_ARG;
    const int64_t Hv = height - 2 * kHalf, Wv = width - 2 * kHalf;
    const size_t need = sizeof(float) * 9 * (size_t)(Hv * Wv);
    if (!ws) {
        *ws_bytes = need;
        return VEGS_OK;
    }
    if (*ws_bytes < need) return VEGS_ERR_CAPACITY;
    if (!x || !y || !d_x || !sums) return VEGS_ERR_ARG;
    // float32 taps exactly as loss.py:39-45 builds them for float32 images
    Taps taps;
    double g[kWin], gs = 0.0;
    for (int t = 0; t < kWin; ++t) {
        const double xs = t - (kWin - 1) / 2.0;
        g[t] = exp(-0.5 * (xs / 1.5) * (xs / 1.5));
        gs += g[t];
    }
    for (int t = 0; t < kWin; ++t) taps.k[t] = (float)(g[t] / gs);
    const float c1 = 0.01f * 0.01f, c2 = 0.03f * 0.03f;
    const double n_pos = (double)Hv * (double)Wv * 3.0;
    const float coeff = (float)(-lam / n_pos);
    const float l1c = (float)(w_l1 / ((double)height * width * 3.0));
    cudaStream_t s = (cudaStream_t)stream;
    dim3 g1((unsigned)((Wv + kLT - 1) / kLT), (unsigned)((Hv + kLT - 1) / kLT));
    ssim_fwd_kernel<<<g1, 256, 0, s>>>(x, y, height, width, taps, c1, c2, coeff, (float *)ws, sums);
    VEGS_CHECK_LAUNCH();
    dim3 g2((unsigned)((width + kLT - 1) / kLT), (unsigned)((height + kLT - 1) / kLT));
    ssim_bwd_kernel<<<g2, 256, 0, s>>>(x, y, height, width, taps, l1c, (const float *)ws, d_x, sums);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" const char *vegs_version(void) { return "vegsplat_b200 0.1 sm_100a"; }
