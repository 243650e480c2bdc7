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

#ifndef VEGS_SSIM_TILE
#define VEGS_SSIM_TILE 32
#endif
#ifndef VEGS_SSIM_T
#define VEGS_SSIM_T 256
#endif
constexpr int kWin = 11, kHalf = 5, kLT = VEGS_SSIM_TILE;  // window, half window, output tile
constexpr int kIn = kLT + kWin - 1;                         // staged input tile side
#ifndef VEGS_SSIM_RB
#define VEGS_SSIM_RB 4
#endif
constexpr int kRB = VEGS_SSIM_RB;  // outputs per thread in each blur pass (register blocking)
static_assert(kLT % kRB == 0, "register blocks tile the output");

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

#ifndef VEGS_SSIM_FWD_MINB
#define VEGS_SSIM_FWD_MINB 3  // 80 registers (a 48-byte spill), 3 CTAs per SM: loss 0.133 -> 0.100 ms per c2 view (4: 0.101)
#endif
__global__ void __launch_bounds__(VEGS_SSIM_T, VEGS_SSIM_FWD_MINB) ssim_fwd_kernel(const float *__restrict__ x, const float *__restrict__ y,
                                                       int H, int W, int xs, Taps taps, float c1, float c2,
                                                       float coeff, float *__restrict__ maps, double *sums) {
    // (x, y) pairs interleaved so the two blurs of x and y (and of x^2, y^2) run as packed
    // FFMA2 on one LDS.64 per tap; x*y is blurred alone
    __shared__ float2 sxy[kIn][kIn + 1];
    __shared__ float2 h01[kIn][kLT + 1], h23[kIn][kLT + 1];
    __shared__ float h4[kIn][kLT + 1];
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
            sxy[r][q] = ok ? make_float2(x[((int64_t)gy * W + gx) * xs + c], y[((int64_t)gy * W + gx) * 3 + c])
                           : make_float2(0.f, 0.f);
        }
        __syncthreads();
        // horizontal pass, register-blocked: one thread, kRB consecutive outputs of a row,
        // each staged value (and its squares / cross product) loaded and formed once
        for (int i = threadIdx.x; i < kIn * (kLT / kRB); i += blockDim.x) {
            const int r = i / (kLT / kRB), q0 = (i - r * (kLT / kRB)) * kRB;
            float2 v[kWin + kRB - 1], sq[kWin + kRB - 1];
            float pr[kWin + kRB - 1];
#pragma unroll
            for (int t = 0; t < kWin + kRB - 1; ++t) {
                v[t] = sxy[r][q0 + t];
                sq[t] = __fmul2_rn(v[t], v[t]);
                pr[t] = v[t].x * v[t].y;
            }
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
                float2 m01 = make_float2(0.f, 0.f), m23 = make_float2(0.f, 0.f);
                float m4 = 0.f;
#pragma unroll
                for (int t = 0; t < kWin; ++t) {
                    const float2 k = make_float2(taps.k[t], taps.k[t]);
                    m01 = __ffma2_rn(k, v[o + t], m01);
                    m23 = __ffma2_rn(k, sq[o + t], m23);
                    m4 += taps.k[t] * pr[o + t];
                }
                h01[r][q0 + o] = m01;
                h23[r][q0 + o] = m23;
                h4[r][q0 + o] = m4;
            }
        }
        __syncthreads();
        // vertical pass, register-blocked: one thread, kRB consecutive rows of a column
        for (int i = threadIdx.x; i < (kLT / kRB) * kLT; i += blockDim.x) {
            const int r0 = (i / kLT) * kRB, q = i - (i / kLT) * kLT;
            float2 a01[kWin + kRB - 1], a23[kWin + kRB - 1];
            float a4[kWin + kRB - 1];
#pragma unroll
            for (int t = 0; t < kWin + kRB - 1; ++t) {
                a01[t] = h01[r0 + t][q];
                a23[t] = h23[r0 + t][q];
                a4[t] = h4[r0 + t][q];
            }
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
            const int r = r0 + o;
            const int u = u0 + r, v = v0 + q;
            if (u >= Hv || v >= Wv) continue;
            float2 m01 = make_float2(0.f, 0.f), m23 = make_float2(0.f, 0.f);
            float m4 = 0.f;
#pragma unroll
            for (int t = 0; t < kWin; ++t) {
                const float2 k = make_float2(taps.k[t], taps.k[t]);
                m01 = __ffma2_rn(k, a01[o + t], m01);
                m23 = __ffma2_rn(k, a23[o + t], m23);
                m4 += taps.k[t] * a4[o + t];
            }
            const float mux = m01.x, muy = m01.y;
            const float sxx = m23.x - mux * mux, syy = m23.y - muy * muy, sxy_ = m4 - mux * muy;
            const float a1 = 2.f * mux * muy + c1, b1 = mux * mux + muy * muy + c1;
            const float a2 = 2.f * sxy_ + c2, b2 = sxx + syy + c2;
            const float inv = 1.f / (b1 * b2);
            const float smap = (a1 * a2) * inv;
            local += smap;
            const float g_mu = coeff * (2.f * muy * a2 * inv - 2.f * mux * smap / b1 - 2.f * muy * a1 * inv +
                                        2.f * mux * smap / b2);
            const float g_xx = coeff * (-smap / b2);
            const float g_xy = coeff * (2.f * a1 * inv);
            const int64_t oo = (int64_t)c * plane + (int64_t)u * Wv + v;
            maps[oo] = g_mu;
            maps[3 * plane + oo] = g_xx;
            maps[6 * plane + oo] = g_xy;
            }
        }
    }
    const float tot = block_sum_f(local, red);
    if (threadIdx.x == 0) atomicAdd(sums + 1, (double)tot);
}

__global__ void __launch_bounds__(VEGS_SSIM_T) ssim_bwd_kernel(const float *__restrict__ x, const float *__restrict__ y,
                                                       int H, int W, int xs, Taps taps, float l1_coeff,
                                                       const float *__restrict__ maps, float *__restrict__ dx,
                                                       double *sums) {
    __shared__ float2 sm01[kIn][kIn + 1];  // maps 0 and 1 interleaved (packed FFMA2 blurs)
    __shared__ float sm2[kIn][kIn + 1];
    __shared__ float2 hs01[kIn][kLT + 1];
    __shared__ float hs2[kIn][kLT + 1];
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
            sm01[r][q] = ok ? make_float2(maps[o], maps[3 * plane + o]) : make_float2(0.f, 0.f);
            sm2[r][q] = ok ? maps[6 * plane + o] : 0.f;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kIn * (kLT / kRB); i += blockDim.x) {  // register-blocked, as in the forward
            const int r = i / (kLT / kRB), q0 = (i - r * (kLT / kRB)) * kRB;
            float2 w01[kWin + kRB - 1];
            float w2[kWin + kRB - 1];
#pragma unroll
            for (int t = 0; t < kWin + kRB - 1; ++t) {
                w01[t] = sm01[r][q0 + t];
                w2[t] = sm2[r][q0 + t];
            }
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
                float2 a01 = make_float2(0.f, 0.f);
                float a2 = 0.f;
#pragma unroll
                for (int t = 0; t < kWin; ++t) {
                    const float k = taps.k[kWin - 1 - t];
                    a01 = __ffma2_rn(make_float2(k, k), w01[o + t], a01);
                    a2 += k * w2[o + t];
                }
                hs01[r][q0 + o] = a01;
                hs2[r][q0 + o] = a2;
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < (kLT / kRB) * kLT; i += blockDim.x) {
            const int r0 = (i / kLT) * kRB, q = i - (i / kLT) * kLT;
            float2 w01[kWin + kRB - 1];
            float w2[kWin + kRB - 1];
#pragma unroll
            for (int t = 0; t < kWin + kRB - 1; ++t) {
                w01[t] = hs01[r0 + t][q];
                w2[t] = hs2[r0 + t][q];
            }
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
            const int r = r0 + o;
            const int gi = i0 + r, gj = j0 + q;
            if (gi >= H || gj >= W) continue;
            float2 a01 = make_float2(0.f, 0.f);
            float a2 = 0.f;
#pragma unroll
            for (int t = 0; t < kWin; ++t) {
                const float k = taps.k[kWin - 1 - t];
                a01 = __ffma2_rn(make_float2(k, k), w01[o + t], a01);
                a2 += k * w2[o + t];
            }
            const float acc[3] = {a01.x, a01.y, a2};
            const int64_t pix = (int64_t)gi * W + gj;
            const int64_t p = pix * xs + c;
            const float xv = x[p], yv = y[pix * 3 + c];
            const float d = xv - yv;
            l1 += fabsf(d);
            const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
            dx[p] = l1_coeff * sgn + acc[0] + 2.f * xv * acc[1] + yv * acc[2];
            }
        }
    }
    const float tot = block_sum_f(l1, red);
    if (threadIdx.x == 0) atomicAdd(sums, (double)tot);
}

}  // namespace vegs

using namespace vegs;

extern "C" int vegs_loss_l1_ssim(const float *x, const float *y, int32_t height, int32_t width, int32_t x_stride,
                                 double w_l1, double lam, float *d_x, double *sums, void *ws, size_t *ws_bytes,
                                 void *stream) {
    if (!ws_bytes || height < kWin || width < kWin || x_stride < 3) return VEGS_ERR_ARG;
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
    ssim_fwd_kernel<<<g1, VEGS_SSIM_T, 0, s>>>(x, y, height, width, x_stride, taps, c1, c2, coeff, (float *)ws, sums);
    VEGS_CHECK_LAUNCH();
    dim3 g2((unsigned)((width + kLT - 1) / kLT), (unsigned)((height + kLT - 1) / kLT));
    ssim_bwd_kernel<<<g2, VEGS_SSIM_T, 0, s>>>(x, y, height, width, x_stride, taps, l1c, (const float *)ws, d_x, sums);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

// ---- auxiliary-plane regularisers (loss.py:175-240) -------------------------------------
// planes: (H, W, 11) = rgb, depth, normal(3), attrs(4); alpha = 1 - T.  Normal consistency
// compares the blended normal with a depth-derived pseudo-normal on interior pixels with
// alpha > 0.5 (mask detached); bilateral smoothness penalises attr-plane differences
// weighted by exp(-|d ref_gray|).  sums += {normal sum (1-dot), mask count, smooth sum}.

namespace vegs {

__device__ __forceinline__ bool normal_mask(const float *T, int H, int W, int y, int x) {
    return y > 0 && x > 0 && y < H - 1 && x < W - 1 && (1.f - T[(int64_t)y * W + x]) > 0.5f;
}

__global__ void normal_count_kernel(const float *T, int H, int W, double *sums) {
    __shared__ float red[8];
    float c = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)H * W;
         i += (int64_t)gridDim.x * blockDim.x)
        c += normal_mask(T, H, W, (int)(i / W), (int)(i % W)) ? 1.f : 0.f;
    const float tot = block_sum_f(c, red);
    if (threadIdx.x == 0) atomicAdd(sums + 1, (double)tot);
}

// per pixel: d normal, the normal term, and g_nd_raw (3 floats) for the depth gather
__global__ void normal_pass_kernel(const float *P, const float *T, int H, int W, float px_scale, float w_n,
                                   double *sums, float *g_raw, float *dP) {
    __shared__ float red[8];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float term = 0.f;
    if (i < (int64_t)H * W) {
        const int y = (int)(i / W), x = (int)(i % W);
        float g3[3] = {0.f, 0.f, 0.f};
        float dn[3] = {0.f, 0.f, 0.f};
        if (normal_mask(T, H, W, y, x)) {
            const float cnt = (float)sums[1];
            const float *p = P + i * 11;
            const float gx = 0.5f * (P[(i + 1) * 11 + 3] - P[(i - 1) * 11 + 3]);
            const float gy = 0.5f * (P[(i + W) * 11 + 3] - P[(i - W) * 11 + 3]);
            const float nd[3] = {-gx, -gy, px_scale * p[3]};
            const float ndl = fmaxf(sqrtf(nd[0] * nd[0] + nd[1] * nd[1] + nd[2] * nd[2]), 1e-12f);
            const float nrl = fmaxf(sqrtf(p[4] * p[4] + p[5] * p[5] + p[6] * p[6]), 1e-12f);
            float ndh[3], nrh[3], dot = 0.f;
            for (int k = 0; k < 3; ++k) {
                ndh[k] = nd[k] / ndl;
                nrh[k] = p[4 + k] / nrl;
                dot += nrh[k] * ndh[k];
            }
            term = 1.f - dot;
            const float sc = -w_n / cnt;
            float pr = 0.f, pd = 0.f;
            for (int k = 0; k < 3; ++k) {
                pr += sc * ndh[k] * nrh[k];
                pd += sc * nrh[k] * ndh[k];
            }
            for (int k = 0; k < 3; ++k) {
                dn[k] = (sc * ndh[k] - pr * nrh[k]) / nrl;
                g3[k] = (sc * nrh[k] - pd * ndh[k]) / ndl;
            }
        }
        for (int k = 0; k < 3; ++k) {
            g_raw[i * 3 + k] = g3[k];
            dP[i * 11 + 4 + k] = dn[k];
        }
    }
    const float tot = block_sum_f(term, red);
    if (threadIdx.x == 0) atomicAdd(sums, (double)tot);
}

__device__ __forceinline__ float gray(const float *ref, int64_t i) {
    return (fabsf(ref[i * 3]) + fabsf(ref[i * 3 + 1]) + fabsf(ref[i * 3 + 2])) / 3.f;
}

// depth gradient (gather of the neighbours' pseudo-normal terms) + attr smoothness
__global__ void aux_gather_kernel(const float *P, const float *ref, const float *g_raw, int H, int W, float px_scale,
                                  float w_s, int smooth, float *dP, double *sums) {
    __shared__ float red[8];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    if (i < (int64_t)H * W) {
        const int y = (int)(i / W), x = (int)(i % W);
        // nd_raw = (-gx, -gy, s z): d z[y,x] = s g_z + 0.5 (g_gx(x-1) - g_gx(x+1) + g_gy(y-1) - g_gy(y+1)),
        // g_gx = -g_raw_x, g_gy = -g_raw_y
        float dz = px_scale * g_raw[i * 3 + 2];
        if (x > 0) dz += -0.5f * g_raw[(i - 1) * 3 + 0];
        if (x < W - 1) dz -= -0.5f * g_raw[(i + 1) * 3 + 0];
        if (y > 0) dz += -0.5f * g_raw[(i - W) * 3 + 1];
        if (y < H - 1) dz -= -0.5f * g_raw[(i + W) * 3 + 1];
        dP[i * 11 + 3] = dz;
        float da[4] = {0.f, 0.f, 0.f, 0.f};
        if (smooth) {
            const float n_terms = 4.f * ((float)H * (W - 1) + (float)(H - 1) * W);
            const float g0 = gray(ref, i);
            const float ex_r = x < W - 1 ? expf(-fabsf(gray(ref, i + 1) - g0)) : 0.f;   // edge (x, x+1)
            const float ex_l = x > 0 ? expf(-fabsf(g0 - gray(ref, i - 1))) : 0.f;       // edge (x-1, x)
            const float ey_d = y < H - 1 ? expf(-fabsf(gray(ref, i + W) - g0)) : 0.f;   // edge (y, y+1)
            const float ey_u = y > 0 ? expf(-fabsf(g0 - gray(ref, i - W))) : 0.f;       // edge (y-1, y)
            for (int k = 0; k < 4; ++k) {
                const float a0 = P[i * 11 + 7 + k];
                if (x < W - 1) {
                    const float d = P[(i + 1) * 11 + 7 + k] - a0;
                    acc += fabsf(d) * ex_r;
                    da[k] -= w_s * (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * ex_r / n_terms;
                }
                if (x > 0) {
                    const float d = a0 - P[(i - 1) * 11 + 7 + k];
                    da[k] += w_s * (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * ex_l / n_terms;
                }
                if (y < H - 1) {
                    const float d = P[(i + W) * 11 + 7 + k] - a0;
                    acc += fabsf(d) * ey_d;
                    da[k] -= w_s * (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * ey_d / n_terms;
                }
                if (y > 0) {
                    const float d = a0 - P[(i - W) * 11 + 7 + k];
                    da[k] += w_s * (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * ey_u / n_terms;
                }
            }
        }
        for (int k = 0; k < 4; ++k) dP[i * 11 + 7 + k] = da[k];
    }
    const float tot = block_sum_f(acc, red);
    if (threadIdx.x == 0) atomicAdd(sums + 2, (double)tot);
}

}  // namespace vegs

extern "C" int vegs_loss_aux(const float *planes, const float *out_t, const float *ref_rgb, int32_t height,
                             int32_t width, double px_scale, double w_normal, double w_smooth, float *d_planes,
                             double *sums, void *ws, size_t *ws_bytes, void *stream) {
    if (!ws_bytes || height < 3 || width < 3) return VEGS_ERR_ARG;
    const int64_t hw = (int64_t)height * width;
    const size_t need = sizeof(float) * 3 * (size_t)hw;
    if (!ws) {
        *ws_bytes = need;
        return VEGS_OK;
    }
    if (*ws_bytes < need) return VEGS_ERR_CAPACITY;
    if (!planes || !out_t || !ref_rgb || !d_planes || !sums) return VEGS_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = (int)((hw + 255) / 256);
    float *g_raw = (float *)ws;
    if (w_normal > 0.0) {
        normal_count_kernel<<<148 * 4, 256, 0, s>>>(out_t, height, width, sums);
        VEGS_CHECK_LAUNCH();
        normal_pass_kernel<<<blocks, 256, 0, s>>>(planes, out_t, height, width, (float)px_scale, (float)w_normal,
                                                  sums, g_raw, d_planes);
    } else {
        VEGS_CUDA(cudaMemsetAsync(g_raw, 0, need, s));
    }
    VEGS_CHECK_LAUNCH();
    aux_gather_kernel<<<blocks, 256, 0, s>>>(planes, ref_rgb, g_raw, height, width, (float)px_scale, (float)w_smooth,
                                             w_smooth > 0.0 ? 1 : 0, d_planes, sums);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" const char *vegs_version(void) { return "vegsplat_b200 0.1 sm_100a"; }
