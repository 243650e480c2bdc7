// Per-Gaussian backward for sm_100a: float64 reduction of the per-instance rows, then the
// projection and shading adjoints (projection.py:186-277, shading.py:97-176,
// pipeline.py:307-366).  Compiled WITH float64 FMA contraction: nothing here feeds an
// integer decision (the kept set and tile counts come from the forward), and the
// gradients are held to 1e-4 of the reference, so the -fmad=false rounding of the forward
// unit (preprocess.cu) buys nothing here and costs ~a quarter of the FP64 instructions.

#include <math.h>
#include <stdlib.h>

#include "preprocess_common.cuh"

#ifndef VEGS_PBWD_T
#define VEGS_PBWD_T 256
#endif
#ifndef VEGS_PBWD_MINB
#define VEGS_PBWD_MINB (1024 / VEGS_PBWD_T)  // 64 registers: 1024 resident threads per SM
#endif

namespace vegs {

// ---------------------------------------------------------------------------------
// Backward, part 1: the sum of each kept Gaussian's instance rows, in duplicate order
// (== sorted-instance order per splat, the order np.add.at applies at pipeline.py:313-316).
// A lean kernel (few registers, full occupancy, 16-byte loads); the visited bitmask
// (L2-resident, one bit per instance) means only the ~30% of rows a pixel actually
// blended are read.  The register-heavy chain runs separately.

#ifndef VEGS_RR_T
#define VEGS_RR_T 64  // small CTAs: the per-Gaussian walks are uneven (3.5 active lanes per warp)
#endif
template <typename Real, int NV>
__device__ __forceinline__ void reduce_rows_one(const uint32_t *tiles, const int64_t *offsets, const Real *rows,
                                                const uint32_t *visited, double *sums, int64_t g);

template <typename Real, int NV>
__global__ void __launch_bounds__(VEGS_RR_T) reduce_rows_kernel(const uint32_t *tiles, const int64_t *offsets,
                                                          const Real *rows, int64_t n, const uint32_t *visited,
                                                          double *sums) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    reduce_rows_one<Real, NV>(tiles, offsets, rows, visited, sums, g);
}

// the same over a compacted list of the kept Gaussians (count on the device)
template <typename Real, int NV>
__global__ void __launch_bounds__(VEGS_RR_T) reduce_rows_list_kernel(const uint32_t *tiles, const int64_t *offsets,
                                                               const Real *rows, const int32_t *list,
                                                               const int32_t *count, const uint32_t *visited,
                                                               double *sums) {
    const int m = *count;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        reduce_rows_one<Real, NV>(tiles, offsets, rows, visited, sums, list[i]);
}

template <typename Real, int NV>
__device__ __forceinline__ void reduce_rows_one(const uint32_t *tiles, const int64_t *offsets, const Real *rows,
                                                const uint32_t *visited, double *sums, int64_t g) {
    const uint32_t cnt = tiles[g];
    if (cnt == 0) return;
    constexpr int RS = ((7 + (NV - 6)) + 3) & ~3;
    constexpr int NF4 = (int)(RS * sizeof(Real) / 16);
    // float32 rows (float32 blends) are summed in float32 and widened once per Gaussian: a
    // Gaussian has ~3 visited rows (<= ~50), so the sum is within ~1e-6 of the float64 one,
    // and the per-row float -> double conversions (XU pipe, 71% busy) are gone
    using Acc = Real;
    Acc acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = (Acc)0;
    // ascending duplicate-order index; only rows whose visited bit is set were written
    const int64_t p0 = offsets[g], pend = p0 + cnt;
    for (int64_t p = p0; p < pend;) {
        const uint32_t sh = (uint32_t)(p & 31);
        const int64_t span = (32 - sh) < (pend - p) ? (32 - sh) : (pend - p);
        uint32_t w = __ldg(visited + (p >> 5)) >> sh;
        if (span < 32) w &= (1u << span) - 1u;
        while (w) {  // up to 4 visited rows in flight per round, summed in ascending order
#ifndef VEGS_RR_Q11
#define VEGS_RR_Q11 4
#endif
            // rows in flight: VEGS_RR_Q3 rgb float32 rows, VEGS_RR_Q11 aux float32 rows, 1 float64 row
#ifndef VEGS_RR_Q3
#define VEGS_RR_Q3 3
#endif
            constexpr int Q = RS * sizeof(Real) <= 48 ? VEGS_RR_Q3 : (RS * sizeof(Real) <= 80 ? VEGS_RR_Q11 : 1);
            int b[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                b[q] = w ? __ffs(w) - 1 : -1;
                w &= w - 1;
            }
            Real row[Q][RS];
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (b[q] >= 0) {
                    const float4 *src = reinterpret_cast<const float4 *>(rows + (int64_t)RS * (p + b[q]));
#pragma unroll
                    for (int k = 0; k < NF4; ++k) reinterpret_cast<float4 *>(row[q])[k] = __ldg(src + k);
                }
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (b[q] >= 0) {
#pragma unroll
                    for (int k = 0; k < NV; ++k) acc[k] = acc[k] + row[q][k];
                }
        }
        p += span;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) sums[(int64_t)NV * g + k] = (double)acc[k];
}

// Backward, part 2: projection and shading adjoints per Gaussian (float64).

__global__ void __launch_bounds__(VEGS_PBWD_T, VEGS_PBWD_MINB) preprocess_bwd_kernel(
    const double *params, int64_t n, VegsCamera cam, VegsTF tf, VegsSettings st, int n_ch,
    const uint32_t *tiles, const double *sums, double scale, int accumulate,
    double *grads, double *vs_norm, uint8_t *visible_out, double *dstats) {
    extern __shared__ double tf_smem[];
    const TFTable tab = stage_tf(tf, tf_smem);
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    GradView G(grads, n);
    const uint32_t cnt = tiles[g];
    if (cnt == 0) {
        if (!accumulate) {
            for (int k = 0; k < 3; ++k) G.pos[3 * g + k] = 0.0, G.log_scale[3 * g + k] = 0.0,
                                         G.normal[3 * g + k] = 0.0;
            for (int k = 0; k < 4; ++k) G.rot[4 * g + k] = 0.0;
            G.raw_value[g] = G.raw_weight[g] = G.raw_ka[g] = G.raw_kd[g] = G.raw_ks[g] =
                G.raw_beta[g] = 0.0;
        }
        if (vs_norm) vs_norm[g] = 0.0;
        if (visible_out) visible_out[g] = 0;
        return;
    }
    const double *red = sums + (int64_t)row_width(n_ch) * g;  // reduce_rows_kernel output
    const double gmx = red[0], gmy = red[1];
    const double d_con[3] = {red[2], red[3], red[4]};
    const double d_ab = red[5];
    const double *d_ch = red + 6;

    const ParamView P(params, n);
#define VEGS_PUT(dst, val) (dst) = accumulate ? (dst) + scale * (val) : scale * (val)
    // projection adjoint first, its outputs written out before the shading recompute so
    // the two halves' working sets are never live together
    double gpos[3];
    {
    Projected p;
    project_one<false>(P, g, 0.0, cam, st, p);
    const double *W = cam.rot;
    const double f = cam.focal;

    // ---- project_backward (projection.py:186-277)
    const double tz = p.t[2];
    const double iz = 1.0 / tz, iz2 = iz * iz;
    const double A = p.conic[0], B = p.conic[1], C = p.conic[2];
    const double ga = d_con[0], gb = 0.5 * d_con[1], gc = d_con[2];
    const double l00 = A * ga + B * gb, l01 = A * gb + B * gc;
    const double l10 = B * ga + C * gb, l11 = B * gb + C * gc;
    const double Gc[2][2] = {{-(l00 * A + l01 * B), -(l00 * B + l01 * C)},
                             {-(l10 * A + l11 * B), -(l10 * B + l11 * C)}};
    double GM[2][3], gM[2][3], gS[3][3], gJ[2][3];
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k) GM[i][k] = Gc[i][0] * p.M[0][k] + Gc[i][1] * p.M[1][k];
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k)
            gM[i][k] = 2.0 * (GM[i][0] * p.sigma[0][k] + GM[i][1] * p.sigma[1][k] + GM[i][2] * p.sigma[2][k]);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            gS[a][b] = p.M[0][a] * (Gc[0][0] * p.M[0][b] + Gc[0][1] * p.M[1][b]) +
                       p.M[1][a] * (Gc[1][0] * p.M[0][b] + Gc[1][1] * p.M[1][b]);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            gJ[i][j] = gM[i][0] * W[3 * j] + gM[i][1] * W[3 * j + 1] + gM[i][2] * W[3 * j + 2];
    const double dxx = p.xhit ? 0.0 : 1.0, dyy = p.yhit ? 0.0 : 1.0;
    const double dxz = p.xhit ? p.txc * iz : 0.0, dyz = p.yhit ? p.tyc * iz : 0.0;
    const double g_tx = gJ[0][2] * (-f * iz2) * dxx + gmx * f * iz;
    const double g_ty = gJ[1][2] * (f * iz2) * dyy + gmy * (-f * iz);
    double g_tz = gJ[0][0] * (-f * iz2) + gJ[1][1] * (f * iz2) +
                  gJ[0][2] * (2.0 * f * p.txc * iz2 * iz - f * iz2 * dxz) +
                  gJ[1][2] * (-2.0 * f * p.tyc * iz2 * iz + f * iz2 * dyz) +
                  gmx * (-f * p.t[0] * iz2) + gmy * (f * p.t[1] * iz2);
    if (n_ch == 11) g_tz += d_ch[3];
    for (int k = 0; k < 3; ++k) gpos[k] = g_tx * W[k] + g_ty * W[3 + k] + g_tz * W[6 + k];
    double s2[3], glog[3], gR[3][3];
    for (int k = 0; k < 3; ++k) s2[k] = p.scale[k] * p.scale[k];
    for (int k = 0; k < 3; ++k) {
        double acc = 0.0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) acc += p.R[i][k] * gS[i][j] * p.R[j][k];
        glog[k] = 2.0 * s2[k] * acc;
    }
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k)
            gR[i][k] = 2.0 * (gS[i][0] * p.R[0][k] + gS[i][1] * p.R[1][k] + gS[i][2] * p.R[2][k]) * s2[k];
    const double qw = p.q_hat[0], qx = p.q_hat[1], qy = p.q_hat[2], qz = p.q_hat[3];
    double gq[4];
    gq[0] = 2.0 * (qz * (gR[1][0] - gR[0][1]) + qy * (gR[0][2] - gR[2][0]) + qx * (gR[2][1] - gR[1][2]));
    gq[1] = 2.0 * (qy * (gR[0][1] + gR[1][0]) + qz * (gR[0][2] + gR[2][0]) + qw * (gR[2][1] - gR[1][2]) -
                   2.0 * qx * (gR[1][1] + gR[2][2]));
    gq[2] = 2.0 * (qx * (gR[0][1] + gR[1][0]) + qz * (gR[1][2] + gR[2][1]) + qw * (gR[0][2] - gR[2][0]) -
                   2.0 * qy * (gR[0][0] + gR[2][2]));
    gq[3] = 2.0 * (qx * (gR[0][2] + gR[2][0]) + qy * (gR[1][2] + gR[2][1]) + qw * (gR[1][0] - gR[0][1]) -
                   2.0 * qz * (gR[0][0] + gR[1][1]));
    const double gqp = gq[0] * qw + gq[1] * qx + gq[2] * qy + gq[3] * qz;
    const double qd = fmax(p.q_norm, 1e-30);
    double grot[4];
    for (int k = 0; k < 4; ++k) grot[k] = (gq[k] - gqp * p.q_hat[k]) / qd;
    for (int k = 0; k < 3; ++k) VEGS_PUT(G.log_scale[3 * g + k], glog[k]);
    for (int k = 0; k < 4; ++k) VEGS_PUT(G.rot[4 * g + k], grot[k]);
    }

    Shaded s;
    shade_one(P, g, tab, cam, st, s);

    // ---- shade_backward (shading.py:97-176)
    const double sa = fabs(s.ndotl);
    const double sgn = s.ndotl > 0.0 ? 1.0 : (s.ndotl < 0.0 ? -1.0 : 0.0);
    const bool lit = sa > 0.0;
    double dcc = 0.0, dcs = 0.0;
    for (int c = 0; c < 3; ++c) {
        dcc += d_ch[c] * s.cmap[c];
        dcs += d_ch[c];
    }
    double g_ka = dcc, g_kd = dcc * sa, g_ks = dcs * s.spec, g_beta_n = 0.0;
    double d_nhat[3] = {0.0, 0.0, 0.0};
    if (n_ch == 11) {
        for (int k = 0; k < 3; ++k) d_nhat[k] = d_ch[4 + k];
        g_ka += d_ch[7];
        g_kd += d_ch[8];
        g_ks += d_ch[9];
        g_beta_n = d_ch[10] / kBetaMax;
    }
    const double raw_ka = g_ka * s.ka * (1.0 - s.ka);
    const double raw_kd = g_kd * s.kd * (1.0 - s.kd);
    const double raw_ks = g_ks * s.ks * (1.0 - s.ks);
    const double e = exp(P.raw_beta[g]);
    const bool active = (e > kBetaMin) && (e < kBetaMax);
    const double log_s = lit ? log(fmax(sa, 1e-300)) : 0.0;
    const double g_beta = dcs * s.ks * s.spec * log_s + g_beta_n;
    const double raw_beta = active ? g_beta * s.beta : 0.0;
    const double g_s = dcc * s.kd + (lit ? dcs * s.ks * s.beta * s.spec / fmax(sa, 1e-300) : 0.0);
    const double g_ndl = g_s * sgn;
    double gnh[3], gl[3], pnh = 0.0, pl = 0.0;
    for (int k = 0; k < 3; ++k) {
        gnh[k] = g_ndl * s.light[k] + d_nhat[k];
        gl[k] = g_ndl * s.n_hat[k];
        pnh += gnh[k] * s.n_hat[k];
        pl += gl[k] * s.light[k];
    }
    const double nd = fmax(s.n_norm, 1e-30);
    double gnormal[3];
    for (int k = 0; k < 3; ++k) {
        gnormal[k] = (gnh[k] - pnh * s.n_hat[k]) / nd;
        gpos[k] += -(gl[k] - pl * s.light[k]) / s.dist;
    }
    const double vc = clip01(s.v);
    const int jo = slope_segment(tab.ts_op, tab.k_op, vc, tab.inv_op);
    const double dO = (tab.op[jo + 1] - tab.op[jo]) / (tab.ts_op[jo + 1] - tab.ts_op[jo]);
    double gcv = 0.0;
    const int jc = slope_segment(tab.ts_col, tab.k_col, vc, tab.inv_col);
    for (int c = 0; c < 3; ++c)
        gcv += d_ch[c] * ((tab.rgb[c][jc + 1] - tab.rgb[c][jc]) / (tab.ts_col[jc + 1] - tab.ts_col[jc]));
    const double g_v = gcv * (s.ka + s.kd * sa) + d_ab * dO * s.w;
    const double raw_value = g_v * s.v * (1.0 - s.v);
    const double raw_weight = d_ab * s.op * s.w * (1.0 - s.w);

    for (int k = 0; k < 3; ++k) {
        VEGS_PUT(G.pos[3 * g + k], gpos[k]);
        VEGS_PUT(G.normal[3 * g + k], gnormal[k]);
    }
    VEGS_PUT(G.raw_value[g], raw_value);
    VEGS_PUT(G.raw_weight[g], raw_weight);
    VEGS_PUT(G.raw_ka[g], raw_ka);
    VEGS_PUT(G.raw_kd[g], raw_kd);
    VEGS_PUT(G.raw_ks[g], raw_ks);
    VEGS_PUT(G.raw_beta[g], raw_beta);
#undef VEGS_PUT
    const double ax = gmx * (0.5 * cam.width), ay = gmy * (0.5 * cam.height);
    const double vsn = sqrt(ax * ax + ay * ay);  // pipeline.py:355-358 (half-resolution NDC units)
    if (vs_norm) vs_norm[g] = vsn;
    if (dstats) {  // DensifyStats.add (train.py:210-214) for this view
        double *st5 = dstats + 5 * g;
        st5[0] = st5[0] + vsn;
        for (int k = 0; k < 3; ++k) st5[1 + k] = st5[1 + k] + gpos[k];
        st5[4] = st5[4] + 1.0;
    }
    if (visible_out) visible_out[g] = 1;
}

// ---------------------------------------------------------------------------------
// Backward, part 2 for float32 blends: the same adjoint chain with the arithmetic in
// float32 (FFMA, MUFU transcendentals) instead of float64.  The float32 blend's own rows
// carry ~1e-6 relative error, so float64 here bought nothing but FP64-pipe time (this
// kernel was FP64-issue bound).  Every discrete choice the chain makes is still taken in
// float64, exactly as the float64 kernel does: the TF segments of the value slopes (from
// the float64 activated value), the frustum-clamp branches (xhit / yhit from the float64
// camera-space position), the shininess clamp gate, and the sign of n.l when it is within
// float32 rounding of zero.  Decisions identical, arithmetic ~1e-6 relative: far inside the
// 1e-4 gradient bar (tests hold the results to the reference at 1e-4).
// Kept Gaussians appended to a list (warp-aggregated, order irrelevant: every Gaussian's
// outputs depend on it alone); the others get their zero outputs here, so the float32
// chain and its row reduction run only over the kept splats (config 4: 8k of 200k).
__global__ void __launch_bounds__(256) kept_list_kernel(const uint32_t *tiles, int64_t n, int accumulate,
                                                        double *grads, double *vs_norm, uint8_t *visible_out,
                                                        int32_t *list, int32_t *count) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = g < n;
    const bool kept = in && tiles[g] != 0u;
    const unsigned bal = __ballot_sync(0xffffffffu, kept);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && bal) base = atomicAdd(count, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (kept) list[base + __popc(bal & ((1u << lane) - 1u))] = (int32_t)g;
    if (!in || kept) return;
    if (!accumulate) {
        GradView G(grads, n);
        for (int k = 0; k < 3; ++k) G.pos[3 * g + k] = 0.0, G.log_scale[3 * g + k] = 0.0, G.normal[3 * g + k] = 0.0;
        for (int k = 0; k < 4; ++k) G.rot[4 * g + k] = 0.0;
        G.raw_value[g] = G.raw_weight[g] = G.raw_ka[g] = G.raw_kd[g] = G.raw_ks[g] = G.raw_beta[g] = 0.0;
    }
    if (vs_norm) vs_norm[g] = 0.0;
    if (visible_out) visible_out[g] = 0;
}

#ifndef VEGS_PBWD32_MINB
#define VEGS_PBWD32_MINB 3  // 80 registers: 3 x 256 threads per SM (2: 0.344 ms, 4: 0.378 ms per c2 view, both worse)
#endif
__device__ __forceinline__ float sigmoid32(float x) { return 1.f / (1.f + expf(-x)); }

__device__ __noinline__ float ndotl_sign_f64(const ParamView &P, int64_t g, const VegsCamera &cam) {
    double d[3], dd = 0.0, nn = 0.0, dot = 0.0;
    for (int k = 0; k < 3; ++k) {
        d[k] = cam.position[k] - P.pos[3 * g + k];
        dd += d[k] * d[k];
        nn += P.normal[3 * g + k] * P.normal[3 * g + k];
    }
    const double dist = sqrt(dd), nd = fmax(sqrt(nn), 1e-30);
    for (int k = 0; k < 3; ++k) dot += (P.normal[3 * g + k] / nd) * (d[k] / dist);
    return dot > 0.0 ? 1.f : (dot < 0.0 ? -1.f : 0.f);
}

template <int n_ch>
__device__ __forceinline__ void preprocess_bwd32_one(const double *params, int64_t n, const VegsCamera &cam,
                                                     const TFTable &tab, const VegsSettings &st, const double *sums,
                                                     double scale, int accumulate, double *grads, double *vs_norm,
                                                     uint8_t *visible_out, double *dstats, int64_t g);

// over the compacted list of kept Gaussians (kept_list_kernel), a persistent grid: the TF
// table is staged once per CTA instead of once per 256 Gaussians
template <int n_ch>
__global__ void __launch_bounds__(VEGS_PBWD_T, VEGS_PBWD32_MINB) preprocess_bwd32_kernel(
    const double *params, int64_t n, VegsCamera cam, VegsTF tf, VegsSettings st, const int32_t *list,
    const int32_t *count, const double *sums, double scale, int accumulate, double *grads, double *vs_norm,
    uint8_t *visible_out, double *dstats) {
    extern __shared__ double tf_smem[];
    const TFTable tab = stage_tf(tf, tf_smem);
    const int m = *count;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        preprocess_bwd32_one<n_ch>(params, n, cam, tab, st, sums, scale, accumulate, grads, vs_norm, visible_out,
                                   dstats, list[i]);
}

template <int n_ch>
__device__ __forceinline__ void preprocess_bwd32_one(const double *params, int64_t n, const VegsCamera &cam,
                                                     const TFTable &tab, const VegsSettings &st, const double *sums,
                                                     double scale, int accumulate, double *grads, double *vs_norm,
                                                     uint8_t *visible_out, double *dstats, int64_t g) {
    GradView G(grads, n);
    // every input of this Gaussian loaded up front (independent loads in flight together;
    // the outputs are written in one batch at the end)
    const double *red = sums + (int64_t)row_width(n_ch) * g;
    const float gmx = (float)__ldg(red), gmy = (float)__ldg(red + 1);
    const float d_con[3] = {(float)__ldg(red + 2), (float)__ldg(red + 3), (float)__ldg(red + 4)};
    const float d_ab = (float)__ldg(red + 5);
    float d_ch[n_ch];
#pragma unroll
    for (int c = 0; c < n_ch; ++c) d_ch[c] = (float)__ldg(red + 6 + c);
    const ParamView P(params, n);
    double ppos[3];  // float64 where a decision needs it (position, value, shininess)
    float pls[3], prot[4], pnrm[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ppos[k] = __ldg(P.pos + 3 * g + k);
        pls[k] = (float)__ldg(P.log_scale + 3 * g + k);
        pnrm[k] = (float)__ldg(P.normal + 3 * g + k);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) prot[k] = (float)__ldg(P.rot + 4 * g + k);
    const double prv = __ldg(P.raw_value + g), pbeta = __ldg(P.raw_beta + g);
    const float prw = (float)__ldg(P.raw_weight + g), pka = (float)__ldg(P.raw_ka + g),
                pkd = (float)__ldg(P.raw_kd + g), pks = (float)__ldg(P.raw_ks + g);
    float res[19];  // class-major: pos 0-2, log_scale 3-5, rot 6-9, value, weight, normal 12-14, ka, kd, ks, beta
    const double *W64 = cam.rot;
    float W[9];
    for (int k = 0; k < 9; ++k) W[k] = (float)W64[k];
    const float f = (float)cam.focal;
    float gpos[3];
    {
        // ---- projection recompute (projection.py:43-176): t and the clamp branches in float64
        double t64[3];
        for (int i = 0; i < 3; ++i) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += (ppos[k] - cam.position[k]) * W64[3 * i + k];
            t64[i] = acc;
        }
        const double lim_x = st.frustum_limit * cam.tan_x, lim_y = st.frustum_limit * cam.tan_y;
        const double txz64 = t64[0] / t64[2], tyz64 = t64[1] / t64[2];
        const bool xhit = fabs(txz64) > lim_x, yhit = fabs(tyz64) > lim_y;
        const float t0 = (float)t64[0], t1 = (float)t64[1], tz = (float)t64[2];
        const float txc = (float)(fmin(fmax(txz64, -lim_x), lim_x) * t64[2]);
        const float tyc = (float)(fmin(fmax(tyz64, -lim_y), lim_y) * t64[2]);
        float q[4], qq = 0.f;
        for (int k = 0; k < 4; ++k) {
            q[k] = prot[k];
            qq = fmaf(q[k], q[k], qq);
        }
        const float q_norm = sqrtf(qq), qd = fmaxf(q_norm, 1e-30f);
        float qh[4];
        for (int k = 0; k < 4; ++k) qh[k] = q[k] / qd;
        const float w = qh[0], x = qh[1], y = qh[2], z = qh[3];
        const float R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                               {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                               {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
        float s2[3];
        for (int k = 0; k < 3; ++k) {
            const float sc = expf(pls[k]);
            s2[k] = sc * sc;
        }
        float sigma[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                float acc = 0.f;
                for (int k = 0; k < 3; ++k) acc = fmaf(R[i][k] * s2[k], R[j][k], acc);
                sigma[i][j] = acc;
            }
        const float iz = 1.f / tz, iz2 = iz * iz;
        const float j00 = f * iz, j02 = -f * txc * iz2, j11 = -f * iz, j12 = f * tyc * iz2;
        float M[2][3];
        for (int k = 0; k < 3; ++k) {
            M[0][k] = j00 * W[k] + j02 * W[6 + k];
            M[1][k] = j11 * W[3 + k] + j12 * W[6 + k];
        }
        float Acv[2][3];
        for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 3; ++k) Acv[i][k] = M[i][0] * sigma[0][k] + M[i][1] * sigma[1][k] + M[i][2] * sigma[2][k];
        float cov[2][2];
        for (int i = 0; i < 2; ++i)
            for (int l = 0; l < 2; ++l) cov[i][l] = Acv[i][0] * M[l][0] + Acv[i][1] * M[l][1] + Acv[i][2] * M[l][2];
        const float ca = cov[0][0] + (float)st.dilation, cb = cov[0][1], cc = cov[1][1] + (float)st.dilation;
        const float inv_det = 1.f / (ca * cc - cb * cb);
        const float A = cc * inv_det, B = -cb * inv_det, C = ca * inv_det;  // the conic

        // ---- project_backward (projection.py:186-277)
        const float ga = d_con[0], gb = 0.5f * d_con[1], gc = d_con[2];
        const float l00 = A * ga + B * gb, l01 = A * gb + B * gc;
        const float l10 = B * ga + C * gb, l11 = B * gb + C * gc;
        const float Gc[2][2] = {{-(l00 * A + l01 * B), -(l00 * B + l01 * C)},
                                {-(l10 * A + l11 * B), -(l10 * B + l11 * C)}};
        float GM[2][3], gM[2][3], gS[3][3], gJ[2][3];
        for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 3; ++k) GM[i][k] = Gc[i][0] * M[0][k] + Gc[i][1] * M[1][k];
        for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 3; ++k)
                gM[i][k] = 2.f * (GM[i][0] * sigma[0][k] + GM[i][1] * sigma[1][k] + GM[i][2] * sigma[2][k]);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                gS[a][b] = M[0][a] * (Gc[0][0] * M[0][b] + Gc[0][1] * M[1][b]) +
                           M[1][a] * (Gc[1][0] * M[0][b] + Gc[1][1] * M[1][b]);
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 3; ++j) gJ[i][j] = gM[i][0] * W[3 * j] + gM[i][1] * W[3 * j + 1] + gM[i][2] * W[3 * j + 2];
        const float dxx = xhit ? 0.f : 1.f, dyy = yhit ? 0.f : 1.f;
        const float dxz = xhit ? txc * iz : 0.f, dyz = yhit ? tyc * iz : 0.f;
        const float g_tx = gJ[0][2] * (-f * iz2) * dxx + gmx * f * iz;
        const float g_ty = gJ[1][2] * (f * iz2) * dyy + gmy * (-f * iz);
        float g_tz = gJ[0][0] * (-f * iz2) + gJ[1][1] * (f * iz2) +
                     gJ[0][2] * (2.f * f * txc * iz2 * iz - f * iz2 * dxz) +
                     gJ[1][2] * (-2.f * f * tyc * iz2 * iz + f * iz2 * dyz) + gmx * (-f * t0 * iz2) +
                     gmy * (f * t1 * iz2);
        if constexpr (n_ch == 11) g_tz += d_ch[3];
        for (int k = 0; k < 3; ++k) gpos[k] = g_tx * W[k] + g_ty * W[3 + k] + g_tz * W[6 + k];
        float glog[3], gR[3][3];
        for (int k = 0; k < 3; ++k) {
            float acc = 0.f;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) acc += R[i][k] * gS[i][j] * R[j][k];
            glog[k] = 2.f * s2[k] * acc;
        }
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k)
                gR[i][k] = 2.f * (gS[i][0] * R[0][k] + gS[i][1] * R[1][k] + gS[i][2] * R[2][k]) * s2[k];
        float gq[4];
        gq[0] = 2.f * (z * (gR[1][0] - gR[0][1]) + y * (gR[0][2] - gR[2][0]) + x * (gR[2][1] - gR[1][2]));
        gq[1] = 2.f * (y * (gR[0][1] + gR[1][0]) + z * (gR[0][2] + gR[2][0]) + w * (gR[2][1] - gR[1][2]) -
                       2.f * x * (gR[1][1] + gR[2][2]));
        gq[2] = 2.f * (x * (gR[0][1] + gR[1][0]) + z * (gR[1][2] + gR[2][1]) + w * (gR[0][2] - gR[2][0]) -
                       2.f * y * (gR[0][0] + gR[2][2]));
        gq[3] = 2.f * (x * (gR[0][2] + gR[2][0]) + y * (gR[1][2] + gR[2][1]) + w * (gR[1][0] - gR[0][1]) -
                       2.f * z * (gR[0][0] + gR[1][1]));
        const float gqp = gq[0] * w + gq[1] * x + gq[2] * y + gq[3] * z;
        for (int k = 0; k < 3; ++k) res[3 + k] = glog[k];
        for (int k = 0; k < 4; ++k) res[6 + k] = (gq[k] - gqp * qh[k]) / qd;
    }

    // ---- shading recompute (shading.py:52-82): value and TF segments in float64
    const double v64 = sigmoid(prv);
    const double vc64 = clip01(v64);
    const float v = (float)v64, wgt = sigmoid32(prw);
    float op, cmap[3];
    {
        if (vc64 < tab.ts_op[0]) op = (float)tab.op[0];
        else if (vc64 > tab.ts_op[tab.k_op - 1]) op = (float)tab.op[tab.k_op - 1];
        else op = (float)interp_on(tab.ts_op, tab.op, tab.k_op, knot_segment_g(tab.ts_op, tab.k_op, vc64, tab.inv_op), vc64);
        if (vc64 < tab.ts_col[0]) {
            for (int c = 0; c < 3; ++c) cmap[c] = (float)tab.rgb[c][0];
        } else if (vc64 > tab.ts_col[tab.k_col - 1]) {
            for (int c = 0; c < 3; ++c) cmap[c] = (float)tab.rgb[c][tab.k_col - 1];
        } else {
            const int j = knot_segment_g(tab.ts_col, tab.k_col, vc64, tab.inv_col);
            for (int c = 0; c < 3; ++c) cmap[c] = (float)interp_on(tab.ts_col, tab.rgb[c], tab.k_col, j, vc64);
        }
    }
    float dvec[3], dd2 = 0.f, nn2 = 0.f, nrm[3];
    for (int k = 0; k < 3; ++k) {
        dvec[k] = (float)(cam.position[k] - ppos[k]);
        dd2 = fmaf(dvec[k], dvec[k], dd2);
        nrm[k] = pnrm[k];
        nn2 = fmaf(nrm[k], nrm[k], nn2);
    }
    const float dist = sqrtf(dd2), n_norm = sqrtf(nn2), nd = fmaxf(n_norm, 1e-30f);
    float light[3], n_hat[3], ndotl = 0.f;
    for (int k = 0; k < 3; ++k) {
        light[k] = dvec[k] / dist;
        n_hat[k] = nrm[k] / nd;
        ndotl = fmaf(n_hat[k], light[k], ndotl);
    }
    const float sa = fabsf(ndotl);
    // sign of n.l: float64 where float32 rounding could flip it
    const float sgn = sa < 1e-5f ? ndotl_sign_f64(P, g, cam) : (ndotl > 0.f ? 1.f : -1.f);
    const bool lit = sa > 0.f;
    const float ka = sigmoid32(pka), kd = sigmoid32(pkd), ks = sigmoid32(pks);
    const double e64 = exp(pbeta);
    const bool active = (e64 > kBetaMin) && (e64 < kBetaMax);  // the clamp gate, in float64
    const float beta = (float)fmin(fmax(e64, kBetaMin), kBetaMax);
    const float log_s = lit ? logf(fmaxf(sa, 1e-37f)) : 0.f;
    const float spec = lit ? expf(beta * log_s) : 0.f;

    // ---- shade_backward (shading.py:97-176)
    float dcc = 0.f, dcs = 0.f;
    for (int c = 0; c < 3; ++c) {
        dcc = fmaf(d_ch[c], cmap[c], dcc);
        dcs += d_ch[c];
    }
    float g_ka = dcc, g_kd = dcc * sa, g_ks = dcs * spec, g_beta_n = 0.f;
    float d_nhat[3] = {0.f, 0.f, 0.f};
    if constexpr (n_ch == 11) {
        for (int k = 0; k < 3; ++k) d_nhat[k] = d_ch[4 + k];
        g_ka += d_ch[7];
        g_kd += d_ch[8];
        g_ks += d_ch[9];
        g_beta_n = d_ch[10] / (float)kBetaMax;
    }
    const float g_beta = dcs * ks * spec * log_s + g_beta_n;
    const float g_s = dcc * kd + (lit ? dcs * ks * beta * spec / fmaxf(sa, 1e-37f) : 0.f);
    const float g_ndl = g_s * sgn;
    float gnh[3], gl[3], pnh = 0.f, pl = 0.f;
    for (int k = 0; k < 3; ++k) {
        gnh[k] = g_ndl * light[k] + d_nhat[k];
        gl[k] = g_ndl * n_hat[k];
        pnh += gnh[k] * n_hat[k];
        pl += gl[k] * light[k];
    }
    float gnormal[3];
    for (int k = 0; k < 3; ++k) {
        gnormal[k] = (gnh[k] - pnh * n_hat[k]) / nd;
        gpos[k] += -(gl[k] - pl * light[k]) / dist;
    }
    const int jo = slope_segment(tab.ts_op, tab.k_op, vc64, tab.inv_op);
    const float dO = (float)((tab.op[jo + 1] - tab.op[jo]) / (tab.ts_op[jo + 1] - tab.ts_op[jo]));
    float gcv = 0.f;
    const int jc = slope_segment(tab.ts_col, tab.k_col, vc64, tab.inv_col);
    for (int c = 0; c < 3; ++c)
        gcv += d_ch[c] * (float)((tab.rgb[c][jc + 1] - tab.rgb[c][jc]) / (tab.ts_col[jc + 1] - tab.ts_col[jc]));
    const float g_v = gcv * (ka + kd * sa) + d_ab * dO * wgt;
    for (int k = 0; k < 3; ++k) {
        res[k] = gpos[k];
        res[12 + k] = gnormal[k];
    }
    res[10] = g_v * v * (1.f - v);
    res[11] = d_ab * op * wgt * (1.f - wgt);
    res[15] = g_ka * ka * (1.f - ka);
    res[16] = g_kd * kd * (1.f - kd);
    res[17] = g_ks * ks * (1.f - ks);
    res[18] = active ? g_beta * beta : 0.f;
    // component u of the 19-value class-major row: class start (units of n), width, lane
    constexpr int kStart[19] = {0, 0, 0, 3, 3, 3, 6, 6, 6, 6, 10, 11, 12, 12, 12, 15, 16, 17, 18};
    constexpr int kWidth[19] = {3, 3, 3, 3, 3, 3, 4, 4, 4, 4, 1, 1, 3, 3, 3, 1, 1, 1, 1};
    constexpr int kLane[19] = {0, 1, 2, 0, 1, 2, 0, 1, 2, 3, 0, 0, 0, 1, 2, 0, 0, 0, 0};
    if (accumulate) {  // 19 independent loads, then 19 stores
        double old[19];
#pragma unroll
        for (int u = 0; u < 19; ++u) old[u] = grads[kStart[u] * n + kWidth[u] * g + kLane[u]];
#pragma unroll
        for (int u = 0; u < 19; ++u) grads[kStart[u] * n + kWidth[u] * g + kLane[u]] = old[u] + scale * (double)res[u];
    } else {
#pragma unroll
        for (int u = 0; u < 19; ++u) grads[kStart[u] * n + kWidth[u] * g + kLane[u]] = scale * (double)res[u];
    }
    const float ax = gmx * (0.5f * (float)cam.width), ay = gmy * (0.5f * (float)cam.height);
    const double vsn = (double)sqrtf(ax * ax + ay * ay);  // pipeline.py:355-358
    if (vs_norm) vs_norm[g] = vsn;
    if (dstats) {  // DensifyStats.add (train.py:210-214) for this view
        double *st5 = dstats + 5 * g;
        st5[0] = st5[0] + vsn;
        for (int k = 0; k < 3; ++k) st5[1 + k] = st5[1 + k] + (double)gpos[k];
        st5[4] = st5[4] + 1.0;
    }
    if (visible_out) visible_out[g] = 1;
}

// ---------------------------------------------------------------------------------

}  // namespace vegs

using namespace vegs;

extern "C" int vegs_preprocess_backward(const double *params, int64_t n, const VegsCamera *cam,
                                        const VegsTF *tf, const VegsSettings *st, int32_t n_channels,
                                        int32_t store_f64, const uint32_t *tiles, const int64_t *offsets,
                                        const void *inst_rows, double scale, int32_t accumulate,
                                        double *grads, double *viewspace_norm, uint8_t *visible,
                                        double *densify_stats, const uint32_t *inst_visited, int64_t kept_bound,
                                        void *ws, size_t *ws_bytes, void *stream) {
    if (!ws_bytes || (n_channels != 3 && n_channels != 11)) return VEGS_ERR_ARG;
    const size_t sums_bytes = (sizeof(double) * (size_t)row_width(n_channels) * (size_t)(n > 0 ? n : 1) + 255) & ~size_t(255);
    const size_t need = sums_bytes + sizeof(int32_t) * (size_t)(n + 64);  // + the kept list and its count
    if (!ws) {
        *ws_bytes = need;
        return VEGS_OK;
    }
    if (*ws_bytes < need) return VEGS_ERR_CAPACITY;
    if (!cam || !st || !tf_ok(tf) || (n > 0 && (!params || !tiles || !offsets || !grads || !inst_rows || !inst_visited)))
        return VEGS_ERR_ARG;
    if (n == 0) return VEGS_OK;
    const int rr_blocks = (int)((n + VEGS_RR_T - 1) / VEGS_RR_T);
    cudaStream_t s = (cudaStream_t)stream;
    double *sums = (double *)ws;
    const char *chain64 = getenv("VEGS_BWD_CHAIN_F64");  // test switch: float64 chain for float32 blends
    if (!store_f64 && !(chain64 && chain64[0] && chain64[0] != '0')) {
        // float32 blends: the kept Gaussians compacted once, the row sums and the float32
        // chain over that list only
        int32_t *count = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(ws) + sums_bytes);
        int32_t *list = count + 64;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        VEGS_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), s));
        kept_list_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(tiles, n, accumulate, grads, viewspace_norm, visible,
                                                                 list, count);
        VEGS_CHECK_LAUNCH();
        const int64_t kb = kept_bound > 0 && kept_bound < n ? kept_bound : n;
        const int kb_blocks = (int)((kb + VEGS_RR_T - 1) / VEGS_RR_T);
        const int rr_list_blocks = kb_blocks < sms * 32 ? kb_blocks : sms * 32;
        if (n_channels == 3)
            reduce_rows_list_kernel<float, 9><<<rr_list_blocks, VEGS_RR_T, 0, s>>>(tiles, offsets, (const float *)inst_rows,
                                                                               list, count, inst_visited, sums);
        else
            reduce_rows_list_kernel<float, 17><<<rr_list_blocks, VEGS_RR_T, 0, s>>>(tiles, offsets, (const float *)inst_rows,
                                                                                list, count, inst_visited, sums);
        VEGS_CHECK_LAUNCH();
        const size_t smem = tf_smem_bytes(*tf);
        const int full = (int)((kb + VEGS_PBWD_T - 1) / VEGS_PBWD_T);
        const int blocks = full < sms * VEGS_PBWD32_MINB ? full : sms * VEGS_PBWD32_MINB;
        if (n_channels == 3) {
            VEGS_CUDA(cudaFuncSetAttribute(preprocess_bwd32_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            preprocess_bwd32_kernel<3><<<blocks, VEGS_PBWD_T, smem, s>>>(params, n, *cam, *tf, *st, list, count, sums,
                                                                         scale, accumulate, grads, viewspace_norm,
                                                                         visible, densify_stats);
        } else {
            VEGS_CUDA(cudaFuncSetAttribute(preprocess_bwd32_kernel<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            preprocess_bwd32_kernel<11><<<blocks, VEGS_PBWD_T, smem, s>>>(params, n, *cam, *tf, *st, list, count, sums,
                                                                          scale, accumulate, grads, viewspace_norm,
                                                                          visible, densify_stats);
        }
        VEGS_CHECK_LAUNCH();
        return VEGS_OK;
    }
    if (store_f64) {
        if (n_channels == 3) reduce_rows_kernel<double, 9><<<rr_blocks, VEGS_RR_T, 0, s>>>(tiles, offsets, (const double *)inst_rows, n, inst_visited, sums);
        else reduce_rows_kernel<double, 17><<<rr_blocks, VEGS_RR_T, 0, s>>>(tiles, offsets, (const double *)inst_rows, n, inst_visited, sums);
    } else {
        if (n_channels == 3) reduce_rows_kernel<float, 9><<<rr_blocks, VEGS_RR_T, 0, s>>>(tiles, offsets, (const float *)inst_rows, n, inst_visited, sums);
        else reduce_rows_kernel<float, 17><<<rr_blocks, VEGS_RR_T, 0, s>>>(tiles, offsets, (const float *)inst_rows, n, inst_visited, sums);
    }
    VEGS_CHECK_LAUNCH();
    const size_t smem = tf_smem_bytes(*tf);
    VEGS_CUDA(cudaFuncSetAttribute(preprocess_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    preprocess_bwd_kernel<<<(int)((n + VEGS_PBWD_T - 1) / VEGS_PBWD_T), VEGS_PBWD_T, smem, s>>>(params, n, *cam, *tf, *st, n_channels, tiles, sums, scale,
                                                    accumulate, grads, viewspace_norm, visible, densify_stats);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}
