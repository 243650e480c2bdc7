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
// Backward, part 1: float64 sum of each kept Gaussian's instance rows, in duplicate order
// (== sorted-instance order per splat, the order np.add.at applies at pipeline.py:313-316).
// A lean kernel (few registers, full occupancy, 16-byte loads); the visited bitmask
// (L2-resident, one bit per instance) means only the ~30% of rows a pixel actually
// blended are read.  The register-heavy chain runs separately.

template <typename Real, int NV>
#ifndef VEGS_RR_T
#define VEGS_RR_T 64  // small CTAs: the per-Gaussian walks are uneven (3.5 active lanes per warp)
#endif
__global__ void __launch_bounds__(VEGS_RR_T) reduce_rows_kernel(const uint32_t *tiles, const int64_t *offsets,
                                                          const Real *rows, int64_t n, const uint32_t *visited,
                                                          double *sums) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const uint32_t cnt = tiles[g];
    if (cnt == 0) return;
    constexpr int RS = ((7 + (NV - 6)) + 3) & ~3;
    constexpr int NF4 = (int)(RS * sizeof(Real) / 16);
    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0.0;
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
                    for (int k = 0; k < NV; ++k) acc[k] = acc[k] + (double)row[q][k];
                }
        }
        p += span;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) sums[(int64_t)NV * g + k] = acc[k];
}

// The same sums, warp-cooperative (the per-thread walks above keep ~3.6 of 32 lanes busy:
// the visited-row counts of neighbouring Gaussians differ a lot).  A warp owns 32
// consecutive Gaussians, i.e. one contiguous span of duplicate-order rows.  It scans the
// span's visited words 32 at a time and compacts the visited rows into batches of 32
// (SMEM); per batch every lane loads one row (contiguous rows: coalesced), finds its
// Gaussian by a 5-step search over the warp's 32 offsets, and stages the row in SMEM; the
// first lane of each Gaussian's run then adds the run's rows, in ascending row order, to
// that Gaussian's float64 accumulator.  Every accumulator therefore sees exactly the
// additions of reduce_rows_kernel in the same order: bitwise the same sums.
#ifndef VEGS_RRW_WARPS
#define VEGS_RRW_WARPS 4
#endif
template <typename Real, int NV>
__global__ void __launch_bounds__(32 * VEGS_RRW_WARPS) reduce_rows_warp_kernel(const int64_t *offsets,
                                                                               const Real *rows, int64_t n,
                                                                               const uint32_t *visited,
                                                                               double *sums) {
    constexpr int RS = ((7 + (NV - 6)) + 3) & ~3;
    constexpr int NF4 = (int)(RS * sizeof(Real) / 16);
    __shared__ int64_t s_p[VEGS_RRW_WARPS][64];           // compacted visited rows (up to 63 pending)
    __shared__ __align__(16) Real s_row[VEGS_RRW_WARPS][32][RS];
    __shared__ int8_t s_own[VEGS_RRW_WARPS][33];
    __shared__ double s_acc[VEGS_RRW_WARPS][32][NV + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g0 = ((int64_t)blockIdx.x * VEGS_RRW_WARPS + warp) * 32;
    if (g0 >= n) return;
    const int64_t off_l = __ldg(offsets + (g0 + lane < n ? g0 + lane : n));
    const int64_t p_begin = __shfl_sync(0xffffffffu, off_l, 0);
    const int64_t p_end = __ldg(offsets + (g0 + 32 < n ? g0 + 32 : n));
#pragma unroll
    for (int k = 0; k < NV; ++k) s_acc[warp][lane][k] = 0.0;
    int64_t *bp = s_p[warp];
    int fill = 0;
    auto flush = [&](int m) {  // m visited rows in bp[0..m)
        const int64_t p = lane < m ? bp[lane] : INT64_MAX;
        int lo = 0;  // last local Gaussian whose offset is <= p (every lane in the shuffles)
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const int cand = lo + step;
            const int64_t oc = __shfl_sync(0xffffffffu, off_l, cand & 31);
            if (cand < 32 && oc <= p) lo = cand;
        }
        if (lane < m) {
            s_own[warp][lane] = (int8_t)lo;
            const float4 *src = reinterpret_cast<const float4 *>(rows + (int64_t)RS * p);
#pragma unroll
            for (int k = 0; k < NF4; ++k) reinterpret_cast<float4 *>(s_row[warp][lane])[k] = __ldg(src + k);
        } else if (lane == m) {
            s_own[warp][lane] = -1;
        }
        __syncwarp();
        if (lane < m) {
            const int o = s_own[warp][lane];
            if (lane == 0 || s_own[warp][lane - 1] != o) {  // head of o's run in this batch
                double a[NV];
#pragma unroll
                for (int k = 0; k < NV; ++k) a[k] = s_acc[warp][o][k];
                for (int r = lane; r < m && s_own[warp][r] == o; ++r) {
#pragma unroll
                    for (int k = 0; k < NV; ++k) a[k] = a[k] + (double)s_row[warp][r][k];
                }
#pragma unroll
                for (int k = 0; k < NV; ++k) s_acc[warp][o][k] = a[k];
            }
        }
        __syncwarp();
    };
    if (p_end > p_begin) {
        const int64_t w_lo = p_begin >> 5, w_hi = (p_end - 1) >> 5;
        for (int64_t wb = w_lo; wb <= w_hi; wb += 32) {
            const int64_t wi = wb + lane;
            uint32_t word = 0;
            if (wi <= w_hi) {
                word = __ldg(visited + wi);
                if (wi == w_lo) word &= ~0u << (uint32_t)(p_begin & 31);
                if (wi == w_hi && ((p_end & 31) != 0)) word &= (1u << (uint32_t)(p_end & 31)) - 1u;
            }
            const int nw = (int)(w_hi - wb + 1 < 32 ? w_hi - wb + 1 : 32);
            for (int k = 0; k < nw; ++k) {
                const uint32_t bits = __shfl_sync(0xffffffffu, word, k);
                if (!bits) continue;
                if ((bits >> lane) & 1u) bp[fill + __popc(bits & ((1u << lane) - 1u))] = ((wb + k) << 5) + lane;
                fill += __popc(bits);
                __syncwarp();
                if (fill >= 32) {
                    flush(32);
                    if (lane < fill - 32) bp[lane] = bp[32 + lane];
                    fill -= 32;
                    __syncwarp();
                }
            }
        }
        if (fill > 0) flush(fill);
    }
    if (g0 + lane < n) {
#pragma unroll
        for (int k = 0; k < NV; ++k) sums[(int64_t)NV * (g0 + lane) + k] = s_acc[warp][lane][k];
    }
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

}  // namespace vegs

using namespace vegs;

extern "C" int vegs_preprocess_backward(const double *params, int64_t n, const VegsCamera *cam,
                                        const VegsTF *tf, const VegsSettings *st, int32_t n_channels,
                                        int32_t store_f64, const uint32_t *tiles, const int64_t *offsets,
                                        const void *inst_rows, double scale, int32_t accumulate,
                                        double *grads, double *viewspace_norm, uint8_t *visible,
                                        double *densify_stats, const uint32_t *inst_visited, void *ws, size_t *ws_bytes,
                                        void *stream) {
    if (!ws_bytes || (n_channels != 3 && n_channels != 11)) return VEGS_ERR_ARG;
    const size_t need = sizeof(double) * (size_t)row_width(n_channels) * (size_t)(n > 0 ? n : 1);
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
    const char *per_thread = getenv("VEGS_RR_PER_THREAD");  // test switch: the per-Gaussian walk
    if (!(per_thread && per_thread[0] && per_thread[0] != '0')) {
        const int wb = (int)((n + 32 * VEGS_RRW_WARPS - 1) / (32 * VEGS_RRW_WARPS));
        if (store_f64) {
            if (n_channels == 3) reduce_rows_warp_kernel<double, 9><<<wb, 32 * VEGS_RRW_WARPS, 0, s>>>(offsets, (const double *)inst_rows, n, inst_visited, sums);
            else reduce_rows_warp_kernel<double, 17><<<wb, 32 * VEGS_RRW_WARPS, 0, s>>>(offsets, (const double *)inst_rows, n, inst_visited, sums);
        } else {
            if (n_channels == 3) reduce_rows_warp_kernel<float, 9><<<wb, 32 * VEGS_RRW_WARPS, 0, s>>>(offsets, (const float *)inst_rows, n, inst_visited, sums);
            else reduce_rows_warp_kernel<float, 17><<<wb, 32 * VEGS_RRW_WARPS, 0, s>>>(offsets, (const float *)inst_rows, n, inst_visited, sums);
        }
    } else if (store_f64) {
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
