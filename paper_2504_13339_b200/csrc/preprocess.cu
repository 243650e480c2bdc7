// Per-Gaussian preprocess (forward + backward), TF lookup and Adam for sm_100a.
//
// This translation unit is compiled with -fmad=false: every float64 multiply/add is
// rounded separately, the way numpy evaluates the reference's elementwise expressions.
// That keeps the values that feed integer decisions -- the culling tests, the pixel
// rectangles (ceil/floor of the 1/255 level set) and the depth keys -- identical to the
// reference's, and makes the float32 casts of the blend inputs agree bit for bit in
// practice (only libm-ulp differences of exp/log/pow remain).
//
// Reference: shading.py:52-82 (shade), projection.py:27-176 (quat_to_rotmat, project),
// pipeline.py:137-160,207-215 (channels, pmin, dtype cast), transfer.py:91-127 (TF),
// projection.py:186-277 (project_backward), shading.py:97-176 (shade_backward),
// pipeline.py:307-366 (per-splat reduction + GradientSet), train.py:176-195 (Adam).

#include <math.h>

#include <cub/cub.cuh>

#include "vegs_common.cuh"

namespace vegs {

// ---------------------------------------------------------------------------------
// Transfer function: np.interp semantics (numpy compiled_base.c arr_interp) and the
// half-open-segment slope of transfer.py:106-127.

__device__ __forceinline__ int knot_segment(const double *ts, int k, double x) {
    // largest j with ts[j] <= x (x inside [ts[0], ts[k-1]])
    int lo = 0, hi = k;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (ts[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

__device__ double tf_interp(const double *ts, const double *vals, int k, double x) {
    if (x != x) return x;
    if (x < ts[0]) return vals[0];
    if (x > ts[k - 1]) return vals[k - 1];
    const int j = knot_segment(ts, k, x);
    if (j == k - 1 || ts[j] == x) return vals[j];
    const double slope = (vals[j + 1] - vals[j]) / (ts[j + 1] - ts[j]);
    return slope * (x - ts[j]) + vals[j];
}

__device__ double tf_slope(const double *ts, const double *vals, int k, double x) {
    int j = (x < ts[0]) ? -1 : knot_segment(ts, k, x);
    j = j < 0 ? 0 : (j > k - 2 ? k - 2 : j);
    return (vals[j + 1] - vals[j]) / (ts[j + 1] - ts[j]);
}

__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

// TF tables staged in shared memory: [ts_op | op | ts_col | r | g | b]
struct TFTable {
    const double *ts_op, *op, *ts_col, *rgb[3];
    int k_op, k_col;
};

__device__ TFTable stage_tf(const VegsTF &tf, double *smem) {
    const int total = 2 * tf.n_opacity + 4 * tf.n_color;
    for (int i = threadIdx.x; i < total; i += blockDim.x) smem[i] = tf.blob[i];
    __syncthreads();
    TFTable t;
    t.k_op = tf.n_opacity;
    t.k_col = tf.n_color;
    t.ts_op = smem;
    t.op = smem + t.k_op;
    t.ts_col = smem + 2 * t.k_op;
    t.rgb[0] = t.ts_col + t.k_col;
    t.rgb[1] = t.rgb[0] + t.k_col;
    t.rgb[2] = t.rgb[1] + t.k_col;
    return t;
}

// ---------------------------------------------------------------------------------
// Forward per-Gaussian state, recomputed by the backward from the raw parameters.

struct Shaded {
    double v, w, op, cmap[3], alpha_base, light[3], dist, n_hat[3], n_norm, ndotl, ka, kd, ks,
        beta, spec, color[3];
    bool visible;
};

struct Projected {
    double t[3], txc, tyc, px, py, q_hat[4], q_norm, R[3][3], scale[3], sigma[3][3], M[2][3],
        a, b, c, det, lam, conic[3], radius;
    bool xhit, yhit, keep;
    int x0, x1, y0, y1;
};

__device__ void shade_one(const ParamView &P, int64_t g, const TFTable &tf, const VegsCamera &cam,
                          const VegsSettings &st, Shaded &s) {
    s.v = sigmoid(P.raw_value[g]);
    s.w = sigmoid(P.raw_weight[g]);
    const double vc = clip01(s.v);
    s.op = tf_interp(tf.ts_op, tf.op, tf.k_op, vc);
    for (int c = 0; c < 3; ++c) s.cmap[c] = tf_interp(tf.ts_col, tf.rgb[c], tf.k_col, vc);
    s.alpha_base = s.op * s.w;
    double d[3], nn2 = 0.0, dd2 = 0.0;
    for (int k = 0; k < 3; ++k) {
        d[k] = cam.position[k] - P.pos[3 * g + k];
        dd2 = dd2 + d[k] * d[k];
    }
    s.dist = sqrt(dd2);
    for (int k = 0; k < 3; ++k) s.light[k] = d[k] / s.dist;
    for (int k = 0; k < 3; ++k) nn2 = nn2 + P.normal[3 * g + k] * P.normal[3 * g + k];
    s.n_norm = sqrt(nn2);
    const double nd = fmax(s.n_norm, 1e-30);
    s.ndotl = 0.0;
    for (int k = 0; k < 3; ++k) {
        s.n_hat[k] = P.normal[3 * g + k] / nd;
        s.ndotl = s.ndotl + s.n_hat[k] * s.light[k];
    }
    const double sa = fabs(s.ndotl);
    s.ka = sigmoid(P.raw_ka[g]);
    s.kd = sigmoid(P.raw_kd[g]);
    s.ks = sigmoid(P.raw_ks[g]);
    s.beta = fmin(fmax(exp(P.raw_beta[g]), kBetaMin), kBetaMax);
    s.spec = sa > 0.0 ? pow(fmax(sa, 1e-300), s.beta) : 0.0;
    const double diffuse = s.ka + s.kd * sa;
    const double specular = s.ks * s.spec;
    for (int c = 0; c < 3; ++c) s.color[c] = diffuse * s.cmap[c] + specular;
    s.visible = s.alpha_base >= st.cull_alpha;
}

template <bool kRect = true>
__device__ void project_one(const ParamView &P, int64_t g, double alpha_base, const VegsCamera &cam,
                            const VegsSettings &st, Projected &p) {
    const double *W = cam.rot;
    double d[3];
    for (int k = 0; k < 3; ++k) d[k] = P.pos[3 * g + k] - cam.position[k];
    for (int i = 0; i < 3; ++i) p.t[i] = d[0] * W[3 * i] + d[1] * W[3 * i + 1] + d[2] * W[3 * i + 2];
    const double tz = p.t[2];
    const bool front = tz > cam.near_z;
    const double lim_x = st.frustum_limit * cam.tan_x;
    const double lim_y = st.frustum_limit * cam.tan_y;
    const double zs = front ? tz : 1.0;
    const double txz = p.t[0] / zs, tyz = p.t[1] / zs;
    p.xhit = fabs(txz) > lim_x;
    p.yhit = fabs(tyz) > lim_y;
    p.txc = fmin(fmax(txz, -lim_x), lim_x) * tz;
    p.tyc = fmin(fmax(tyz, -lim_y), lim_y) * tz;
    const double f = cam.focal;
    p.px = 0.5 * (double)cam.width + f * txz;
    p.py = 0.5 * (double)cam.height - f * tyz;

    double q[4], qq = 0.0;
    for (int k = 0; k < 4; ++k) {
        q[k] = P.rot[4 * g + k];
        qq = qq + q[k] * q[k];
    }
    p.q_norm = sqrt(qq);
    const double qd = fmax(p.q_norm, 1e-30);
    for (int k = 0; k < 4; ++k) p.q_hat[k] = q[k] / qd;
    const double w = p.q_hat[0], x = p.q_hat[1], y = p.q_hat[2], z = p.q_hat[3];
    p.R[0][0] = 1 - 2 * (y * y + z * z);
    p.R[0][1] = 2 * (x * y - w * z);
    p.R[0][2] = 2 * (x * z + w * y);
    p.R[1][0] = 2 * (x * y + w * z);
    p.R[1][1] = 1 - 2 * (x * x + z * z);
    p.R[1][2] = 2 * (y * z - w * x);
    p.R[2][0] = 2 * (x * z - w * y);
    p.R[2][1] = 2 * (y * z + w * x);
    p.R[2][2] = 1 - 2 * (x * x + y * y);
    double s2[3];
    for (int k = 0; k < 3; ++k) {
        p.scale[k] = exp(P.log_scale[3 * g + k]);
        s2[k] = p.scale[k] * p.scale[k];
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc = acc + (p.R[i][k] * s2[k]) * p.R[j][k];
            p.sigma[i][j] = acc;
        }
    const double iz = 1.0 / zs, iz2 = iz * iz;
    const double j00 = f * iz, j02 = -f * p.txc * iz2;
    const double j11 = -f * iz, j12 = f * p.tyc * iz2;
    for (int k = 0; k < 3; ++k) {
        p.M[0][k] = j00 * W[k] + j02 * W[6 + k];
        p.M[1][k] = j11 * W[3 + k] + j12 * W[6 + k];
    }
    double A[2][3];
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k)
            A[i][k] = (p.M[i][0] * p.sigma[0][k] + p.M[i][1] * p.sigma[1][k]) + p.M[i][2] * p.sigma[2][k];
    double cov[2][2];
    for (int i = 0; i < 2; ++i)
        for (int l = 0; l < 2; ++l)
            cov[i][l] = (A[i][0] * p.M[l][0] + A[i][1] * p.M[l][1]) + A[i][2] * p.M[l][2];
    p.a = cov[0][0] + st.dilation;
    p.b = cov[0][1];
    p.c = cov[1][1] + st.dilation;
    p.det = p.a * p.c - p.b * p.b;
    const double mid = 0.5 * (p.a + p.c);
    p.lam = mid + sqrt(fmax(mid * mid - p.det, 0.0));
    p.radius = st.radius_sigma * sqrt(fmax(p.lam, 0.0));
    const double inv_det = p.det > 0 ? 1.0 / p.det : 0.0;
    p.conic[0] = p.c * inv_det;
    p.conic[1] = -p.b * inv_det;
    p.conic[2] = p.a * inv_det;
    if constexpr (!kRect) {  // the backward only needs the projection, not the rect
        p.keep = front && (p.det > 0);
        return;
    }
    const double ratio = fmax(alpha_base, st.alpha_skip) / st.alpha_skip;
    const double rc = sqrt(fmax(p.lam, 0.0) * 2.0 * log(ratio)) + st.rect_margin_px;
    const double Wd = (double)cam.width, Hd = (double)cam.height;
    const double fx0 = fmin(fmax(ceil(p.px - rc - 0.5), 0.0), Wd);
    const double fx1 = fmin(fmax(floor(p.px + rc - 0.5) + 1.0, 0.0), Wd);
    const double fy0 = fmin(fmax(ceil(p.py - rc - 0.5), 0.0), Hd);
    const double fy1 = fmin(fmax(floor(p.py + rc - 0.5) + 1.0, 0.0), Hd);
    const bool finite = isfinite(p.px) && isfinite(p.py);
    p.x0 = finite ? (int)fx0 : 0;
    p.x1 = finite ? (int)fx1 : 0;
    p.y0 = finite ? (int)fy0 : 0;
    p.y1 = finite ? (int)fy1 : 0;
    p.keep = front && (p.det > 0) && (p.x1 > p.x0) && (p.y1 > p.y0) && finite;
}

// Total order on float64 -> uint64 (negative values flipped), so a radix sort of the
// keys is a sort of the depths; culled splats carry ~0.
__device__ __forceinline__ uint64_t depth_order_key(double d) {
    const uint64_t b = (uint64_t)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <typename Real>
__device__ void write_record(Real *r, double px, double py, const double *conic, double alpha_base,
                             double alpha_skip) {
    const double pmin = log(alpha_skip / fmax(alpha_base, alpha_skip * 1e-6));  // pipeline.py:207
    r[0] = (Real)px;
    r[1] = (Real)py;
    r[2] = (Real)conic[0];
    r[3] = (Real)conic[1];
    r[4] = (Real)conic[2];
    r[5] = (Real)alpha_base;
    r[6] = (Real)pmin;
}

// ---------------------------------------------------------------------------------

template <typename Real>
#ifndef VEGS_PFWD_MINB
#define VEGS_PFWD_MINB 4  // 64 registers: 4x the resident warps of the unbounded build, ~2x faster
#endif
#ifndef VEGS_PBWD_MINB
#define VEGS_PBWD_MINB 4
#endif
__global__ void __launch_bounds__(256, VEGS_PFWD_MINB) preprocess_fwd_kernel(
    const double *params, int64_t n, VegsCamera cam, VegsTF tf, VegsSettings st, int n_ch,
    VegsSplatTable out) {
    extern __shared__ double tf_smem[];
    const TFTable tab = stage_tf(tf, tf_smem);
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const ParamView P(params, n);
    Shaded s;
    shade_one(P, g, tab, cam, st, s);
    if (out.alpha_base) out.alpha_base[g] = s.alpha_base;
    if (out.color)
        for (int c = 0; c < 3; ++c) out.color[3 * g + c] = s.color[c];
    if (out.visible) out.visible[g] = s.visible ? 1 : 0;
    bool kept = false;
    Projected p;
    if (s.visible) {
        project_one(P, g, s.alpha_base, cam, st, p);
        kept = p.keep;
    }
    if (out.aux) {
        double *a = out.aux + 24 * g;
        const double vals[24] = {s.v, s.w, s.op, s.cmap[0], s.cmap[1], s.cmap[2], s.light[0], s.light[1],
                                 s.light[2], s.dist, s.n_hat[0], s.n_hat[1], s.n_hat[2], s.n_norm, s.ndotl,
                                 s.ka, s.kd, s.ks, s.beta, s.spec, s.visible ? p.a : 0.0,
                                 s.visible ? p.b : 0.0, s.visible ? p.c : 0.0, 0.0};
        for (int k = 0; k < 24; ++k) a[k] = vals[k];
    }
    if (!kept) {
        out.tiles[g] = 0u;
        out.depth_key[g] = ~0ull;
        return;
    }
    const int ts = st.tile_size;
    const int nx = (p.x1 - 1) / ts - p.x0 / ts + 1;
    const int ny = (p.y1 - 1) / ts - p.y0 / ts + 1;
    out.tiles[g] = (uint32_t)(nx * ny);
    out.depth_key[g] = depth_order_key(p.t[2]);
    out.rect[4 * g + 0] = p.x0;
    out.rect[4 * g + 1] = p.x1;
    out.rect[4 * g + 2] = p.y0;
    out.rect[4 * g + 3] = p.y1;
    Real *r = reinterpret_cast<Real *>(out.record) + (int64_t)rec_stride(n_ch) * g;
    write_record(r, p.px, p.py, p.conic, s.alpha_base, st.alpha_skip);
    for (int c = 0; c < 3; ++c) r[7 + c] = (Real)s.color[c];
    if (n_ch == 11) {  // pipeline.py:31-37,150-157
        r[10] = (Real)p.t[2];
        for (int k = 0; k < 3; ++k) r[11 + k] = (Real)s.n_hat[k];
        r[14] = (Real)s.ka;
        r[15] = (Real)s.kd;
        r[16] = (Real)s.ks;
        r[17] = (Real)(s.beta / kBetaMax);
    }
    if (out.mean2d) {
        out.mean2d[2 * g] = p.px;
        out.mean2d[2 * g + 1] = p.py;
    }
    if (out.conic)
        for (int k = 0; k < 3; ++k) out.conic[3 * g + k] = p.conic[k];
    if (out.depth) out.depth[g] = p.t[2];
    if (out.radius) out.radius[g] = p.radius;
}

template <typename Real>
__global__ void __launch_bounds__(256) table_from_arrays_kernel(
    const double *mean2d, const double *conic, const double *alpha_base, const double *depth,
    const int32_t *rect, const double *channels, int64_t m, VegsSettings st, int n_ch, VegsSplatTable out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int x0 = rect[4 * i], x1 = rect[4 * i + 1], y0 = rect[4 * i + 2], y1 = rect[4 * i + 3];
    const int ts = st.tile_size;
    const int nx = (x1 - 1) / ts - x0 / ts + 1, ny = (y1 - 1) / ts - y0 / ts + 1;
    out.tiles[i] = (uint32_t)(nx * ny);
    out.depth_key[i] = depth_order_key(depth[i]);
    for (int k = 0; k < 4; ++k) out.rect[4 * i + k] = rect[4 * i + k];
    Real *r = reinterpret_cast<Real *>(out.record) + (int64_t)rec_stride(n_ch) * i;
    write_record(r, mean2d[2 * i], mean2d[2 * i + 1], conic + 3 * i, alpha_base[i], st.alpha_skip);
    for (int c = 0; c < n_ch; ++c) r[7 + c] = (Real)channels[(int64_t)n_ch * i + c];
}

// ---------------------------------------------------------------------------------
// Backward, part 1: float64 sum of each kept Gaussian's instance rows, in duplicate order
// (== sorted-instance order per splat, the order np.add.at applies at pipeline.py:313-316).
// A lean kernel (few registers, full occupancy, 16-byte loads); the visited bitmask
// (L2-resident, one bit per instance) means only the ~30% of rows a pixel actually
// blended are read.  The register-heavy chain runs separately.

template <typename Real, int NV>
__global__ void __launch_bounds__(256) reduce_rows_kernel(const uint32_t *tiles, const int64_t *offsets,
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
            constexpr int Q = RS * sizeof(Real) <= 48 ? 4 : 1;  // rgb float32 rows: 4 in flight
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

// Backward, part 2: projection and shading adjoints per Gaussian (float64).

__global__ void __launch_bounds__(256, VEGS_PBWD_MINB) preprocess_bwd_kernel(
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
    const double dO = tf_slope(tab.ts_op, tab.op, tab.k_op, vc);
    double gcv = 0.0;
    for (int c = 0; c < 3; ++c) gcv += d_ch[c] * tf_slope(tab.ts_col, tab.rgb[c], tab.k_col, vc);
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

__global__ void tf_eval_kernel(const double *ts, const double *vals, int k, int n_cols,
                               const double *q, int64_t nq, int derivative, double *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const double x = clip01(q[i]);
    for (int c = 0; c < n_cols; ++c) {
        const double *col = vals + (int64_t)c * k;  // column-major: vals[c * k + j]
        out[i * n_cols + c] = derivative ? tf_slope(ts, col, k, x) : tf_interp(ts, col, k, x);
    }
}

// Adam over the class-major flat buffer; class boundaries in units of n.
__constant__ int kClassEnd[10] = {3, 6, 10, 11, 12, 15, 16, 17, 18, 19};

__global__ void __launch_bounds__(256) adam_kernel(double *params, const double *grads, double *m,
                                                   double *v, int64_t n, const double *lr,
                                                   double grad_scale, double bias1, double bias2,
                                                   int *nonfinite) {
    const int64_t total = 19 * n;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-15;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t unit = i / n;
        int cls = 0;
        while (unit >= kClassEnd[cls]) ++cls;
        const double gr = grads[i] * grad_scale;
        if (!isfinite(gr)) {
            atomicOr(nonfinite + cls, 1);
            continue;
        }
        double mi = m[i] * b1;
        mi = mi + (1.0 - b1) * gr;
        double vi = v[i] * b2;
        vi = vi + (1.0 - b2) * gr * gr;
        m[i] = mi;
        v[i] = vi;
        const double upd = (mi / bias1) / (sqrt(vi / bias2) + eps);
        params[i] = params[i] - lr[cls] * upd;
    }
}

static size_t tf_smem_bytes(const VegsTF &tf) {
    return sizeof(double) * (size_t)(2 * tf.n_opacity + 4 * tf.n_color);
}

static bool tf_ok(const VegsTF *tf) {
    return tf && tf->blob && tf->n_opacity >= 2 && tf->n_color >= 2 && tf->n_opacity <= VEGS_MAX_KNOTS &&
           tf->n_color <= VEGS_MAX_KNOTS;
}

}  // namespace vegs

using namespace vegs;

extern "C" int vegs_tf_eval(const double *ts, const double *vals, int32_t n_knots, int32_t n_cols,
                            const double *query, int64_t n_query, int32_t derivative, double *out,
                            void *stream) {
    if (!ts || !vals || !query || !out || n_knots < 2 || n_cols < 1) return VEGS_ERR_ARG;
    if (n_query == 0) return VEGS_OK;
    const int blocks = (int)((n_query + 255) / 256);
    tf_eval_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(ts, vals, n_knots, n_cols, query, n_query,
                                                             derivative, out);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" int vegs_preprocess_forward(const double *params, int64_t n, const VegsCamera *cam,
                                       const VegsTF *tf, const VegsSettings *st, int32_t n_channels,
                                       int32_t store_f64, VegsSplatTable *out, void *stream) {
    if (!cam || !st || !out || !tf_ok(tf) || (n > 0 && !params)) return VEGS_ERR_ARG;
    if (n_channels != 3 && n_channels != 11) return VEGS_ERR_ARG;
    if (st->tile_size != kTile) return VEGS_ERR_ARG;
    if (!out->record || !out->rect || !out->tiles || !out->depth_key) return VEGS_ERR_ARG;
    if (n == 0) return VEGS_OK;
    const size_t smem = tf_smem_bytes(*tf);
    const int blocks = (int)((n + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    if (store_f64) {
        VEGS_CUDA(cudaFuncSetAttribute(preprocess_fwd_kernel<double>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        preprocess_fwd_kernel<double><<<blocks, 256, smem, s>>>(params, n, *cam, *tf, *st, n_channels, *out);
    } else {
        VEGS_CUDA(cudaFuncSetAttribute(preprocess_fwd_kernel<float>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        preprocess_fwd_kernel<float><<<blocks, 256, smem, s>>>(params, n, *cam, *tf, *st, n_channels, *out);
    }
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" int vegs_splat_table_from_arrays(const double *mean2d, const double *conic,
                                            const double *alpha_base, const double *depth, const int32_t *rect,
                                            const double *channels, int64_t m, const VegsSettings *st,
                                            int32_t n_channels, int32_t store_f64, VegsSplatTable *out,
                                            void *stream) {
    if (!st || !out || (n_channels != 3 && n_channels != 11) || st->tile_size != kTile) return VEGS_ERR_ARG;
    if (m == 0) return VEGS_OK;
    if (!mean2d || !conic || !alpha_base || !depth || !rect || !channels || !out->record || !out->tiles ||
        !out->depth_key || !out->rect)
        return VEGS_ERR_ARG;
    const int blocks = (int)((m + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    if (store_f64)
        table_from_arrays_kernel<double><<<blocks, 256, 0, s>>>(mean2d, conic, alpha_base, depth, rect, channels,
                                                                m, *st, n_channels, *out);
    else
        table_from_arrays_kernel<float><<<blocks, 256, 0, s>>>(mean2d, conic, alpha_base, depth, rect, channels,
                                                               m, *st, n_channels, *out);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

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
    const int blocks = (int)((n + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    double *sums = (double *)ws;
    if (store_f64) {
        if (n_channels == 3) reduce_rows_kernel<double, 9><<<blocks, 256, 0, s>>>(tiles, offsets, (const double *)inst_rows, n, inst_visited, sums);
        else reduce_rows_kernel<double, 17><<<blocks, 256, 0, s>>>(tiles, offsets, (const double *)inst_rows, n, inst_visited, sums);
    } else {
        if (n_channels == 3) reduce_rows_kernel<float, 9><<<blocks, 256, 0, s>>>(tiles, offsets, (const float *)inst_rows, n, inst_visited, sums);
        else reduce_rows_kernel<float, 17><<<blocks, 256, 0, s>>>(tiles, offsets, (const float *)inst_rows, n, inst_visited, sums);
    }
    VEGS_CHECK_LAUNCH();
    const size_t smem = tf_smem_bytes(*tf);
    VEGS_CUDA(cudaFuncSetAttribute(preprocess_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    preprocess_bwd_kernel<<<blocks, 256, smem, s>>>(params, n, *cam, *tf, *st, n_channels, tiles, sums, scale,
                                                    accumulate, grads, viewspace_norm, visible, densify_stats);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" int vegs_adam_step(double *params, const double *grads, double *m, double *v, int64_t n,
                              const double *lr, double grad_scale, double bias1, double bias2,
                              int32_t *nonfinite, void *stream) {
    if (n > 0 && (!params || !grads || !m || !v || !lr || !nonfinite)) return VEGS_ERR_ARG;
    if (n == 0) return VEGS_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t total = 19 * n;
    int blocks = (int)((total + 255) / 256);
    if (blocks > sms * 16) blocks = sms * 16;
    adam_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(params, grads, m, v, n, lr, grad_scale, bias1,
                                                          bias2, nonfinite);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

// ---------------------------------------------------------------------------------
// Densify / prune (train.py:237-284), float64, reproducing the reference's output order:
//   [kept originals that survive | surviving clones | surviving split children, round 0 |
//    round 1], each block in Gaussian order, optimizer moments kept for originals and zero
//   for new rows.  Split offsets use host-drawn normals eps[round][split_rank][3] so the
//   caller can replay the reference's rng.standard_normal draws exactly.

namespace vegs {

struct Int4Sum {
    __device__ __forceinline__ int4 operator()(const int4 &a, const int4 &b) const {
        return make_int4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
};

__device__ __forceinline__ void densify_flags(const ParamView &P, int64_t g, const double *stats,
                                              const VegsDensify &dp, bool &small, bool &big, bool &survive) {
    const double cnt = fmax(stats[5 * g + 4], 1.0);
    const bool cand = stats[5 * g] / cnt > dp.grad_threshold;
    double ms = exp(P.log_scale[3 * g]);
    ms = fmax(ms, exp(P.log_scale[3 * g + 1]));
    ms = fmax(ms, exp(P.log_scale[3 * g + 2]));
    small = cand && ms <= dp.percent_dense * dp.scene_extent;
    big = cand && !small;
    survive = dp.no_weights || sigmoid(P.raw_weight[g]) >= dp.prune_threshold;
}

__global__ void densify_classify_kernel(const double *params, int64_t n, const double *stats, VegsDensify dp,
                                        int4 *flags) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g > n) return;
    if (g == n) {
        flags[g] = make_int4(0, 0, 0, 0);
        return;
    }
    const ParamView P(params, n);
    bool small, big, surv;
    densify_flags(P, g, stats, dp, small, big, surv);
    flags[g] = make_int4(!big && surv, small && surv, big && surv, big);
}

__device__ __forceinline__ void copy_row(const double *src, int64_t n, int64_t g, double *dst, int64_t n_out,
                                         int64_t r) {
    ParamView S(src, n);
    GradView D(dst, n_out);
    for (int k = 0; k < 3; ++k) {
        D.pos[3 * r + k] = S.pos[3 * g + k];
        D.log_scale[3 * r + k] = S.log_scale[3 * g + k];
        D.normal[3 * r + k] = S.normal[3 * g + k];
    }
    for (int k = 0; k < 4; ++k) D.rot[4 * r + k] = S.rot[4 * g + k];
    D.raw_value[r] = S.raw_value[g];
    D.raw_weight[r] = S.raw_weight[g];
    D.raw_ka[r] = S.raw_ka[g];
    D.raw_kd[r] = S.raw_kd[g];
    D.raw_ks[r] = S.raw_ks[g];
    D.raw_beta[r] = S.raw_beta[g];
}

__device__ __forceinline__ void zero_row(double *dst, int64_t n_out, int64_t r) {
    GradView D(dst, n_out);
    for (int k = 0; k < 3; ++k) D.pos[3 * r + k] = D.log_scale[3 * r + k] = D.normal[3 * r + k] = 0.0;
    for (int k = 0; k < 4; ++k) D.rot[4 * r + k] = 0.0;
    D.raw_value[r] = D.raw_weight[r] = D.raw_ka[r] = D.raw_kd[r] = D.raw_ks[r] = D.raw_beta[r] = 0.0;
}

__global__ void densify_apply_kernel(const double *params, const double *m, const double *v, int64_t n,
                                     const double *stats, VegsDensify dp, const int4 *flags, const int4 *offs,
                                     const double *eps, int64_t n_out, double *out_params, double *out_m,
                                     double *out_v) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const int4 f = flags[g];
    if (!(f.x | f.y | f.z)) return;
    const int4 o = offs[g], tot = offs[n];
    const ParamView P(params, n);
    if (f.x) {
        copy_row(params, n, g, out_params, n_out, o.x);
        copy_row(m, n, g, out_m, n_out, o.x);
        copy_row(v, n, g, out_v, n_out, o.x);
    }
    if (f.y) {  // clone: step along the negative mean positional gradient (train.py:255-259)
        const int64_t r = (int64_t)tot.x + o.y;
        copy_row(params, n, g, out_params, n_out, r);
        zero_row(out_m, n_out, r);
        zero_row(out_v, n_out, r);
        const double cnt = fmax(stats[5 * g + 4], 1.0);
        double d[3], nn = 0.0;
        for (int k = 0; k < 3; ++k) {
            d[k] = stats[5 * g + 1 + k] / cnt;
            nn = nn + d[k] * d[k];
        }
        const double norm = sqrt(nn);
        GradView D(out_params, n_out);
        for (int k = 0; k < 3; ++k) {
            const double dir = norm > 0 ? d[k] / fmax(norm, 1e-30) : 0.0;
            D.pos[3 * r + k] = P.pos[3 * g + k] - dp.position_lr * dir;
        }
    }
    if (f.z) {  // split into two children (train.py:261-271)
        double q[4], qq = 0.0;
        for (int k = 0; k < 4; ++k) {
            q[k] = P.rot[4 * g + k];
            qq = qq + q[k] * q[k];
        }
        const double qn = sqrt(qq);
        for (int k = 0; k < 4; ++k) q[k] = q[k] / qn;
        const double w = q[0], x = q[1], y = q[2], z = q[3];
        const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                                {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                                {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
        double sc[3];
        for (int k = 0; k < 3; ++k) sc[k] = exp(P.log_scale[3 * g + k]);
        for (int round = 0; round < 2; ++round) {
            const int64_t r = (int64_t)tot.x + tot.y + (int64_t)round * tot.z + o.z;
            copy_row(params, n, g, out_params, n_out, r);
            zero_row(out_m, n_out, r);
            zero_row(out_v, n_out, r);
            const double *e = eps + ((int64_t)round * tot.w + o.w) * 3;
            GradView D(out_params, n_out);
            for (int i = 0; i < 3; ++i) {
                double off = 0.0;
                for (int j = 0; j < 3; ++j) off = off + R[i][j] * (sc[j] * e[j]);
                D.pos[3 * r + i] = P.pos[3 * g + i] + off;
                D.log_scale[3 * r + i] = P.log_scale[3 * g + i] - dp.log_split_factor;
            }
        }
    }
}

}  // namespace vegs

extern "C" int vegs_densify_count(const double *params, int64_t n, const double *stats, const VegsDensify *dp,
                                  int32_t *flags, int32_t *offsets, void *ws, size_t *ws_bytes, void *stream) {
    if (!ws_bytes || !dp) return VEGS_ERR_ARG;
    size_t scan_bytes = 0;
    int4 *dummy = nullptr;
    VEGS_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, scan_bytes, dummy, dummy, Int4Sum(), make_int4(0, 0, 0, 0),
                                             n + 1, (cudaStream_t)stream));
    if (!ws) {
        *ws_bytes = scan_bytes;
        return VEGS_OK;
    }
    if (*ws_bytes < scan_bytes) return VEGS_ERR_CAPACITY;
    if (n >= (int64_t(1) << 30) || !flags || !offsets || (n > 0 && (!params || !stats))) return VEGS_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    densify_classify_kernel<<<(int)((n + 1 + 255) / 256), 256, 0, s>>>(params, n, stats, *dp, (int4 *)flags);
    VEGS_CHECK_LAUNCH();
    VEGS_CUDA(cub::DeviceScan::ExclusiveScan(ws, scan_bytes, (int4 *)flags, (int4 *)offsets, Int4Sum(),
                                             make_int4(0, 0, 0, 0), n + 1, s));
    return VEGS_OK;
}

extern "C" int vegs_densify_apply(const double *params, const double *m, const double *v, int64_t n,
                                  const double *stats, const VegsDensify *dp, const int32_t *flags,
                                  const int32_t *offsets, const double *eps, int64_t n_out, double *out_params,
                                  double *out_m, double *out_v, void *stream) {
    if (!dp || (n > 0 && (!params || !m || !v || !stats || !flags || !offsets)) ||
        (n_out > 0 && (!out_params || !out_m || !out_v)))
        return VEGS_ERR_ARG;
    if (n == 0) return VEGS_OK;
    densify_apply_kernel<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        params, m, v, n, stats, *dp, (const int4 *)flags, (const int4 *)offsets, eps, n_out, out_params, out_m, out_v);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}
