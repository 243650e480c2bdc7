// Per-Gaussian device helpers shared by the preprocess (forward, -fmad=false) and the
// preprocess backward (FMA contraction allowed) translation units: TF lookup, shading,
// projection, record layout.  Header-only: every includer compiles its own copy with
// its own floating-point contraction setting.
#pragma once

#include <math.h>

#include "vegs_common.cuh"

namespace vegs {
namespace {  // internal linkage: each translation unit compiles its own copy


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

// The same segment from a guess: for (near-)uniform knots j = floor((x - ts[0]) / dt) is
// exact or one off, and one step each way settles it; anything else falls back to the
// binary search, so the result is the binary search's for any sorted knots.  x >= ts[0].
__device__ __forceinline__ int knot_segment_g(const double *ts, int k, double x, double inv_dt) {
    int j = (int)((x - ts[0]) * inv_dt);
    j = j < 0 ? 0 : (j > k - 1 ? k - 1 : j);
    if (ts[j] > x) {
        --j;
        if (ts[j] > x) return knot_segment(ts, k, x);
    } else if (j + 1 < k && ts[j + 1] <= x) {
        ++j;
        if (j + 1 < k && ts[j + 1] <= x) return knot_segment(ts, k, x);
    }
    return j;
}

__device__ __forceinline__ double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

// np.interp at x on the segment j found for x (x inside [ts[0], ts[k-1]])
__device__ __forceinline__ double interp_on(const double *ts, const double *vals, int k, int j, double x) {
    if (j == k - 1 || ts[j] == x) return vals[j];
    const double slope = (vals[j + 1] - vals[j]) / (ts[j + 1] - ts[j]);
    return slope * (x - ts[j]) + vals[j];
}

__device__ double tf_interp(const double *ts, const double *vals, int k, double x) {
    if (x != x) return x;
    if (x < ts[0]) return vals[0];
    if (x > ts[k - 1]) return vals[k - 1];
    return interp_on(ts, vals, k, knot_segment(ts, k, x), x);
}

__device__ double tf_slope(const double *ts, const double *vals, int k, double x) {
    int j = (x < ts[0]) ? -1 : knot_segment(ts, k, x);
    j = j < 0 ? 0 : (j > k - 2 ? k - 2 : j);
    return (vals[j + 1] - vals[j]) / (ts[j + 1] - ts[j]);
}

// segment index of the half-open slope convention (tf_slope) for the table's knots
__device__ __forceinline__ int slope_segment(const double *ts, int k, double x, double inv_dt) {
    int j = (x < ts[0]) ? -1 : knot_segment_g(ts, k, x, inv_dt);
    return j < 0 ? 0 : (j > k - 2 ? k - 2 : j);
}

__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

// TF tables staged in shared memory: [ts_op | op | ts_col | r | g | b]
struct TFTable {
    const double *ts_op, *op, *ts_col, *rgb[3];
    int k_op, k_col;
    double inv_op, inv_col;  // (k - 1) / (ts[k-1] - ts[0]): the uniform-spacing segment guess
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
    const double sop = t.ts_op[t.k_op - 1] - t.ts_op[0], scol = t.ts_col[t.k_col - 1] - t.ts_col[0];
    t.inv_op = sop > 0.0 ? (t.k_op - 1) / sop : 0.0;
    t.inv_col = scol > 0.0 ? (t.k_col - 1) / scol : 0.0;
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

// One Gaussian's 19 parameters loaded up front (read-only path, all loads in flight
// together) behind ParamView's indexing: P.pos[3 * g + k] etc. read registers.  Kernels
// that store (record, table) between parameter reads otherwise serialise the loads behind
// the stores (the compiler must assume they may alias).
template <int N>
struct RegArr {
    double v[N];
};
struct ParamRegs {
    RegArr<3> pos, log_scale, normal;
    RegArr<4> rot;
    RegArr<1> raw_value, raw_weight, raw_ka, raw_kd, raw_ks, raw_beta;
    __device__ __forceinline__ ParamRegs(const ParamView &P, int64_t g) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            pos.v[k] = __ldg(P.pos + 3 * g + k);
            log_scale.v[k] = __ldg(P.log_scale + 3 * g + k);
            normal.v[k] = __ldg(P.normal + 3 * g + k);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) rot.v[k] = __ldg(P.rot + 4 * g + k);
        raw_value.v[0] = __ldg(P.raw_value + g);
        raw_weight.v[0] = __ldg(P.raw_weight + g);
        raw_ka.v[0] = __ldg(P.raw_ka + g);
        raw_kd.v[0] = __ldg(P.raw_kd + g);
        raw_ks.v[0] = __ldg(P.raw_ks + g);
        raw_beta.v[0] = __ldg(P.raw_beta + g);
    }
};
// component k of Gaussian g's parameter (w values per Gaussian), from memory or registers
__device__ __forceinline__ double pget(const double *a, int64_t g, int w, int k) { return a[w * g + k]; }
template <int N>
__device__ __forceinline__ double pget(const RegArr<N> &a, int64_t, int, int k) { return a.v[k]; }

template <class PV>
__device__ void shade_one(const PV &P, int64_t g, const TFTable &tf, const VegsCamera &cam,
                          const VegsSettings &st, Shaded &s) {
    s.v = sigmoid(pget(P.raw_value, g, 1, 0));
    s.w = sigmoid(pget(P.raw_weight, g, 1, 0));
    const double vc = clip01(s.v);
    // np.interp on both maps (the three colour channels share one segment search)
    if (vc != vc) {
        s.op = vc;
        for (int c = 0; c < 3; ++c) s.cmap[c] = vc;
    } else {
        if (vc < tf.ts_op[0]) s.op = tf.op[0];
        else if (vc > tf.ts_op[tf.k_op - 1]) s.op = tf.op[tf.k_op - 1];
        else s.op = interp_on(tf.ts_op, tf.op, tf.k_op, knot_segment_g(tf.ts_op, tf.k_op, vc, tf.inv_op), vc);
        if (vc < tf.ts_col[0]) {
            for (int c = 0; c < 3; ++c) s.cmap[c] = tf.rgb[c][0];
        } else if (vc > tf.ts_col[tf.k_col - 1]) {
            for (int c = 0; c < 3; ++c) s.cmap[c] = tf.rgb[c][tf.k_col - 1];
        } else {
            const int j = knot_segment_g(tf.ts_col, tf.k_col, vc, tf.inv_col);
            for (int c = 0; c < 3; ++c) s.cmap[c] = interp_on(tf.ts_col, tf.rgb[c], tf.k_col, j, vc);
        }
    }
    s.alpha_base = s.op * s.w;
    double d[3], nn2 = 0.0, dd2 = 0.0;
    for (int k = 0; k < 3; ++k) {
        d[k] = cam.position[k] - pget(P.pos, g, 3, k);
        dd2 = dd2 + d[k] * d[k];
    }
    s.dist = sqrt(dd2);
    for (int k = 0; k < 3; ++k) s.light[k] = d[k] / s.dist;
    for (int k = 0; k < 3; ++k) nn2 = nn2 + pget(P.normal, g, 3, k) * pget(P.normal, g, 3, k);
    s.n_norm = sqrt(nn2);
    const double nd = fmax(s.n_norm, 1e-30);
    s.ndotl = 0.0;
    for (int k = 0; k < 3; ++k) {
        s.n_hat[k] = pget(P.normal, g, 3, k) / nd;
        s.ndotl = s.ndotl + s.n_hat[k] * s.light[k];
    }
    const double sa = fabs(s.ndotl);
    s.ka = sigmoid(pget(P.raw_ka, g, 1, 0));
    s.kd = sigmoid(pget(P.raw_kd, g, 1, 0));
    s.ks = sigmoid(pget(P.raw_ks, g, 1, 0));
    s.beta = fmin(fmax(exp(pget(P.raw_beta, g, 1, 0)), kBetaMin), kBetaMax);
    s.spec = sa > 0.0 ? pow(fmax(sa, 1e-300), s.beta) : 0.0;
    const double diffuse = s.ka + s.kd * sa;
    const double specular = s.ks * s.spec;
    for (int c = 0; c < 3; ++c) s.color[c] = diffuse * s.cmap[c] + specular;
    s.visible = s.alpha_base >= st.cull_alpha;
}

__device__ __forceinline__ void project_rect(double alpha_base, const VegsCamera &cam, const VegsSettings &st,
                                             bool front_ok, Projected &p);

template <bool kRect = true, class PV>
__device__ void project_one(const PV &P, int64_t g, double alpha_base, const VegsCamera &cam,
                            const VegsSettings &st, Projected &p) {
    const double *W = cam.rot;
    double d[3];
    for (int k = 0; k < 3; ++k) d[k] = pget(P.pos, g, 3, k) - cam.position[k];
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
        q[k] = pget(P.rot, g, 4, k);
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
        p.scale[k] = exp(pget(P.log_scale, g, 3, k));
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
    project_rect(alpha_base, cam, st, front && (p.det > 0), p);
}

// The level-set rectangle of a projected splat and its keep flag (the TF-dependent tail of
// project_one: the radius follows the activated opacity).  front_ok = in front of the near
// plane with a positive-definite footprint.
__device__ __forceinline__ void project_rect(double alpha_base, const VegsCamera &cam, const VegsSettings &st,
                                             bool front_ok, Projected &p) {
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
    p.keep = front_ok && (p.x1 > p.x0) && (p.y1 > p.y0) && finite;
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


static inline size_t tf_smem_bytes(const VegsTF &tf) {
    return sizeof(double) * (size_t)(2 * tf.n_opacity + 4 * tf.n_color);
}

static inline bool tf_ok(const VegsTF *tf) {
    return tf && tf->blob && tf->n_opacity >= 2 && tf->n_color >= 2 && tf->n_opacity <= VEGS_MAX_KNOTS &&
           tf->n_color <= VEGS_MAX_KNOTS;
}

}  // namespace
}  // namespace vegs
