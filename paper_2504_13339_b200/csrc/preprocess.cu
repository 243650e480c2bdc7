// Per-Gaussian preprocess (forward), TF lookup, Adam and densify/prune for sm_100a.
// The backward chain lives in preprocess_bwd.cu (compiled with FMA contraction).
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

#include "preprocess_common.cuh"

namespace vegs {

template <typename Real>
#ifndef VEGS_PFWD_T
#define VEGS_PFWD_T 256
#endif
#ifndef VEGS_PFWD_MINB
#define VEGS_PFWD_MINB 3  // 80 registers with the parameters in registers (ParamRegs): 0.131 -> 0.115 ms per c2 view (4: 0.126, 2: 0.127)
#endif
__global__ void __launch_bounds__(VEGS_PFWD_T, VEGS_PFWD_MINB) preprocess_fwd_kernel(
    const double *params, int64_t n, VegsCamera cam, VegsTF tf, VegsSettings st, int n_ch,
    VegsSplatTable out, const double *proj) {
    extern __shared__ double tf_smem[];
    const TFTable tab = stage_tf(tf, tf_smem);
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const ParamRegs P(ParamView(params, n), g);
    Shaded s;
    shade_one(P, g, tab, cam, st, s);
    if (out.alpha_base) out.alpha_base[g] = s.alpha_base;
    if (out.color)
        for (int c = 0; c < 3; ++c) out.color[3 * g + c] = s.color[c];
    if (out.visible) out.visible[g] = s.visible ? 1 : 0;
    bool kept = false;
    Projected p;
    if (s.visible) {
        if (proj) {  // the camera's projection from vegs_project (TF-independent), then the rect
            const double *c = proj + (int64_t)kProjStride * g;
            p.px = c[0];
            p.py = c[1];
            p.conic[0] = c[2];
            p.conic[1] = c[3];
            p.conic[2] = c[4];
            p.lam = c[5];
            p.t[2] = c[6];
            p.radius = st.radius_sigma * sqrt(fmax(p.lam, 0.0));
            project_rect(s.alpha_base, cam, st, c[7] != 0.0, p);
        } else {
            project_one(P, g, s.alpha_base, cam, st, p);
        }
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

// The TF-independent part of the preprocess for one camera (projection.py:43-176 up to the
// conic): px, py, conic, the footprint's major eigenvalue, view depth and the front / positive-
// definite flag, float64, kProjStride per Gaussian.  A sweep of several TFs through one camera
// projects once and each TF's preprocess only shades and takes the level-set rect
// (project_rect); the arithmetic is project_one's, so the tables are identical.
__global__ void __launch_bounds__(256) project_kernel(const double *params, int64_t n, VegsCamera cam,
                                                      VegsSettings st, double *proj) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const ParamView P(params, n);
    Projected p;
    project_one<false>(P, g, 0.0, cam, st, p);
    double *c = proj + (int64_t)kProjStride * g;
    c[0] = p.px;
    c[1] = p.py;
    c[2] = p.conic[0];
    c[3] = p.conic[1];
    c[4] = p.conic[2];
    c[5] = p.lam;
    c[6] = p.t[2];
    c[7] = p.keep ? 1.0 : 0.0;
}

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

// Adam over the class-major flat buffer.  blockIdx.y is the unit (0..18) of the 19 n
// layout, so the class is a table lookup, not a 64-bit division per element.  The step
// gradient is the sum of up to four per-stream partial buffers, added in a fixed order
// (((g0 + g1) + g2) + g3) and written back into g0 (the trainer's step gradient).
__constant__ int kUnitClass[19] = {0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 4, 5, 5, 5, 6, 7, 8, 9};

struct GradParts {
    double *g0;
    const double *g[3];
    int n_extra;
};

__global__ void __launch_bounds__(256) adam_kernel(double *params, GradParts gp, const float *pay32, double *m,
                                                   double *v, int64_t n, int unit0, const double *lr,
                                                   double grad_scale, double bias1, double bias2, int *nonfinite,
                                                   const int64_t *skip) {
    if (skip && skip[0]) return;  // a view of the step overflowed its buffers: the step is redone
    const int unit = unit0 + (int)blockIdx.y;
    const int cls = kUnitClass[unit];
    const double b1 = 0.9, b2 = 0.999, eps = 1e-15;
    const double lr_c = params ? lr[cls] : 0.0;
    if (params && bias1 != bias1) {  // NaN marks "from the device": lr[10], lr[11] hold 1 - beta^t (graph replay)
        bias1 = lr[10];
        bias2 = lr[11];
    }
    const int64_t base = (int64_t)unit * n;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + j;
        double gs;
        if (pay32) {  // the all-reduced float32 payload, widened (and kept as the step gradient)
            gs = (double)pay32[i];
            gp.g0[i] = gs;
        } else {
            gs = gp.g0[i];
        }
        if (!pay32 && gp.n_extra > 0) {
            for (int k = 0; k < gp.n_extra; ++k) gs = gs + gp.g[k][i];
            gp.g0[i] = gs;
        }
        if (!params) continue;  // sum only (before a cross-rank all-reduce)
        const double gr = gs * grad_scale;
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
        params[i] = params[i] - lr_c * upd;
    }
}

// Cross-rank exchange, first half: the lanes' partial gradients of units [unit0, unit0 +
// gridDim.y) summed in the Adam kernel's fixed order, into g0 (float64 payload) or into a
// float32 payload for the all-reduce.
__global__ void __launch_bounds__(256) grad_pack_kernel(GradParts gp, float *pay32, int64_t n, int unit0) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int64_t i = (int64_t)(unit0 + (int)blockIdx.y) * n + j;
    double gs = gp.g0[i];
    for (int k = 0; k < gp.n_extra; ++k) gs = gs + gp.g[k][i];
    if (pay32) pay32[i] = (float)gs;
    else if (gp.n_extra > 0) gp.g0[i] = gs;
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

static int preprocess_launch(const double *params, int64_t n, const VegsCamera *cam, const VegsTF *tf,
                             const VegsSettings *st, int32_t n_channels, int32_t store_f64, VegsSplatTable *out,
                             const double *proj, void *stream);

extern "C" int vegs_preprocess_forward(const double *params, int64_t n, const VegsCamera *cam,
                                       const VegsTF *tf, const VegsSettings *st, int32_t n_channels,
                                       int32_t store_f64, VegsSplatTable *out, void *stream) {
    return preprocess_launch(params, n, cam, tf, st, n_channels, store_f64, out, nullptr, stream);
}

extern "C" int vegs_project(const double *params, int64_t n, const VegsCamera *cam, const VegsSettings *st,
                            double *proj, void *stream) {
    if (!cam || !st || (n > 0 && (!params || !proj))) return VEGS_ERR_ARG;
    if (n == 0) return VEGS_OK;
    project_kernel<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(params, n, *cam, *st, proj);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" int vegs_preprocess_forward_projected(const double *params, int64_t n, const VegsCamera *cam,
                                                 const VegsTF *tf, const VegsSettings *st, int32_t n_channels,
                                                 int32_t store_f64, const double *proj, VegsSplatTable *out,
                                                 void *stream) {
    if ((n > 0 && !proj) || (out && out->aux)) return VEGS_ERR_ARG;  // aux views need the full projection
    return preprocess_launch(params, n, cam, tf, st, n_channels, store_f64, out, proj, stream);
}

static int preprocess_launch(const double *params, int64_t n, const VegsCamera *cam, const VegsTF *tf,
                             const VegsSettings *st, int32_t n_channels, int32_t store_f64, VegsSplatTable *out,
                             const double *proj, void *stream) {
    if (!cam || !st || !out || !tf_ok(tf) || (n > 0 && !params)) return VEGS_ERR_ARG;
    if (n_channels != 3 && n_channels != 11) return VEGS_ERR_ARG;
    if (st->tile_size != kTile) return VEGS_ERR_ARG;
    if (!out->record || !out->rect || !out->tiles || !out->depth_key) return VEGS_ERR_ARG;
    if (n == 0) return VEGS_OK;
    const size_t smem = tf_smem_bytes(*tf);
    cudaStream_t s = (cudaStream_t)stream;
    if (store_f64) {
        VEGS_CUDA(cudaFuncSetAttribute(preprocess_fwd_kernel<double>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        preprocess_fwd_kernel<double><<<(int)((n + VEGS_PFWD_T - 1) / VEGS_PFWD_T), VEGS_PFWD_T, smem, s>>>(params, n, *cam, *tf, *st, n_channels, *out, proj);
    } else {
        VEGS_CUDA(cudaFuncSetAttribute(preprocess_fwd_kernel<float>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        preprocess_fwd_kernel<float><<<(int)((n + VEGS_PFWD_T - 1) / VEGS_PFWD_T), VEGS_PFWD_T, smem, s>>>(params, n, *cam, *tf, *st, n_channels, *out, proj);
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

static int adam_launch(double *params, GradParts gp, double *m, double *v, int64_t n, const double *lr,
                       double grad_scale, double bias1, double bias2, int32_t *nonfinite, void *stream,
                       const int64_t *skip = nullptr, const float *pay32 = nullptr, int unit0 = 0,
                       int units = 19) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // one element per thread: every load of the step (4 gradient partials, params, m, v) in
    // flight at once across the grid (the grid-stride version capped at 8 CTAs per SM was
    // load-latency bound: 55% long-scoreboard stalls, 42% of HBM)
    const int bx = (int)((n + 255) / 256);
    (void)sms;
    adam_kernel<<<dim3(bx, units), 256, 0, (cudaStream_t)stream>>>(params, gp, pay32, m, v, n, unit0, lr,
                                                                   grad_scale, bias1, bias2, nonfinite, skip);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" int vegs_adam_step(double *params, const double *grads, double *m, double *v, int64_t n,
                              const double *lr, double grad_scale, double bias1, double bias2,
                              int32_t *nonfinite, void *stream) {
    if (n > 0 && (!params || !grads || !m || !v || !lr || !nonfinite)) return VEGS_ERR_ARG;
    if (n == 0) return VEGS_OK;
    GradParts gp{const_cast<double *>(grads), {nullptr, nullptr, nullptr}, 0};  // g0 is only read
    return adam_launch(params, gp, m, v, n, lr, grad_scale, bias1, bias2, nonfinite, stream);
}

extern "C" int vegs_adam_step_sum(double *params, double *grads0, const double *grads1, const double *grads2,
                                  const double *grads3, double *m, double *v, int64_t n, const double *hyper,
                                  double grad_scale, int32_t *nonfinite, const int64_t *skip, void *stream) {
    if (n > 0 && !grads0) return VEGS_ERR_ARG;
    if (n > 0 && params && (!m || !v || !hyper || !nonfinite)) return VEGS_ERR_ARG;
    const double *extra[3] = {grads1, grads2, grads3};
    GradParts gp{grads0, {nullptr, nullptr, nullptr}, 0};
    for (int k = 0; k < 3; ++k)
        if (extra[k]) gp.g[gp.n_extra++] = extra[k];
    if (n == 0 || (!params && gp.n_extra == 0)) return VEGS_OK;
    return adam_launch(params, gp, m, v, n, hyper, grad_scale, NAN, NAN, nonfinite, stream, skip);
}

extern "C" int vegs_grad_pack(double *grads0, const double *grads1, const double *grads2, const double *grads3,
                              float *payload32, int64_t n, int32_t unit0, int32_t units, void *stream) {
    if (unit0 < 0 || units < 0 || unit0 + units > 19) return VEGS_ERR_ARG;
    if (n > 0 && units > 0 && !grads0) return VEGS_ERR_ARG;
    const double *extra[3] = {grads1, grads2, grads3};
    GradParts gp{grads0, {nullptr, nullptr, nullptr}, 0};
    for (int k = 0; k < 3; ++k)
        if (extra[k]) gp.g[gp.n_extra++] = extra[k];
    if (n == 0 || units == 0 || (!payload32 && gp.n_extra == 0)) return VEGS_OK;
    grad_pack_kernel<<<dim3((unsigned)((n + 255) / 256), units), 256, 0, (cudaStream_t)stream>>>(gp, payload32, n,
                                                                                                 unit0);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" int vegs_adam_step_range(double *params, double *grads0, const float *payload32, double *m, double *v,
                                    int64_t n, int32_t unit0, int32_t units, const double *hyper,
                                    int32_t *nonfinite, const int64_t *skip, void *stream) {
    if (unit0 < 0 || units < 0 || unit0 + units > 19) return VEGS_ERR_ARG;
    if (n > 0 && units > 0 && (!params || !grads0 || !m || !v || !hyper || !nonfinite)) return VEGS_ERR_ARG;
    if (n == 0 || units == 0) return VEGS_OK;
    GradParts gp{grads0, {nullptr, nullptr, nullptr}, 0};
    return adam_launch(params, gp, m, v, n, hyper, 1.0, NAN, NAN, nonfinite, stream, skip, payload32, unit0, units);
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

// Max over transfer functions of the opacity map at each Gaussian's value (BASELINE config
// 4's prune criterion "max TF opacity < 0.005"): out[g] = max(out[g], O_tf(sigmoid(raw_value)))
// (init: out[g] = O_tf(...)), np.interp semantics as eval_opacity (transfer.py:91-95).
__global__ void tf_max_opacity_kernel(const double *params, int64_t n, VegsTF tf, int init, double *out) {
    extern __shared__ double s_tf[];
    for (int i = threadIdx.x; i < 2 * tf.n_opacity; i += blockDim.x) s_tf[i] = tf.blob[i];
    __syncthreads();
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const ParamView P(params, n);
    const double o = tf_interp(s_tf, s_tf + tf.n_opacity, tf.n_opacity, clip01(sigmoid(P.raw_value[g])));
    out[g] = init ? o : fmax(out[g], o);
}

__device__ __forceinline__ void densify_flags(const ParamView &P, int64_t g, const double *stats,
                                              const VegsDensify &dp, bool &small, bool &big, bool &survive) {
    const double cnt = fmax(stats[5 * g + 4], 1.0);
    const bool cand = stats[5 * g] / cnt > dp.grad_threshold;
    double ms = exp(P.log_scale[3 * g]);
    ms = fmax(ms, exp(P.log_scale[3 * g + 1]));
    ms = fmax(ms, exp(P.log_scale[3 * g + 2]));
    small = cand && ms <= dp.percent_dense * dp.scene_extent;
    big = cand && !small;
    // prune rule: the reference's activated weight (train.py:277-280), or BASELINE config 4's
    // max TF opacity over the training TFs (dp.prune_opacity, from vegs_tf_max_opacity)
    survive = dp.no_weights ||
              (dp.prune_opacity ? dp.prune_opacity[g] >= dp.prune_threshold
                                : sigmoid(P.raw_weight[g]) >= dp.prune_threshold);
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

extern "C" int vegs_tf_max_opacity(const double *params, int64_t n, const VegsTF *tf, int32_t init, double *out,
                                   void *stream) {
    if (!tf_ok(tf) || (n > 0 && (!params || !out))) return VEGS_ERR_ARG;
    if (n == 0) return VEGS_OK;
    const size_t smem = sizeof(double) * 2 * (size_t)tf->n_opacity;
    VEGS_CUDA(cudaFuncSetAttribute(tf_max_opacity_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    tf_max_opacity_kernel<<<(int)((n + 255) / 256), 256, smem, (cudaStream_t)stream>>>(params, n, *tf, init, out);
    VEGS_CHECK_LAUNCH();
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
