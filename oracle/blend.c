/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle, never linked into the product.
 *
 * Plain-C restatement of the reference's two numba tile kernels:
 *   blend_forward   /root/reference/pkg/src/vegsplat/raster/kernels.py:26-100
 *   blend_backward  /root/reference/pkg/src/vegsplat/raster/kernels.py:103-208
 *
 * Precision follows the numba typing of the reference exactly:
 * the per-pixel offsets dx, dy are float64 (an int + 0.5 minus a stored mean), so the
 * exponent pw, exp(pw), alpha, the transmittance test and the blend weight are float64;
 * the transmittance T, the output planes and the per-instance gradient slots are
 * stored in the blend storage type STORE (float for training, double for tests), and
 * the backward dot products dot_ug / dot_sg / hterm stay in STORE arithmetic.  The
 * numba kernels are fastmath; here we keep IEEE order (-ffp-contract=off), which only
 * moves results at the last-ulp level.
 *
 * One extra output over the reference: n_contrib, the number of instances blended at
 * each pixel (the "contributor count" the north star pins bit-exact).
 *
 * Tiles are independent (a tile owns its pixels and instance slots), so the tile loop
 * is an OpenMP parallel-for like the reference's prange.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEFINE_BLEND(SUFFIX, STORE)                                                        \
void oracle_blend_forward_##SUFFIX(                                                        \
    const int64_t *tile_start, const int64_t *tile_end, int64_t n_tiles, int64_t tiles_x,  \
    int64_t tile_size, const STORE *mean2d, const STORE *conic, const STORE *alpha_b,      \
    const STORE *pmin, const int32_t *rect, const STORE *channels, int64_t n_ch,           \
    const STORE *bg, int64_t width, int64_t height, STORE alpha_clamp, STORE trans_stop,   \
    STORE *out_img, STORE *out_t, int64_t *out_last, int32_t *n_contrib)                   \
{                                                                                          \
    _Pragma("omp parallel for schedule(dynamic, 1)")                                       \
    for (int64_t tile = 0; tile < n_tiles; ++tile) {                                       \
        const int64_t ty = tile / tiles_x, tx = tile % tiles_x;                            \
        const int64_t x_lo = tx * tile_size, y_lo = ty * tile_size;                        \
        const int64_t x_hi = x_lo + tile_size < width ? x_lo + tile_size : width;          \
        const int64_t y_hi = y_lo + tile_size < height ? y_lo + tile_size : height;        \
        const int64_t tw = x_hi - x_lo;                                                    \
        STORE T[256 * 4];                                                                  \
        unsigned char fin[256 * 4];                                                        \
        STORE *tloc = tile_size * tile_size <= 1024 ? T                                    \
                      : (STORE *)malloc(sizeof(STORE) * tile_size * tile_size);            \
        unsigned char *done = tile_size * tile_size <= 1024 ? fin                          \
                      : (unsigned char *)malloc(tile_size * tile_size);                    \
        for (int64_t y = y_lo; y < y_hi; ++y)                                              \
            for (int64_t x = x_lo; x < x_hi; ++x) {                                        \
                int64_t l = (y - y_lo) * tw + (x - x_lo);                                  \
                tloc[l] = (STORE)1; done[l] = 0;                                           \
                out_last[y * width + x] = -1; n_contrib[y * width + x] = 0;                \
                for (int64_t c = 0; c < n_ch; ++c) out_img[(y * width + x) * n_ch + c] = 0;\
            }                                                                              \
        for (int64_t i = tile_start[tile]; i < tile_end[tile]; ++i) {                      \
            const int32_t *r = rect + 4 * i;                                               \
            int64_t x0 = r[0] > x_lo ? r[0] : x_lo, x1 = r[1] < x_hi ? r[1] : x_hi;        \
            int64_t y0 = r[2] > y_lo ? r[2] : y_lo, y1 = r[3] < y_hi ? r[3] : y_hi;        \
            if (x0 >= x1 || y0 >= y1) continue;                                            \
            const double ca = conic[3 * i], cb = conic[3 * i + 1], cc = conic[3 * i + 2];  \
            const double mx = mean2d[2 * i], my = mean2d[2 * i + 1];                       \
            const double ab = alpha_b[i], pm = pmin[i];                                    \
            for (int64_t y = y0; y < y1; ++y) {                                            \
                const double dy = ((double)y + 0.5) - my;                                  \
                for (int64_t x = x0; x < x1; ++x) {                                        \
                    const int64_t l = (y - y_lo) * tw + (x - x_lo);                        \
                    if (done[l]) continue;                                                 \
                    const double dx = ((double)x + 0.5) - mx;                              \
                    const double pw = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy; \
                    if (pw < pm) continue;                                                 \
                    double a = ab * exp(pw);                                               \
                    if (a > (double)alpha_clamp) a = (double)alpha_clamp;                  \
                    const STORE t = tloc[l];                                               \
                    const double test_t = (double)t * ((double)(STORE)1 - a);              \
                    if (test_t < (double)trans_stop) { done[l] = 1; continue; }            \
                    const double wgt = a * (double)t;                                      \
                    STORE *o = out_img + (y * width + x) * n_ch;                           \
                    for (int64_t c = 0; c < n_ch; ++c)                                     \
                        o[c] = (STORE)((double)o[c] + (double)channels[i * n_ch + c] * wgt);\
                    tloc[l] = (STORE)test_t;                                               \
                    out_last[y * width + x] = i;                                           \
                    n_contrib[y * width + x] += 1;                                         \
                }                                                                          \
            }                                                                              \
        }                                                                                  \
        for (int64_t y = y_lo; y < y_hi; ++y)                                              \
            for (int64_t x = x_lo; x < x_hi; ++x) {                                        \
                const STORE t = tloc[(y - y_lo) * tw + (x - x_lo)];                        \
                STORE *o = out_img + (y * width + x) * n_ch;                               \
                for (int64_t c = 0; c < n_ch; ++c) o[c] = o[c] + t * bg[c];                \
                out_t[y * width + x] = t;                                                  \
            }                                                                              \
        if (tloc != T) free(tloc);                                                         \
        if (done != fin) free(done);                                                       \
    }                                                                                      \
}                                                                                          \
                                                                                           \
void oracle_blend_backward_##SUFFIX(                                                       \
    const int64_t *tile_start, const int64_t *tile_end, int64_t n_tiles, int64_t tiles_x,  \
    int64_t tile_size, const STORE *mean2d, const STORE *conic, const STORE *alpha_b,      \
    const STORE *pmin, const int32_t *rect, const STORE *channels, int64_t n_ch,           \
    const STORE *bg, int64_t width, int64_t height, STORE alpha_clamp,                     \
    const STORE *out_t, const int64_t *out_last, const STORE *d_img,                       \
    const STORE *d_alpha_plane, STORE *g_mean2d, STORE *g_conic, STORE *g_alpha,           \
    STORE *g_channels)                                                                     \
{                                                                                          \
    _Pragma("omp parallel for schedule(dynamic, 1)")                                       \
    for (int64_t tile = 0; tile < n_tiles; ++tile) {                                       \
        const int64_t ty = tile / tiles_x, tx = tile % tiles_x;                            \
        const int64_t x_lo = tx * tile_size, y_lo = ty * tile_size;                        \
        const int64_t x_hi = x_lo + tile_size < width ? x_lo + tile_size : width;          \
        const int64_t y_hi = y_lo + tile_size < height ? y_lo + tile_size : height;        \
        const int64_t tw = x_hi - x_lo, np_ = tw * (y_hi - y_lo);                          \
        STORE *tloc = (STORE *)malloc(sizeof(STORE) * np_);                                \
        STORE *hterm = (STORE *)malloc(sizeof(STORE) * np_);                               \
        STORE *suffix = (STORE *)calloc(np_ * n_ch, sizeof(STORE));                        \
        for (int64_t y = y_lo; y < y_hi; ++y)                                              \
            for (int64_t x = x_lo; x < x_hi; ++x) {                                        \
                const int64_t l = (y - y_lo) * tw + (x - x_lo), p = y * width + x;         \
                const STORE tn = out_t[p];                                                 \
                STORE gb = 0;                                                              \
                for (int64_t c = 0; c < n_ch; ++c) gb = gb + d_img[p * n_ch + c] * bg[c];  \
                tloc[l] = tn;                                                              \
                hterm[l] = (gb - d_alpha_plane[p]) * tn;                                   \
            }                                                                              \
        for (int64_t i = tile_end[tile] - 1; i >= tile_start[tile]; --i) {                 \
            const int32_t *r = rect + 4 * i;                                               \
            int64_t x0 = r[0] > x_lo ? r[0] : x_lo, x1 = r[1] < x_hi ? r[1] : x_hi;        \
            int64_t y0 = r[2] > y_lo ? r[2] : y_lo, y1 = r[3] < y_hi ? r[3] : y_hi;        \
            if (x0 >= x1 || y0 >= y1) continue;                                            \
            const double ca = conic[3 * i], cb = conic[3 * i + 1], cc = conic[3 * i + 2];  \
            const double mx = mean2d[2 * i], my = mean2d[2 * i + 1];                       \
            const double ab = alpha_b[i], pm = pmin[i];                                    \
            double s_a = 0, s_mx = 0, s_my = 0, s_ca = 0, s_cb = 0, s_cc = 0;              \
            for (int64_t y = y0; y < y1; ++y) {                                            \
                const double dy = ((double)y + 0.5) - my;                                  \
                for (int64_t x = x0; x < x1; ++x) {                                        \
                    const int64_t p = y * width + x, l = (y - y_lo) * tw + (x - x_lo);     \
                    if (out_last[p] < i) continue;                                         \
                    const double dx = ((double)x + 0.5) - mx;                              \
                    const double pw = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy; \
                    if (pw < pm) continue;                                                 \
                    const double fall = exp(pw);                                           \
                    double a = ab * fall;                                                  \
                    const int clamped = a > (double)alpha_clamp;                           \
                    if (clamped) a = (double)alpha_clamp;                                  \
                    const double om = (double)(STORE)1 - a;                                \
                    const double ti = (double)tloc[l] / om;                                \
                    const double wgt = a * ti;                                             \
                    STORE dug = 0, dsg = 0;                                                \
                    for (int64_t c = 0; c < n_ch; ++c) {                                   \
                        const STORE gc = d_img[p * n_ch + c];                              \
                        const STORE u = channels[i * n_ch + c];                            \
                        STORE *gch = g_channels + i * n_ch + c;                            \
                        *gch = (STORE)((double)*gch + (double)gc * wgt);                   \
                        dug = dug + u * gc;                                                \
                        dsg = dsg + suffix[l * n_ch + c] * gc;                             \
                        suffix[l * n_ch + c] =                                             \
                            (STORE)((double)suffix[l * n_ch + c] + (double)u * wgt);       \
                    }                                                                      \
                    if (!clamped) {                                                        \
                        const double da = ti * (double)dug - (double)(dsg + hterm[l]) / om;\
                        s_a += da * fall;                                                  \
                        const double dpw = da * a;                                         \
                        s_mx += dpw * (ca * dx + cb * dy);                                 \
                        s_my += dpw * (cc * dy + cb * dx);                                 \
                        s_ca += dpw * (-0.5 * dx * dx);                                    \
                        s_cb += dpw * (-dx * dy);                                          \
                        s_cc += dpw * (-0.5 * dy * dy);                                    \
                    }                                                                      \
                    tloc[l] = (STORE)ti;                                                   \
                }                                                                          \
            }                                                                              \
            g_alpha[i] = (STORE)s_a;                                                       \
            g_mean2d[2 * i] = (STORE)s_mx; g_mean2d[2 * i + 1] = (STORE)s_my;              \
            g_conic[3 * i] = (STORE)s_ca; g_conic[3 * i + 1] = (STORE)s_cb;                \
            g_conic[3 * i + 2] = (STORE)s_cc;                                              \
        }                                                                                  \
        free(tloc); free(hterm); free(suffix);                                             \
    }                                                                                      \
}

DEFINE_BLEND(f32, float)
DEFINE_BLEND(f64, double)

/* Per-splat reduction of per-instance rows in sorted-instance order, float64
 * accumulation: the restatement of np.add.at at pipeline.py:307-316. */
void oracle_scatter_add(const int64_t *order, int64_t n_inst, const double *rows, int64_t width,
                        double *out)
{
    for (int64_t s = 0; s < n_inst; ++s)
        for (int64_t c = 0; c < width; ++c) out[order[s] * width + c] += rows[s * width + c];
}
