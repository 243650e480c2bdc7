/*
 * vegsplat_b200 -- C-ABI of the B200-native differentiable VEG rasteriser.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t passed as
 * void*, never throws, and returns an int status (VEGS_OK or a negative error).  All
 * memory is owned by the caller (the Python host allocates it as torch tensors);
 * functions needing scratch follow the CUB convention: call once with ws == NULL to
 * receive the byte count in *ws_bytes.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/vegsplat/):
 *   vegs_blend_forward          raster/kernels.py:26-100  blend_forward(...)      (same arguments)
 *   vegs_blend_backward         raster/kernels.py:103-208 blend_backward(...)     (same arguments)
 *   vegs_preprocess_forward     raster/shading.py:52-82 shade + raster/projection.py:69-176 project
 *                               + raster/pipeline.py:137-160 build_splat_data, pipeline.py:207-215 (pmin,
 *                               f32 instance cast)
 *   vegs_bin_count / vegs_bin_sort
 *   vegs_bin_count_dev / _sort_dev  the same with the counts kept on the device (graph capture)
 *                               raster/pipeline.py:163-194 _build_instances (repeat + lexsort + searchsorted)
 *   vegs_composite_forward      raster/pipeline.py:197-237 rasterize_forward (tile blend on the splat table)
 *   vegs_composite_forward_fast the same with T carried in float32 (exact decisions; training / render path)
 *   vegs_composite_backward     raster/pipeline.py:291-305 (blend_backward on the splat table, per-instance
 *                               rows written in duplicate order for the deterministic reduction)
 *   vegs_preprocess_backward    raster/pipeline.py:307-366 (np.add.at reduction, project_backward
 *                               projection.py:186-277, shade_backward shading.py:97-176, GradientSet)
 *   vegs_loss_l1_ssim           loss.py:80-168 ssim / ssim_backward / compute_loss (L1 + SSIM part)
 *   vegs_loss_aux               loss.py:175-240 normal-consistency + bilateral-smoothness regularisers
 *   vegs_adam_step              train.py:176-195 adam_step (+ learning_rates :156-173 on the host)
 *   vegs_adam_step_sum          the same on the sum of the trainer's per-lane gradient buffers
 *   vegs_grad_pack / vegs_adam_step_range  the view-sharded step's gradient exchange (no reference
 *                               counterpart: the reference is single-process), bucketed by unit
 *   vegs_tf_eval                transfer.py:91-127 eval_opacity / eval_color / d_*_dv
 *   vegs_densify_count / _apply train.py:237-284 densify_and_prune (+ DensifyStats.add :210-214,
 *                               fused into vegs_preprocess_backward)
 *   vegs_tf_max_opacity         BASELINE config 4's prune criterion (max TF opacity per Gaussian)
 *
 * Test switches (environment, read at each launch; results are identical either way):
 *   VEGS_GENERIC_COMPOSITE=1  float32 compositing on the one-pixel kernels instead of the
 *                             two-pixel forward / four-pixel backward (cross-checks)
 *   VEGS_BIN_RADIX=1          binning by duplication + radix sort instead of counting
 *                             placement (the path views above 12288 tiles always take)
 *   VEGS_FAST_T_DEFER_ALL=1   vegs_composite_forward_fast hands every terminating pixel to its
 *                             float64 fix-up pass (exercises the fix-up)
 *   VEGS_PLACE_FLAT=1 / =0    counting placement in one level / in two levels (4x4-tile blocks,
 *                             then per-tile runs) regardless of the tile count (default: two
 *                             levels from 4096 tiles); the tile lists are identical
 *   VEGS_SMALL_SORT=0         the device-wide depth sort even for <= 16384 keys (default: one CTA)
 */
#ifndef VEGSPLAT_B200_H
#define VEGSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VEGS_OK 0
#define VEGS_ERR_ARG (-1)      /* bad argument (null pointer, unsupported size/tile/channels) */
#define VEGS_ERR_CUDA (-2)     /* a CUDA launch or runtime call failed */
#define VEGS_ERR_CAPACITY (-3) /* caller buffer too small */

#define VEGS_MAX_KNOTS 1024

/* Per-view camera constants, computed on the host exactly as camera.py:54-90 does. */
typedef struct {
    double position[3];
    double rot[9];   /* world->camera rows: right, up, forward (positive depth in front) */
    double focal;    /* 0.5 * height / tan(fov_y / 2) */
    double tan_x;    /* tan(fov_y / 2) * width / height */
    double tan_y;    /* tan(fov_y / 2) */
    double near_z;
    int32_t width;
    int32_t height;
} VegsCamera;

/* raster/constants.py:15-25 */
typedef struct {
    double dilation;
    double alpha_clamp;
    double alpha_skip;
    double transmittance_stop;
    double radius_sigma;
    double rect_margin_px;
    double cull_alpha;
    double frustum_limit;
    int32_t tile_size; /* must be 16: one 256-thread CTA per tile */
    int32_t pad_;
} VegsSettings;

/* Transfer-function knot blob (transfer.py:30-88), float64:
 * [ts_op(n_op) | op(n_op) | ts_col(n_col) | r(n_col) | g(n_col) | b(n_col)] */
typedef struct {
    const double *blob;
    int32_t n_opacity;
    int32_t n_color;
} VegsTF;

/* Per-Gaussian splat table written by vegs_preprocess_forward (n entries, indexed by
 * Gaussian id; entries of culled Gaussians are left untouched except tiles = 0).
 * record: n x rec_stride values of the blend storage type (float or double):
 *   [mx, my, conic_a, conic_b, conic_c, alpha_base, pmin, ch_0 .. ch_{C-1}, pad]
 * rec_stride = round_up(7 + C, 4). */
typedef struct {
    void *record;            /* float or double, see store_f64 */
    int32_t *rect;           /* n x 4: x0, x1, y0, y1 (exclusive ends) */
    uint32_t *tiles;         /* n: tiles touched (0 = not kept) */
    uint64_t *depth_key;     /* n: order-preserving key of the float64 depth (UINT64 max when not kept) */
    /* optional float64 views for the reference-shaped API (NULL to skip) */
    double *mean2d;          /* n x 2 */
    double *conic;           /* n x 3 */
    double *depth;           /* n */
    double *alpha_base;      /* n (written for every Gaussian, kept or not) */
    double *color;           /* n x 3 shaded colour (every Gaussian) */
    double *radius;          /* n */
    uint8_t *visible;        /* n: alpha_base >= cull (shading.py:75) */
    double *aux;             /* n x 24 shading / projection caches (ShadeResult, ProjectResult):
                                v, w, opacity, cmap[3], light[3], light_dist, n_hat[3], n_norm, ndotl,
                                ka, kd, ks, beta, spec_pow, cov2d[3] (a, b, c incl. dilation), pad */
} VegsSplatTable;

/* ---- TF lookup (tests / host API) ------------------------------------------------- */
int vegs_tf_eval(const double *ts, const double *vals, int32_t n_knots, int32_t n_cols,
                 const double *query, int64_t n_query, int32_t derivative, double *out,
                 void *stream);

/* ---- preprocess ------------------------------------------------------------------- */
int vegs_preprocess_forward(const double *params, int64_t n, const VegsCamera *cam,
                            const VegsTF *tf, const VegsSettings *st, int32_t n_channels,
                            int32_t store_f64, VegsSplatTable *out, void *stream);

/* The TF-independent half of the preprocess for one camera: proj (n x 8 float64: px, py,
 * conic a b c, the footprint's major eigenvalue, view depth, front/positive-definite flag).
 * vegs_preprocess_forward_projected = vegs_preprocess_forward taking that projection instead
 * of recomputing it (a sweep of several TFs through one camera projects once); identical
 * tables.  out->aux must be NULL there. */
int vegs_project(const double *params, int64_t n, const VegsCamera *cam, const VegsSettings *st, double *proj,
                 void *stream);
int vegs_preprocess_forward_projected(const double *params, int64_t n, const VegsCamera *cam, const VegsTF *tf,
                                      const VegsSettings *st, int32_t n_channels, int32_t store_f64,
                                      const double *proj, VegsSplatTable *out, void *stream);

/* Splat table from already-projected splats (the reference's SplatData, pipeline.py:40-49):
 * m rows of float64 mean2d (m x 2), conic (m x 3), alpha_base, depth, channels (m x C) and
 * int32 rect (m x 4).  Every row counts as kept.  Same record / key layout as above. */
int vegs_splat_table_from_arrays(const double *mean2d, const double *conic, const double *alpha_base,
                                 const double *depth, const int32_t *rect, const double *channels,
                                 int64_t m, const VegsSettings *st, int32_t n_channels, int32_t store_f64,
                                 VegsSplatTable *out, void *stream);

/* ---- binning ---------------------------------------------------------------------- */
/* Scan of (kept, tiles): offsets[n+1] (instance offset per Gaussian, duplicate order),
 * kept_idx[n+1] (index in the kept list), counts[2] = {n_kept, n_instances} (device). */
int vegs_bin_count(const uint32_t *tiles, int64_t n, int64_t *offsets, int64_t *kept_idx,
                   int64_t *counts, void *ws, size_t *ws_bytes, void *stream);

/* Duplicate + radix sort on (tile, depth rank) == np.lexsort((depth, tile)).
 * Outputs (n_inst): sorted_gauss (Gaussian id); optional (may be NULL): inst_pid
 * (duplicate-order index) and order (kept index, the reference's `order`);
 * tile_start/tile_end (n_tiles); optional tile_order (n_tiles): tile ids by decreasing
 * instance count, the launch order the compositing kernels accept (scheduling only).
 * n_inst must be < 2^31 (int32 instance positions); larger views return VEGS_ERR_ARG.
 * cull_record (nullable; float32 splat table of n_channels, counting-placement path only,
 * inst_pid / order must be NULL): bin each splat on its rect clipped to the tight bounding
 * box of its pass ellipse {pw >= pmin} instead of the whole rect.  The tile lists then hold
 * only instances that can blend in their tile (about 3/4 of them): images, T, contributor
 * counts and gradients are identical, tile_start / tile_end / out_last index the shorter
 * lists, and sorted_gauss needs at most n_inst entries.  NULL: the reference's lists. */
int vegs_bin_sort(const uint32_t *tiles, const uint64_t *depth_key, const int32_t *rect,
                  const int64_t *offsets, const int64_t *kept_idx, int64_t n, int64_t n_kept,
                  int64_t n_inst, int32_t width, int32_t height, int32_t tile_size,
                  uint32_t *sorted_gauss, uint32_t *inst_pid, int64_t *order,
                  int32_t *tile_start, int32_t *tile_end, int32_t *tile_order,
                  const float *cull_record, int32_t n_channels, void *ws, size_t *ws_bytes, void *stream);

/* Device-count binning (no host round trip per view; CUDA-graph capturable).
 * vegs_bin_count_dev = vegs_bin_count, then: step_state[1] = max(step_state[1], n_instances),
 * step_state[2] = max(step_state[2], n_kept); if n_instances > inst_capacity or n_kept >
 * kept_capacity the view is emptied (counts, tiles, offsets zeroed: every later stage of
 * the view runs on nothing, inside its buffers), *poison = 1 and step_state[0] = 1 (the
 * caller grows its capacities and redoes the step; the trainer's Adam skips on it).  tiles
 * is therefore read-write.  Same ws as vegs_bin_count.
 * vegs_bin_sort_dev = vegs_bin_sort's counting placement with n_kept read from counts
 * (device); launches and the workspace are sized for kept_capacity kept splats and
 * inst_capacity instances (the sorted_gauss capacity, which also bounds the placement's
 * per-block lists).  Views
 * above 12288 tiles need the radix path and host counts: VEGS_ERR_ARG.  cull_record as
 * in vegs_bin_sort. */
int vegs_bin_count_dev(uint32_t *tiles, int64_t n, int64_t *offsets, int64_t *kept_idx, int64_t *counts,
                       int64_t inst_capacity, int64_t kept_capacity, int64_t *step_state, int32_t *poison,
                       void *ws, size_t *ws_bytes, void *stream);
int vegs_bin_sort_dev(const uint64_t *depth_key, const int32_t *rect, const int64_t *offsets,
                      const int64_t *kept_idx, int64_t n, const int64_t *counts, int64_t kept_capacity,
                      int64_t inst_capacity,
                      int32_t width, int32_t height, int32_t tile_size, uint32_t *sorted_gauss,
                      int32_t *tile_start, int32_t *tile_end, int32_t *tile_order, const float *cull_record,
                      int32_t n_channels, void *ws, size_t *ws_bytes, void *stream);

/* ---- composite -------------------------------------------------------------------- */
/* Tile blend on the splat table.  out_img H x W x C, out_t H x W (storage type),
 * out_last H x W int32 (sorted-instance index, -1 = none), n_contrib H x W int32 (may be
 * NULL: the per-pixel contributor counts are then not computed).
 * tile_order (may be NULL) only permutes the order tiles are launched in. */
int vegs_composite_forward(const int32_t *tile_start, const int32_t *tile_end,
                           const uint32_t *sorted_gauss, const void *record, const int32_t *rect,
                           int32_t n_channels, int32_t store_f64, const double *bg, int32_t width,
                           int32_t height, double alpha_clamp, double trans_stop, void *out_img,
                           void *out_t, int32_t *out_last, int32_t *n_contrib,
                           const int32_t *tile_order, void *stream);

/* vegs_composite_forward for float32 splat tables with the transmittance chain in float32
 * (FFMA2 / MUFU) instead of float64.  Every decision of the reference stays exact -- the
 * 1/255 skip (float32 guard band, float64 inside it), the alpha clamp (float64 for the
 * instances that can reach it) and the 1e-4 termination (a rigorous per-pixel bound on
 * the float32 T error; a pixel whose test falls inside it is re-blended from its tile start
 * in float64 by a fix-up kernel) -- so out_last and n_contrib equal vegs_composite_forward's
 * and the reference's; out_t and out_img carry the float32 chain's rounding (~1e-6
 * relative).  defer: 1 + width * height int32 scratch; defer[0] receives the number of
 * re-blended pixels.  Replaces the same pipeline.py:197-237 / kernels.py:26-100 call. */
int vegs_composite_forward_fast(const int32_t *tile_start, const int32_t *tile_end,
                                const uint32_t *sorted_gauss, const float *record, const int32_t *rect,
                                int32_t n_channels, const double *bg, int32_t width, int32_t height,
                                double alpha_clamp, double trans_stop, float *out_img, float *out_t,
                                int32_t *out_last, int32_t *n_contrib, const int32_t *tile_order,
                                int32_t *defer, void *stream);

/* Backward tile blend.  d_img H x W x C, d_alpha H x W (storage type).  offsets: the
 * per-Gaussian instance offsets of vegs_bin_count.  Writes per-instance rows [g_mx, g_my,
 * g_ca, g_cb, g_cc, g_alpha, g_ch..., pad] (row stride rec_stride) at the instance's
 * duplicate-order index p (offsets[g] + the tile's row-major position in the splat's
 * tile rectangle; == the inst_pid output of vegs_bin_sort) and sets bit p of
 * inst_visited (ceil(n_inst / 32) words, zeroed by this call).  Rows of instances no
 * pixel blended are not written; vegs_preprocess_backward reads only visited rows. */
int vegs_composite_backward(const int32_t *tile_start, const int32_t *tile_end,
                            const uint32_t *sorted_gauss, const int64_t *offsets,
                            const void *record, const int32_t *rect, int32_t n_channels,
                            int32_t store_f64, const double *bg, int32_t width, int32_t height,
                            double alpha_clamp, const void *out_t, const int32_t *out_last,
                            const void *d_img, const void *d_alpha, void *inst_rows,
                            uint32_t *inst_visited, int64_t n_inst, const int32_t *tile_order,
                            void *stream);

/* Per-Gaussian: reduction of its instance rows (duplicate order == np.add.at order;
 * float64 rows in float64, float32 rows in float32), then projection and shading
 * backward.  grads: flat float64 class-major buffer (19 n); grads = accumulate ? grads +
 * scale * g : scale * g.  viewspace_norm / visible may be NULL.  Only rows whose
 * inst_visited bit is set are summed.  densify_stats (n x 5, may be NULL) accumulates
 * DensifyStats for the kept splats.  kept_bound: an upper bound on the kept splats (<= 0:
 * n) that sizes the float32 path's grids over its compacted kept list.  ws holds the
 * per-Gaussian sums (n x (6 + C) float64) and the kept list. */
int vegs_preprocess_backward(const double *params, int64_t n, const VegsCamera *cam,
                             const VegsTF *tf, const VegsSettings *st, int32_t n_channels,
                             int32_t store_f64, const uint32_t *tiles, const int64_t *offsets,
                             const void *inst_rows, double scale, int32_t accumulate,
                             double *grads, double *viewspace_norm, uint8_t *visible,
                             double *densify_stats, const uint32_t *inst_visited, int64_t kept_bound,
                             void *ws, size_t *ws_bytes, void *stream);

/* ---- drop-in raw kernels (reference argument lists) -------------------------------- */
int vegs_blend_forward(const int64_t *tile_start, const int64_t *tile_end, int64_t n_tiles,
                       int64_t tiles_x, int64_t tile_size, const void *inst_mean2d,
                       const void *inst_conic, const void *inst_alpha, const void *inst_pmin,
                       const int32_t *inst_rect, const void *inst_channels, int32_t n_channels,
                       int32_t store_f64, const void *bg, int64_t width, int64_t height,
                       double alpha_clamp, double trans_stop, void *out_img, void *out_t,
                       int64_t *out_last, int32_t *n_contrib, void *stream);

int vegs_blend_backward(const int64_t *tile_start, const int64_t *tile_end, int64_t n_tiles,
                        int64_t tiles_x, int64_t tile_size, const void *inst_mean2d,
                        const void *inst_conic, const void *inst_alpha, const void *inst_pmin,
                        const int32_t *inst_rect, const void *inst_channels, int32_t n_channels,
                        int32_t store_f64, const void *bg, int64_t width, int64_t height,
                        double alpha_clamp, const void *out_t, const int64_t *out_last,
                        const void *d_img, const void *d_alpha_plane, void *g_mean2d,
                        void *g_conic, void *g_alpha, void *g_channels, void *stream);

/* ---- densify / prune (train.py:237-284) ------------------------------------------- */
typedef struct {
    double grad_threshold;   /* densify_grad_threshold */
    double percent_dense;
    double scene_extent;
    double prune_threshold;  /* prune_weight_threshold on sigmoid(raw_weight) */
    double position_lr;      /* clone step */
    double log_split_factor; /* log(1.6) */
    int32_t no_weights;      /* 1: pruning off */
    int32_t pad_;
    /* NULL: prune on sigmoid(raw_weight) < prune_threshold (the reference, train.py:277-280).
     * Else n float64 per-Gaussian max TF opacities (vegs_tf_max_opacity): prune where
     * < prune_threshold (BASELINE config 4: "max TF opacity < 0.005"). */
    const double *prune_opacity;
} VegsDensify;

/* out[g] = O(sigmoid(raw_value[g])) for the opacity map of tf (init != 0), else
 * max(out[g], O(...)): called once per training TF, the per-Gaussian max TF opacity of
 * BASELINE config 4's prune rule (eval_opacity semantics, transfer.py:91-95). */
int vegs_tf_max_opacity(const double *params, int64_t n, const VegsTF *tf, int32_t init, double *out,
                        void *stream);

/* stats: n x 5 float64 [sum viewspace_norm, sum position grad (3), count] (DensifyStats).
 * flags / offsets: (n+1) x int4 = (keep, clone, split, split-any); offsets[n] holds the
 * block totals.  Output rows n_out = tot.x + tot.y + 2 tot.z. */
int vegs_densify_count(const double *params, int64_t n, const double *stats, const VegsDensify *dp,
                       int32_t *flags, int32_t *offsets, void *ws, size_t *ws_bytes, void *stream);

/* eps: 2 x tot.w x 3 float64 standard normals (round-major, as the reference draws them). */
int vegs_densify_apply(const double *params, const double *m, const double *v, int64_t n,
                       const double *stats, const VegsDensify *dp, const int32_t *flags,
                       const int32_t *offsets, const double *eps, int64_t n_out, double *out_params,
                       double *out_m, double *out_v, void *stream);

/* ---- loss / optimiser ------------------------------------------------------------- */
/* (w_l1) * mean|x - y| + lam * (1 - mean SSIM) on the rgb channels of x (H x W x
 * x_stride float32, rgb first; 3 for plain images, 11 for aux planes) against y (H x W x 3);
 * writes the rgb channels of d_x (same layout as x) and accumulates {sum |x-y|,
 * sum ssim_map} into sums[2] (float64, caller zeroes).  ws holds the SSIM gradient maps. */
int vegs_loss_l1_ssim(const float *x, const float *y, int32_t height, int32_t width, int32_t x_stride,
                      double w_l1, double lam, float *d_x, double *sums, void *ws,
                      size_t *ws_bytes, void *stream);

/* Aux-plane regularisers (loss.py:175-240) on planes (H x W x 11: rgb, depth, normal,
 * attrs) with alpha = 1 - out_t: writes channels 3..10 of d_planes and accumulates
 * {normal sum (1 - dot), mask count, smooth sum} into sums[3] (float64, caller zeroes).
 * w_normal = 0 / w_smooth = 0 switch a term off (its gradient channels are written 0). */
int vegs_loss_aux(const float *planes, const float *out_t, const float *ref_rgb, int32_t height,
                  int32_t width, double px_scale, double w_normal, double w_smooth, float *d_planes,
                  double *sums, void *ws, size_t *ws_bytes, void *stream);

/* In-place bias-corrected Adam over the flat class-major float64 buffers (19 n).
 * lr[10] per class, grad_scale multiplies g first, bias1/bias2 = 1 - beta^t.
 * nonfinite[10] (int32) receives 1 for classes that saw a non-finite gradient. */
int vegs_adam_step(double *params, const double *grads, double *m, double *v, int64_t n,
                   const double *lr, double grad_scale, double bias1, double bias2,
                   int32_t *nonfinite, void *stream);

/* The trainer's step update: g = ((grads0 + grads1) + grads2) + grads3 over the non-NULL
 * partial buffers (one per stream lane), written back into grads0, then Adam as
 * vegs_adam_step on g.  hyper (device, 12 float64): lr[10] per class, then the bias
 * corrections 1 - beta1^t, 1 - beta2^t -- read at execution time, so a captured CUDA graph
 * replays every step.  skip (device, nullable): when skip[0] != 0 nothing is updated (a
 * view of the step overflowed its buffers, see vegs_bin_count_dev).  params == NULL: only
 * the sum is formed (before a cross-rank all-reduce; m, v, hyper, nonfinite may be NULL).
 * Replaces the trainer's eager per-lane adds in front of train.py:176-195. */
int vegs_adam_step_sum(double *params, double *grads0, const double *grads1, const double *grads2,
                       const double *grads3, double *m, double *v, int64_t n, const double *hyper,
                       double grad_scale, int32_t *nonfinite, const int64_t *skip, void *stream);

/* Gradient exchange of the view-sharded step, per bucket of units
 * [unit0, unit0 + units) of the 19 n class-major layout (one unit = one parameter
 * component, n values):
 *   vegs_grad_pack: g = ((grads0 + grads1) + grads2) + grads3 over the non-NULL partials (the
 *     order vegs_adam_step_sum uses), written to payload32 (float32, 19 n, same indexing)
 *     when it is non-NULL, else back into grads0 -- the buffer the all-reduce then sums;
 *   vegs_adam_step_range: Adam (hyper / skip as vegs_adam_step_sum) over the units on the
 *     all-reduced gradient, read from payload32 (widened to float64 and stored into grads0)
 *     or from grads0.
 * Packing bucket b + 1 overlaps bucket b's all-reduce, which overlaps Adam on bucket b - 1. */
int vegs_grad_pack(double *grads0, const double *grads1, const double *grads2, const double *grads3,
                   float *payload32, int64_t n, int32_t unit0, int32_t units, void *stream);
int vegs_adam_step_range(double *params, double *grads0, const float *payload32, double *m, double *v,
                         int64_t n, int32_t unit0, int32_t units, const double *hyper, int32_t *nonfinite,
                         const int64_t *skip, void *stream);

/* Library build identity (for the loader's sanity check). */
const char *vegs_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VEGSPLAT_B200_H */
