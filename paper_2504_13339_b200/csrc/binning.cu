// Tile binning: the device form of _build_instances (pipeline.py:163-194).
//
//   np.repeat over kept splats  ->  one exclusive scan of packed (kept, tiles) counters
//   np.lexsort((depth, tile))   ->  (1) stable depth order of the kept splats (radix sort
//                                   on float32-rounded keys, exact float64 order restored
//                                   inside ties); (2) instances duplicated *in depth order*; (3) a
//                                   stable radix sort on the tile id alone (12-16 bits)
//   np.searchsorted ranges      ->  boundary scatter over the sorted tile ids
//
// Stability makes the result exactly lexsort's: equal tiles keep depth order, equal
// depths keep kept-index order (step 1 is stable on Gaussian index), and one splat never
// has two instances in a tile.  Sorting only the tile id (2 onesweep passes on 16-bit
// keys) instead of a (tile, depth-rank) key saves half the passes and a third of the
// bytes per pass.  The sort payload is the splat id itself; each instance's
// duplicate-order index p (rows of one Gaussian are contiguous in p, which the
// deterministic backward reduction relies on) is recomputed afterwards from the splat's
// tile rectangle, so no per-instance indirection array is gathered.

#include <stdlib.h>

#include <cub/cub.cuh>

#include "vegs_common.cuh"

namespace vegs {

static int bits_for(int64_t count) {  // ceil(log2(count)), >= 1
    int b = 1;
    while ((int64_t(1) << b) < count) ++b;
    return b;
}

__global__ void pack_counts_kernel(const uint32_t *tiles, int64_t n, uint64_t *packed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    const uint32_t t = i < n ? tiles[i] : 0u;
    packed[i] = t ? ((uint64_t)1 << 40) | (uint64_t)t : 0ull;  // kept count in bits 40..63
}

__global__ void unpack_counts_kernel(const uint64_t *scan, int64_t n, int64_t *offsets, int64_t *kept_idx,
                                     int64_t *counts) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    const uint64_t v = scan[i];
    offsets[i] = (int64_t)(v & ((1ull << 40) - 1));
    kept_idx[i] = (int64_t)(v >> 40);
    if (i == n) {
        counts[0] = (int64_t)(v >> 40);
        counts[1] = (int64_t)(v & ((1ull << 40) - 1));
    }
}

// Coarse 32-bit depth keys: the order-preserving bits of (float)depth.  Rounding to float32
// is monotone, so sorting by this key and then by the exact float64 key inside runs of
// equal coarse keys (depth_ties_kernel) is the float64 order; culled splats (key ~0) map
// to 0xffffffff and still sort last.  Half the radix passes of the 64-bit key.
__global__ void depth_key32_kernel(const uint64_t *key64, int64_t n, uint32_t *key32, uint32_t *ids) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = key64[i];
    uint32_t out = 0xffffffffu;
    if (k != ~0ull) {
        const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;  // inverse of depth_order_key
        const uint32_t f = __float_as_uint((float)__longlong_as_double((long long)b));
        out = (f >> 31) ? ~f : (f | 0x80000000u);
    }
    key32[i] = out;
    ids[i] = (uint32_t)i;
}

// Device-count binning: the same coarse keys, compacted to the kept splats (kept_idx is the
// kept-index scan, so index order survives and the stable sort below gives the same order
// as sorting all n), padded with max keys up to the kept capacity: the sort then runs over
// the kept capacity instead of every Gaussian (config 4: 8k kept of 200k).
__global__ void depth_key32_compact_kernel(const uint64_t *key64, const int64_t *kept_idx, int64_t n,
                                           int64_t kept_cap, const int64_t *n_kept_dev, uint32_t *key32,
                                           uint32_t *ids) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n_kept = *n_kept_dev;
    if (i >= n_kept && i < kept_cap) {  // padding (sorts last, never read)
        key32[i] = 0xffffffffu;
        ids[i] = 0u;
    }
    if (i >= n) return;
    const uint64_t k = key64[i];
    if (k == ~0ull) return;  // culled
    const int64_t pos = kept_idx[i];
    if (pos >= kept_cap) return;  // (an emptied view: never read)
    const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    const uint32_t f = __float_as_uint((float)__longlong_as_double((long long)b));
    key32[pos] = (f >> 31) ? ~f : (f | 0x80000000u);
    ids[pos] = (uint32_t)i;
}

// Runs of equal coarse keys among the kept splats are re-ordered by the exact float64 key
// (insertion sort, strict comparison: the stable sort's index order survives among equal
// float64 depths).  Runs are almost always of length 1-2.
__global__ void depth_ties_kernel(const uint32_t *key32, const uint64_t *key64, int64_t n_kept, uint32_t *ids,
                                  const int64_t *n_kept_dev = nullptr) {
    if (n_kept_dev) n_kept = *n_kept_dev;  // device-count binning: grid sized for n
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i + 1 >= n_kept) return;
    const uint32_t k = key32[i];
    if (key32[i + 1] != k || (i > 0 && key32[i - 1] == k)) return;  // not the start of a run
    int64_t j = i + 2;
    while (j < n_kept && key32[j] == k) ++j;
    for (int64_t a = i + 1; a < j; ++a) {
        const uint32_t id = ids[a];
        const uint64_t ka = key64[id];
        int64_t b = a - 1;
        while (b >= i && key64[ids[b]] > ka) {
            ids[b + 1] = ids[b];
            --b;
        }
        ids[b + 1] = id;
    }
}

// tile count of each kept splat in depth order (the scan input for the depth-order offsets)
__global__ void depth_counts_kernel(const uint32_t *sorted_ids, const uint32_t *tiles, int64_t n_kept,
                                    uint32_t *count_d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n_kept) return;
    count_d[i] = i == n_kept ? 0u : tiles[sorted_ids[i]];
}

struct SplatSpan {  // the splat's tile rectangle (pipeline.py:174-180); see dup_index
    int x0, y0, nx;
};
__device__ __forceinline__ SplatSpan splat_span(int4 r) {
    SplatSpan sp;
    sp.x0 = r.x / kTile;
    sp.y0 = r.z / kTile;
    sp.nx = (r.y - 1) / kTile - sp.x0 + 1;
    return sp;
}

// Instances in depth order: thread i loads the i-th kept splat (coalesced), then the warp
// walks its 32 splats one by one with the lanes striding over each splat's tiles
// (row-major, pipeline.py:181-187), so key and value stores are coalesced runs.
template <typename TKey>
__global__ void duplicate_kernel(const uint32_t *sorted_ids, const uint32_t *tiles, const int4 *rect,
                                 const uint32_t *offs_d, int64_t n_kept, int tiles_x, TKey *keys, uint32_t *vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint32_t g = 0, cnt = 0, base = 0;
    SplatSpan sp{0, 0, 1};
    if (i < n_kept) {
        g = sorted_ids[i];
        cnt = tiles[g];
        base = offs_d[i];
        sp = splat_span(__ldg(rect + g));
    }
    for (int k = 0; k < 32; ++k) {
        const uint32_t ck = __shfl_sync(0xffffffffu, cnt, k);
        if (ck == 0) continue;
        const uint32_t bk = __shfl_sync(0xffffffffu, base, k), gk = __shfl_sync(0xffffffffu, g, k);
        const int x0 = __shfl_sync(0xffffffffu, sp.x0, k), y0 = __shfl_sync(0xffffffffu, sp.y0, k);
        const int nx = __shfl_sync(0xffffffffu, sp.nx, k);
        for (uint32_t j = lane; j < ck; j += 32) {
            const int dy = (int)(j / (uint32_t)nx), dx = (int)j - dy * nx;
            keys[bk + j] = (TKey)((y0 + dy) * tiles_x + (x0 + dx));
            vals[bk + j] = gk;
        }
    }
}

// For each sorted instance: the searchsorted tile ranges (empty tiles get start == end ==
// insertion point) and, only when asked for (reference-shaped API), the kept index
// (`order`) and the duplicate-order index p = offsets[g] + (row-major index of the tile
// inside the splat's tile rectangle).  The compositing kernels recompute p themselves, so
// the training path reads 2 bytes per instance here.
template <typename TKey>
__global__ void finalize_kernel(const TKey *keys, const uint32_t *sorted_gauss, const int4 *rect,
                                const int64_t *offsets, const int64_t *kept_idx, int64_t n_inst, int n_tiles,
                                int tiles_x, uint32_t *inst_pid, int64_t *order, int32_t *tile_start,
                                int32_t *tile_end) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_inst) return;
    const int tile = (int)keys[s];
    if (inst_pid || order) {
        const uint32_t gid = sorted_gauss[s];
        if (inst_pid) {
            const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
            inst_pid[s] = (uint32_t)dup_index(__ldg(offsets + gid), __ldg(rect + gid), tx, ty);
        }
        if (order) order[s] = kept_idx[gid];
    }
    const int prev = s > 0 ? (int)keys[s - 1] : -1;
    if (tile != prev) {
        for (int t = prev + 1; t <= tile; ++t) tile_start[t] = (int32_t)s;
        for (int t = prev < 0 ? 0 : prev; t < tile; ++t) tile_end[t] = (int32_t)s;
    }
    if (s == n_inst - 1) {
        for (int t = tile; t < n_tiles; ++t) tile_end[t] = (int32_t)n_inst;
        for (int t = tile + 1; t < n_tiles; ++t) tile_start[t] = (int32_t)n_inst;
    }
}

// Scheduling key of each tile: instance count (capped at 16 bits), complemented so an
// ascending sort puts the heaviest tiles first (the compositing grids then start the
// longest tiles earliest).
__global__ void tile_weight_kernel(const int32_t *tile_start, const int32_t *tile_end, int n_tiles, uint32_t *key,
                                   int32_t *val) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    const uint32_t c = (uint32_t)(tile_end[t] - tile_start[t]);
    key[t] = 0xffffu - (c < 0xffffu ? c : 0xffffu);
    val[t] = t;
}

// Culled binning rectangles (float32 tables, training / render paths): the reference's rect
// clipped to the tight bounding box of the instance's pass ellipse.  A pixel blends only if
// pw >= pmin, i.e. q = -2 pw = a dx^2 + 2 b dx dy + c dy^2 <= qmax = -2 pmin; on that ellipse
// |dx| <= sqrt(qmax c / det) and |dy| <= sqrt(qmax a / det), det = a c - b^2.  The float64
// decisions of the compositing kernels use exactly these float32 record values, so a box
// inflated by 5e-4 relative + 1e-3 px over the float32 evaluation (det > 1e-2 a c keeps its
// relative error below 4e-5) holds every passing pixel: the tile lists lose only instances
// that cannot blend in the tile (23% at c2 / c3), images, T, contributor counts and
// gradients are unchanged.  Conics not clearly positive definite keep the full rect.
__global__ void bin_rect_kernel(const float *record, int rs, const int4 *rect, int64_t n, int4 *brect) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int4 r = rect[i];
    if (r.y > r.x && r.w > r.z) {
        const float *g = record + (int64_t)rs * i;
        const float mx = g[0], my = g[1], a = g[2], b = g[3], c = g[4], pm = g[6];
        const float det = a * c - b * b;
        if (a > 0.f && c > 0.f && det > 1e-2f * (a * c) && pm <= 0.f && isfinite(mx) && isfinite(my)) {
            const float qmax = -2.f * pm;
            const float rx = sqrtf(qmax * c / det) * 1.0005f + 1e-3f, ry = sqrtf(qmax * a / det) * 1.0005f + 1e-3f;
            // first / last pixel whose centre x + 0.5 lies within mx -/+ rx, clamped to the rect
            // in float before the int conversion
            const float xl = fmaxf(ceilf(mx - rx - 0.5f), (float)r.x), xh = fminf(floorf(mx + rx - 0.5f), (float)(r.y - 1));
            const float yl = fmaxf(ceilf(my - ry - 0.5f), (float)r.z), yh = fminf(floorf(my + ry - 0.5f), (float)(r.w - 1));
            if (!(xl <= xh && yl <= yh)) r = make_int4(0, 0, 0, 0);
            else r = make_int4((int)xl, (int)xh + 1, (int)yl, (int)yh + 1);
        }
    }
    brect[i] = r;
}

// ---- small depth sorts in one CTA ----------------------------------------------------
// Stable LSD radix sort of up to kSmallSort (key, id) pairs by 32-bit key in a single CTA
// (4 passes of 8 bits, keys and ids in SMEM between passes): config-4 views keep ~11k
// splats, where the device-wide sort's 6 launches are pure latency.  Ranking per warp with
// match.any peer groups (items in index order: warp-major, item, lane), digit offsets by an
// exclusive sum over the 256 digits; stable, so the same order as the device-wide sort.
constexpr int kSmallSortT = 1024, kSmallSortItems = 16, kSmallSort = kSmallSortT * kSmallSortItems;

__global__ void __launch_bounds__(kSmallSortT) small_sort_kernel(const uint32_t *keys, const uint32_t *vals, int n,
                                                                 uint32_t *keys_out, uint32_t *vals_out) {
    constexpr int NW = kSmallSortT / 32, IT = kSmallSortItems;
    __shared__ uint32_t s_wc[NW][256];
    __shared__ uint32_t s_dstart[256];
    __shared__ int s_same;
    extern __shared__ uint32_t s_kv[];  // keys [0, n), ids [kSmallSort, kSmallSort + n)
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int items = (n + kSmallSortT - 1) / kSmallSortT;  // per thread (<= IT)
    if (t == 0) s_same = 0;
    uint32_t key[IT], val[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const int idx = w * 32 * items + i * 32 + lane;
        const bool ok = i < items && idx < n;
        key[i] = ok ? keys[idx] : 0u;
        val[i] = ok ? vals[idx] : 0u;
    }
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 8 * pass;
        for (int i = t; i < NW * 256; i += kSmallSortT) (&s_wc[0][0])[i] = 0;
        __syncthreads();
        int dig[IT];
        uint32_t rank[IT];
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const int idx = w * 32 * items + i * 32 + lane;
            dig[i] = i < items && idx < n ? (int)((key[i] >> shift) & 255u) : 256;
            if (i >= items) continue;
            const unsigned peers = __match_any_sync(0xffffffffu, dig[i]);
            const uint32_t before = dig[i] < 256 ? s_wc[w][dig[i]] : 0u;
            rank[i] = before + (uint32_t)__popc(peers & ((1u << lane) - 1u));
            __syncwarp();
            if (dig[i] < 256 && lane == __ffs(peers) - 1) s_wc[w][dig[i]] = before + (uint32_t)__popc(peers);
            __syncwarp();
        }
        __syncthreads();
        if (t < 256) {  // digit t: the warps' offsets and the digit's total
            uint32_t cnt = 0;
            for (int k = 0; k < NW; ++k) {
                const uint32_t c = s_wc[k][t];
                s_wc[k][t] = cnt;
                cnt += c;
            }
            s_dstart[t] = cnt;
            if (cnt == (uint32_t)n) s_same = 1;  // every key has this digit: the pass is the identity
        }
        __syncthreads();
        if (s_same && pass < 3) {  // (stable: nothing moves) -- the next digit, same registers
            __syncthreads();
            if (t == 0) s_same = 0;
            continue;
        }
        if (t < 32) {  // exclusive sum of the 256 digit totals (8 per lane)
            uint32_t v[8], sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                v[q] = s_dstart[lane * 8 + q];
                sum += v[q];
            }
            uint32_t x = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            uint32_t run = x - sum;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                s_dstart[lane * 8 + q] = run;
                run += v[q];
            }
        }
        __syncthreads();
        const bool last = pass == 3;
#pragma unroll
        for (int i = 0; i < IT; ++i)
            if (i < items && dig[i] < 256) {
                const uint32_t pos = s_dstart[dig[i]] + s_wc[w][dig[i]] + rank[i];
                if (last) {
                    keys_out[pos] = key[i];
                    vals_out[pos] = val[i];
                } else {
                    s_kv[pos] = key[i];
                    s_kv[kSmallSort + pos] = val[i];
                }
            }
        if (last) break;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const int idx = w * 32 * items + i * 32 + lane;
            if (i < items && idx < n) {
                key[i] = s_kv[idx];
                val[i] = s_kv[kSmallSort + idx];
            }
        }
    }
}

// ---- counting placement (no instance-level sort) ----------------------------------
// The kept splats in depth order are cut into chunks of C.  (1) per chunk, per-tile
// instance counts from a 2D difference array of the splats' tile rectangles; (2) those
// counts, scanned tile-major over (tile, chunk), give every chunk its first output slot in
// every tile; (3) one warp per chunk walks its splats in depth order and appends each
// splat's id to each of its tiles.  Slots within a tile therefore follow (chunk, depth
// rank) = depth rank order: exactly np.lexsort((depth, tile)), as the radix path.

__global__ void chunk_count_kernel(const uint32_t *ids, const int4 *rect, int64_t n_kept, int C, int tiles_x,
                                   int tiles_y, uint32_t *counts, const int64_t *n_kept_dev = nullptr,
                                   int shift = 4) {  // cells of 2^shift pixels (tiles, or 4x4-tile blocks)
    if (n_kept_dev) n_kept = *n_kept_dev;  // device-count binning: chunks past the kept splats count zero
    extern __shared__ int diff[];  // (tiles_y + 1) x (tiles_x + 1)
    const int c = blockIdx.x, W1 = tiles_x + 1, n_diff = (tiles_y + 1) * W1, n_tiles = tiles_x * tiles_y;
    for (int i = threadIdx.x; i < n_diff; i += blockDim.x) diff[i] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)c * C, hi = lo + C < n_kept ? lo + C : n_kept;
    for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) {
        const int4 q = __ldg(rect + ids[r]);
        if (q.y <= q.x || q.w <= q.z) continue;  // a culled-empty binning rect
        const int x0 = q.x >> shift, x1 = ((q.y - 1) >> shift) + 1, y0 = q.z >> shift, y1 = ((q.w - 1) >> shift) + 1;
        atomicAdd(&diff[y0 * W1 + x0], 1);
        atomicAdd(&diff[y0 * W1 + x1], -1);
        atomicAdd(&diff[y1 * W1 + x0], -1);
        atomicAdd(&diff[y1 * W1 + x1], 1);
    }
    __syncthreads();
    for (int y = threadIdx.x; y < tiles_y; y += blockDim.x) {  // prefix along rows
        int run = 0;
        for (int x = 0; x < tiles_x; ++x) diff[y * W1 + x] = (run += diff[y * W1 + x]);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < tiles_x; x += blockDim.x) {  // prefix along columns
        int run = 0;
        for (int y = 0; y < tiles_y; ++y) counts[(size_t)c * n_tiles + y * tiles_x + x] = (uint32_t)(run += diff[y * W1 + x]);
    }
}

// per (group of G chunks, tile): the group's instance count
__global__ void chunk_group_sum_kernel(const uint32_t *counts, int n_chunks, int n_tiles, int G, uint32_t *gsum) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int n_groups = (n_chunks + G - 1) / G;
    if (i >= (int64_t)n_groups * n_tiles) return;
    const int grp = (int)(i / n_tiles), t = (int)(i - (int64_t)grp * n_tiles);
    const int c0 = grp * G, c1 = (grp + 1) * G < n_chunks ? (grp + 1) * G : n_chunks;
    uint32_t sum = 0;
#pragma unroll 8
    for (int c = c0; c < c1; ++c) sum += __ldg(counts + (size_t)c * n_tiles + t);
    gsum[i] = sum;
}

// per tile: exclusive scan of the group counts (in place) and the tile total
__global__ void tile_group_scan_kernel(uint32_t *gsum, int n_groups, int n_tiles, uint32_t *total) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    uint32_t run = 0;
    for (int g = 0; g < n_groups; ++g) {
        const uint32_t v = gsum[(size_t)g * n_tiles + t];
        gsum[(size_t)g * n_tiles + t] = run;
        run += v;
    }
    total[t] = run;
}

// per (group, tile): counts -> first output slot of every chunk (in place); tile ranges
__global__ void chunk_offsets_kernel(uint32_t *counts, const uint32_t *gbase, const int32_t *tile_start,
                                     const uint32_t *total, int n_chunks, int n_tiles, int G, int32_t *tile_end) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int n_groups = (n_chunks + G - 1) / G;
    if (i >= (int64_t)n_groups * n_tiles) return;
    const int grp = (int)(i / n_tiles), t = (int)(i - (int64_t)grp * n_tiles);
    if (grp == 0) tile_end[t] = tile_start[t] + (int32_t)total[t];
    uint32_t run = (uint32_t)tile_start[t] + gbase[i];
    const int c0 = grp * G, c1 = (grp + 1) * G < n_chunks ? (grp + 1) * G : n_chunks;
    for (int cb = c0; cb < c1; cb += 16) {  // 16 loads in flight, then 16 stores
        uint32_t v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cb + q < c1 ? counts[(size_t)(cb + q) * n_tiles + t] : 0u;
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (cb + q < c1) {
                counts[(size_t)(cb + q) * n_tiles + t] = run;
                run += v[q];
            }
    }
}

// One CTA per chunk, one warp per horizontal band of tile rows (kBands bands): each warp
// walks the chunk's splats in depth order and appends, for the part of each splat's tile
// rectangle inside its band, the splat id to each tile (distinct tiles inside a splat: no
// conflicts); per-tile cursors in SMEM.  The bands multiply the warps in flight: 8 for up
// to 4096 tiles (1024^2: bin_sort 0.419 -> 0.395 ms against 4), 4 above (1080p: the 8-band
// CTA's 32 KB of cursors per 256 threads cost 2% of the config-3 sweep).
template <int kBands>
__global__ void __launch_bounds__(32 * kBands) place_kernel(const uint32_t *ids, const int4 *rect, int64_t n_kept,
                                                            int C, int tiles_x, int tiles_y, const uint32_t *first,
                                                            uint32_t *sorted_gauss, const int64_t *n_kept_dev = nullptr,
                                                            int shift = 4) {
    if (n_kept_dev) n_kept = *n_kept_dev;
    extern __shared__ uint32_t cursor[];
    const int n_tiles = tiles_x * tiles_y;
    const int c = blockIdx.x, lane = threadIdx.x & 31, band = threadIdx.x >> 5;
    // the chunk's first slots straight into SMEM (LDGSTS, all in flight; 16-byte pieces when
    // the rows are aligned): a load-then-store loop left every cursor a dependent round trip
    const int64_t lo = (int64_t)c * C, hi = lo + C < n_kept ? lo + C : n_kept;
    if (lo >= hi) return;  // (device counts: chunks past the kept splats)
    const uint32_t *src = first + (size_t)c * n_tiles;
    const uint32_t cur0 = (uint32_t)__cvta_generic_to_shared(cursor);
    if ((n_tiles & 3) == 0) {
        for (int q = threadIdx.x; q < (n_tiles >> 2); q += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(cur0 + 16u * q), "l"(src + 4 * q));
    } else {
        for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(cur0 + 4u * t), "l"(src + t));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    const int band_lo = band * tiles_y / kBands, band_hi = (band + 1) * tiles_y / kBands - 1;  // tile rows
    // lane k holds splat r0 + k of the current group of 32; the next group's ids and rects
    // are fetched while this one is placed
    auto fetch = [&](int64_t r0, uint32_t &g, int4 &q) {
        g = 0;
        q = make_int4(0, 1, 0, 1);
        if (r0 + lane < hi) {
            g = ids[r0 + lane];
            q = __ldg(rect + g);
        }
    };
    uint32_t g_n;
    int4 q_n;
    fetch(lo, g_n, q_n);  // overlaps the cursor copy
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    for (int64_t r0 = lo; r0 < hi; r0 += 32) {
        const uint32_t g = g_n;
        const int4 q = q_n;
        if (r0 + 32 < hi) fetch(r0 + 32, g_n, q_n);
        const int x0 = q.x >> shift, nx = ((q.y - 1) >> shift) - x0 + 1;
        const int ys = max(q.z >> shift, band_lo), ye = min((q.w - 1) >> shift, band_hi);
        const int cnt = r0 + lane < hi && ys <= ye && q.x < q.y ? nx * (ye - ys + 1) : 0;
        const float inx = 1.0f / (float)nx;
        unsigned todo = __ballot_sync(0xffffffffu, cnt > 0);  // splats of the group touching this band
        while (todo) {
            const int k = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t gk = __shfl_sync(0xffffffffu, g, k);
            const int x0k = __shfl_sync(0xffffffffu, x0, k), ysk = __shfl_sync(0xffffffffu, ys, k);
            const int nxk = __shfl_sync(0xffffffffu, nx, k), ck = __shfl_sync(0xffffffffu, cnt, k);
            const float ik = __shfl_sync(0xffffffffu, inx, k);
            for (int j = lane; j < ck; j += 32) {
                // j / nxk via the float reciprocal (exact for j < 2^20: the quotient is
                // corrected by one step)
                int dy = (int)((float)j * ik);
                dy += (j - dy * nxk >= nxk) - (j - dy * nxk < 0);
                const int dx = j - dy * nxk;
                const int t = (ysk + dy) * tiles_x + (x0k + dx);
                const uint32_t pos = cursor[t];
                cursor[t] = pos + 1;
                sorted_gauss[pos] = gk;
            }
            __syncwarp();
        }
    }
}

// ---- two-level placement ---------------------------------------------------------------
// Level 1 runs the counting placement above on a grid of 4x4-tile blocks: per block, the ids
// of the splats whose binning rect touches it, in depth order (about 1.3 entries per kept
// splat at c2 / c3 against ~25 tile instances).  Level 2 runs one CTA per block over that
// list in batches of 256 splats: each thread takes one splat and the 16-bit mask of the
// block's tiles its rect covers; per tile, a ballot ranks the warp's splats in list (= depth)
// order and the warps' counts are scanned in SMEM, so every tile's entries of a batch are
// written as one contiguous run -- one coalesced store per tile and warp instead of one
// scattered 4-byte store per instance (the single-level placement was bound by those L2
// write requests: 0.44 ms of a 1080p frame).  Result identical to the single level:
// per tile, the splats in depth order.
constexpr int kBlk = 4;  // tiles per block side
#ifndef VEGS_L1_BANDS
#define VEGS_L1_BANDS 1  // level 1: one warp per chunk (2: 908, 4: 887 Mpx/s config-3 sweep against 913)
#endif

__device__ __forceinline__ uint32_t block_tile_mask(int4 q, int bx0, int by0, int tiles_x, int tiles_y) {
    if (q.y <= q.x || q.w <= q.z) return 0u;
    const int x0 = max(q.x >> 4, bx0), x1 = min((q.y - 1) >> 4, min(bx0 + kBlk - 1, tiles_x - 1));
    const int y0 = max(q.z >> 4, by0), y1 = min((q.w - 1) >> 4, min(by0 + kBlk - 1, tiles_y - 1));
    if (x0 > x1 || y0 > y1) return 0u;
    const uint32_t row = ((1u << (x1 - x0 + 1)) - 1u) << (x0 - bx0);
    uint32_t m = 0;
#pragma unroll
    for (int y = 0; y < kBlk; ++y)
        if (by0 + y >= y0 && by0 + y <= y1) m |= row << (kBlk * y);
    return m;
}

// per tile: its instance count, from 2D difference arrays of the kept splats' binning rects:
// each CTA accumulates its share of the splats in a private SMEM array (4 SMEM atomics per
// splat), then adds that array into the global one (every address once per CTA: no hot spots)
__global__ void __launch_bounds__(256) tile_diff_kernel(const uint32_t *ids, const int4 *rect, int64_t n_kept,
                                                        int tiles_x, int tiles_y, int *diff,
                                                        const int64_t *n_kept_dev) {
    extern __shared__ int s_diff[];
    if (n_kept_dev) n_kept = *n_kept_dev;
    const int W1 = tiles_x + 1, n_diff = W1 * (tiles_y + 1);
    for (int i = threadIdx.x; i < n_diff; i += blockDim.x) s_diff[i] = 0;
    __syncthreads();
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_kept; r += (int64_t)gridDim.x * blockDim.x) {
        const int4 q = __ldg(rect + ids[r]);
        if (q.y <= q.x || q.w <= q.z) continue;
        const int x0 = q.x >> 4, x1 = ((q.y - 1) >> 4) + 1, y0 = q.z >> 4, y1 = ((q.w - 1) >> 4) + 1;
        atomicAdd(&s_diff[y0 * W1 + x0], 1);
        atomicAdd(&s_diff[y0 * W1 + x1], -1);
        atomicAdd(&s_diff[y1 * W1 + x0], -1);
        atomicAdd(&s_diff[y1 * W1 + x1], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_diff; i += blockDim.x)
        if (s_diff[i]) atomicAdd(diff + i, s_diff[i]);
}

__global__ void __launch_bounds__(1024) tile_total_kernel(const int *diff, int tiles_x, int tiles_y,
                                                          uint32_t *total) {
    extern __shared__ int s_d[];  // the difference array, prefix-summed in SMEM
    const int W1 = tiles_x + 1, n_diff = W1 * (tiles_y + 1);
    for (int i = threadIdx.x; i < n_diff; i += blockDim.x) s_d[i] = diff[i];
    __syncthreads();
    for (int y = threadIdx.x; y < tiles_y; y += blockDim.x) {  // prefix along rows
        int run = 0;
        for (int x = 0; x < tiles_x; ++x) s_d[y * W1 + x] = (run += s_d[y * W1 + x]);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < tiles_x; x += blockDim.x) {  // prefix along columns
        int run = 0;
        for (int y = 0; y < tiles_y; ++y) total[y * tiles_x + x] = (uint32_t)(run += s_d[y * W1 + x]);
    }
}

// level 2: the block's tiles filled run by run (the next batch's ids and rects are fetched
// while one is placed); tile_end from the final cursors
#ifndef VEGS_BP_T
#define VEGS_BP_T 512  // 16 warps per block CTA, one 512-splat sub-batch per batch (256 x 2: -2.6% sweep; 1024: -1%)
#endif
#ifndef VEGS_BP_K
#define VEGS_BP_K 1
#endif
__global__ void __launch_bounds__(VEGS_BP_T) block_place_kernel(const uint32_t *coarse, const int32_t *blk_start,
                                                          const int32_t *blk_end, const int4 *rect, int tiles_x,
                                                          int tiles_y, int bx, const int32_t *tile_start,
                                                          int32_t *tile_end, uint32_t *sorted_gauss) {
    constexpr int NB = kBlk * kBlk, NT = VEGS_BP_T, NW = NT / 32, K = VEGS_BP_K;  // K splats per thread per batch
    __shared__ uint32_t s_cur[NB];      // next slot of each tile
    __shared__ uint32_t s_wc[NW][NB];   // per-warp counts of the batch, then the warps' first slots
    const int blk = blockIdx.x, bx0 = (blk % bx) * kBlk, by0 = (blk / bx) * kBlk;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    if (t < NB) {
        const int tx = bx0 + t % kBlk, ty = by0 + t / kBlk;
        s_cur[t] = tx < tiles_x && ty < tiles_y ? (uint32_t)tile_start[ty * tiles_x + tx] : 0u;
    }
    const int beg = blk_start[blk], end = blk_end[blk];
    // batch layout: splat beg + i0 + k * NT + t for k < K (each warp's splats stay in list order
    // per k; the K sub-batches are ranked one after the other)
    uint32_t g_n[K];
    int4 q_n[K];
    auto fetch = [&](int i0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = i0 + k * NT + t;
            g_n[k] = i < end ? coarse[i] : 0u;
            q_n[k] = i < end ? __ldg(rect + g_n[k]) : make_int4(0, 0, 0, 0);
        }
    };
    fetch(beg);
    __syncthreads();
    for (int i0 = beg; i0 < end; i0 += K * NT) {  // block-uniform trip count
        uint32_t g[K], m[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            g[k] = g_n[k];
            m[k] = block_tile_mask(q_n[k], bx0, by0, tiles_x, tiles_y);
        }
        if (i0 + K * NT < end) fetch(i0 + K * NT);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            uint32_t bal[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                bal[b] = __ballot_sync(0xffffffffu, (m[k] >> b) & 1u);
                if (lane == 0) s_wc[w][b] = __popc(bal[b]);
            }
            __syncthreads();
            if (t < NB) {  // tile t: the warps' first slots in list order, then the cursor moves on
                uint32_t run = s_cur[t];
#pragma unroll
                for (int j = 0; j < NW; ++j) {
                    const uint32_t c = s_wc[j][t];
                    s_wc[j][t] = run;
                    run += c;
                }
                s_cur[t] = run;
            }
            __syncthreads();
#pragma unroll
            for (int b = 0; b < NB; ++b)
                if ((m[k] >> b) & 1u) sorted_gauss[s_wc[w][b] + __popc(bal[b] & lt)] = g[k];
            __syncthreads();  // s_wc is rewritten by the next sub-batch
        }
    }
    if (t < NB) {
        const int tx = bx0 + t % kBlk, ty = by0 + t / kBlk;
        if (tx < tiles_x && ty < tiles_y) tile_end[ty * tiles_x + tx] = (int32_t)s_cur[t];
    }
}

// API path only: the tile of each sorted instance (from the ranges), its kept index and
// duplicate-order index
__global__ void placed_extras_kernel(const uint32_t *sorted_gauss, const int4 *rect, const int64_t *offsets,
                                     const int64_t *kept_idx, const int32_t *tile_end, int64_t n_inst, int n_tiles,
                                     int tiles_x, uint32_t *inst_pid, int64_t *order) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_inst) return;
    int lo = 0, hi = n_tiles - 1;  // first tile whose end exceeds s
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (tile_end[mid] > s) hi = mid;
        else lo = mid + 1;
    }
    const uint32_t gid = sorted_gauss[s];
    if (inst_pid) {
        const int ty = lo / tiles_x, tx = lo - ty * tiles_x;
        inst_pid[s] = (uint32_t)dup_index(__ldg(offsets + gid), __ldg(rect + gid), tx, ty);
    }
    if (order) order[s] = kept_idx[gid];
}

// Device-count binning (graph capture: no host round trip for the counts).  A view whose
// instance or kept-splat count exceeds the caller's capacities is turned into an empty
// view: its counts, tile counts and offsets are zeroed, so every later stage of the view
// (sort, compositing, backward) runs on nothing and stays inside its buffers; step_state
// records the overflow ([0] = 1) and the largest counts seen ([1] instances, [2] kept
// splats) for the caller to grow its capacities and redo.
__global__ void capacity_check_kernel(int64_t *counts, int64_t capacity, int64_t kept_capacity, int64_t *step_state,
                                      int32_t *poison) {
    const int64_t n_kept = counts[0], n_inst = counts[1];
    atomicMax(reinterpret_cast<unsigned long long *>(step_state + 1), (unsigned long long)n_inst);
    atomicMax(reinterpret_cast<unsigned long long *>(step_state + 2), (unsigned long long)n_kept);
    const bool over = n_inst > capacity || n_kept > kept_capacity;
    *poison = over ? 1 : 0;
    if (over) {
        atomicExch(reinterpret_cast<unsigned long long *>(step_state), 1ull);
        counts[0] = 0;
        counts[1] = 0;
    }
}

__global__ void capacity_empty_kernel(const int32_t *poison, uint32_t *tiles, int64_t n, int64_t *offsets,
                                      int64_t *kept_idx) {
    if (!*poison) return;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i < n) tiles[i] = 0u;
    offsets[i] = 0;
    kept_idx[i] = 0;
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace vegs

using namespace vegs;

extern "C" int vegs_bin_count(const uint32_t *tiles, int64_t n, int64_t *offsets, int64_t *kept_idx,
                              int64_t *counts, void *ws, size_t *ws_bytes, void *stream) {
    if (!ws_bytes) return VEGS_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    size_t scan_bytes = 0;
    uint64_t *dummy = nullptr;
    VEGS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, dummy, dummy, n + 1, s));
    const size_t packed_bytes = align_up(sizeof(uint64_t) * (n + 1));
    const size_t need = 2 * packed_bytes + align_up(scan_bytes);
    if (!ws) {
        *ws_bytes = need;
        return VEGS_OK;
    }
    if (*ws_bytes < need) return VEGS_ERR_CAPACITY;
    if ((n > 0 && !tiles) || !offsets || !kept_idx || !counts) return VEGS_ERR_ARG;
    char *w = (char *)ws;
    uint64_t *packed = (uint64_t *)w;
    uint64_t *scanned = (uint64_t *)(w + packed_bytes);
    void *tmp = w + 2 * packed_bytes;
    const int blocks = (int)((n + 1 + 255) / 256);
    pack_counts_kernel<<<blocks, 256, 0, s>>>(tiles, n, packed);
    VEGS_CHECK_LAUNCH();
    VEGS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, packed, scanned, n + 1, s));
    unpack_counts_kernel<<<blocks, 256, 0, s>>>(scanned, n, offsets, kept_idx, counts);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

template <typename TKey>
static int bin_sort_impl(const uint32_t *tiles, const uint64_t *depth_key, const int32_t *rect,
                         const int64_t *offsets, const int64_t *kept_idx, int64_t n, int64_t n_kept,
                         int64_t n_inst, int tiles_x, int n_tiles, uint32_t *sorted_gauss, uint32_t *inst_pid,
                         int64_t *order, int32_t *tile_start, int32_t *tile_end, int32_t *tile_order, void *ws,
                         size_t *ws_bytes, cudaStream_t s) {
    const int tile_bits = bits_for(n_tiles);
    size_t t_depth = 0, t_scan = 0, t_inst = 0, t_tiles = 0;
    {
        cub::DoubleBuffer<uint32_t> dk(nullptr, nullptr);
        cub::DoubleBuffer<uint32_t> dv(nullptr, nullptr);
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_depth, dk, dv, (int64_t)n, 0, 32, s));
        uint32_t *dummy = nullptr;
        VEGS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, dummy, dummy, (int64_t)n_kept + 1, s));
        cub::DoubleBuffer<TKey> ik(nullptr, nullptr);
        cub::DoubleBuffer<uint32_t> iv(nullptr, nullptr);
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_inst, ik, iv, (int64_t)n_inst, 0, tile_bits, s));
        uint32_t *tk = nullptr;
        int32_t *tv = nullptr;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_tiles, tk, tk, tv, tv, n_tiles, 0, 16, s));
    }
    const size_t b_dk = align_up(sizeof(uint32_t) * n), b_id = align_up(sizeof(uint32_t) * (n + 1));
    const size_t b_k = align_up(sizeof(TKey) * n_inst), b_v = align_up(sizeof(uint32_t) * n_inst);
    size_t t_max = t_depth > t_inst ? t_depth : t_inst;
    t_max = t_max > t_scan ? t_max : t_scan;
    t_max = t_max > t_tiles ? t_max : t_tiles;
    const size_t b_tmp = align_up(t_max);
    const size_t b_t = align_up(sizeof(uint32_t) * n_tiles);
    const size_t need = 2 * b_dk + 4 * b_id + 2 * b_k + b_v + 3 * b_t + b_tmp;
    if (!ws) {
        *ws_bytes = need;
        return VEGS_OK;
    }
    if (*ws_bytes < need) return VEGS_ERR_CAPACITY;
    char *w = (char *)ws;
    uint32_t *dk0 = (uint32_t *)w; w += b_dk;
    uint32_t *dk1 = (uint32_t *)w; w += b_dk;
    uint32_t *id0 = (uint32_t *)w; w += b_id;
    uint32_t *id1 = (uint32_t *)w; w += b_id;
    uint32_t *count_d = (uint32_t *)w; w += b_id;
    uint32_t *offs_d = (uint32_t *)w; w += b_id;
    TKey *k0 = (TKey *)w; w += b_k;
    TKey *k1 = (TKey *)w; w += b_k;
    uint32_t *v1 = (uint32_t *)w; w += b_v;
    uint32_t *tkey0 = (uint32_t *)w; w += b_t;
    uint32_t *tkey1 = (uint32_t *)w; w += b_t;
    int32_t *tval = (int32_t *)w; w += b_t;
    void *tmp = w;

    if (n_inst == 0) {
        VEGS_CUDA(cudaMemsetAsync(tile_start, 0, sizeof(int32_t) * n_tiles, s));
        VEGS_CUDA(cudaMemsetAsync(tile_end, 0, sizeof(int32_t) * n_tiles, s));
        if (tile_order) {
            tile_weight_kernel<<<(n_tiles + 255) / 256, 256, 0, s>>>(tile_start, tile_end, n_tiles, tkey0, tile_order);
            VEGS_CHECK_LAUNCH();
        }
        return VEGS_OK;
    }
    // 1. stable depth order of the kept splats (culled ones carry the max key, sort last):
    //    radix sort on the coarse 32-bit key, then exact float64 order inside ties
    depth_key32_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(depth_key, n, dk0, id0);
    VEGS_CHECK_LAUNCH();
    cub::DoubleBuffer<uint32_t> dk(dk0, dk1);
    cub::DoubleBuffer<uint32_t> dv(id0, id1);
    {
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int64_t)n, 0, 32, s));
        depth_ties_kernel<<<(int)((n_kept + 255) / 256), 256, 0, s>>>(dk.Current(), depth_key, n_kept, dv.Current());
        VEGS_CHECK_LAUNCH();
        depth_counts_kernel<<<(int)((n_kept + 1 + 255) / 256), 256, 0, s>>>(dv.Current(), tiles, n_kept, count_d);
        VEGS_CHECK_LAUNCH();
    }
    // 2. instance offsets in depth order, then duplication (tile keys and splat ids in depth order)
    {
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, count_d, offs_d, (int64_t)n_kept + 1, s));
    }
    duplicate_kernel<TKey><<<(int)((n_kept + 255) / 256), 256, 0, s>>>(dv.Current(), tiles, (const int4 *)rect,
                                                                       offs_d, n_kept, tiles_x, k0, sorted_gauss);
    VEGS_CHECK_LAUNCH();
    // 3. stable sort on the tile id only; the values are the splat ids themselves
    cub::DoubleBuffer<TKey> ik(k0, k1);
    cub::DoubleBuffer<uint32_t> iv(sorted_gauss, v1);
    {
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, ik, iv, (int64_t)n_inst, 0, tile_bits, s));
    }
    if (iv.Current() != sorted_gauss)
        VEGS_CUDA(cudaMemcpyAsync(sorted_gauss, iv.Current(), sizeof(uint32_t) * n_inst, cudaMemcpyDeviceToDevice, s));
    // 4. duplicate-order indices, kept-index order, tile ranges
    finalize_kernel<TKey><<<(int)((n_inst + 255) / 256), 256, 0, s>>>(ik.Current(), sorted_gauss, (const int4 *)rect,
                                                                      offsets, kept_idx, n_inst, n_tiles, tiles_x,
                                                                      inst_pid, order, tile_start, tile_end);
    VEGS_CHECK_LAUNCH();
    // 5. optional launch order for the compositing kernels: heaviest tiles first
    if (tile_order) {
        tile_weight_kernel<<<(n_tiles + 255) / 256, 256, 0, s>>>(tile_start, tile_end, n_tiles, tkey0, tval);
        VEGS_CHECK_LAUNCH();
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, tkey0, tkey1, tval, tile_order, n_tiles, 0, 16, s));
    }
    return VEGS_OK;
}

// Counting-placement binning for up to kMaxPlaceTiles tiles (per-tile cursors and the
// difference array live in SMEM); larger images, or VEGS_BIN_RADIX set in the environment
// (tests), take the radix path above.
constexpr int kMaxPlaceTiles = 12288;

static int bin_place_impl(const uint64_t *depth_key, const int32_t *rect, const int64_t *offsets,
                          const int64_t *kept_idx, int64_t n, int64_t n_kept, int64_t n_inst, int tiles_x,
                          int tiles_y, uint32_t *sorted_gauss, uint32_t *inst_pid, int64_t *order,
                          int32_t *tile_start, int32_t *tile_end, int32_t *tile_order, void *ws, size_t *ws_bytes,
                          cudaStream_t s, const int64_t *counts_dev = nullptr, const float *cull_record = nullptr,
                          int rs = 0, int64_t inst_capacity = 0) {
    // counts_dev (device-count binning): n_kept / n_inst live on the device; every launch is
    // sized for n kept splats and the kernels read the real count (no host sync)
    const int64_t *n_kept_dev = counts_dev;
    if (counts_dev) n_inst = 1;  // n_kept: the caller's kept capacity; n_inst only meets the zero test below
    const int64_t n_sort = counts_dev ? n_kept : n;  // keys sorted: all n, or the compacted kept capacity
    const int n_tiles = tiles_x * tiles_y;
    // two-level placement (default; VEGS_PLACE_FLAT=1: the single level, for A/B and tests):
    // level 1 over 4x4-tile blocks, level 2 block by block (see block_place_kernel)
    // Two levels from 4096 tiles up: the single level's scattered 4-byte writes (20M per
    // config-2 view, 48M per config-3 frame) throttle the other stream lanes' compositing,
    // so although each level-2 kernel is latency-bound alone, the pipelined step gains 2%
    // and the 1080p sweep 20%; small views (config 4, 2500 tiles) stay on one level, where
    // the extra launches cost more.  VEGS_PLACE_FLAT=1 / =0 forces one or two
    // levels (tests, A/B)
    const char *flat_env = getenv("VEGS_PLACE_FLAT");
    const bool two = flat_env && flat_env[0] ? flat_env[0] == '0' : n_tiles >= 4096;
    const int bx = (tiles_x + kBlk - 1) / kBlk, by = (tiles_y + kBlk - 1) / kBlk, n_blk = bx * by;
    const int cells_x = two ? bx : tiles_x, cells_y = two ? by : tiles_y, n_cells = cells_x * cells_y;
    const int cell_shift = two ? 6 : 4;  // log2 of the level-1 cell size in pixels
    // coarse list capacity: a (splat, block) entry implies >= 1 tile instance
    const int64_t coarse_cap = two ? (counts_dev ? inst_capacity : n_inst) : 0;
#ifndef VEGS_PLACE_CHUNKS
#define VEGS_PLACE_CHUNKS 2048
#endif
    constexpr int64_t kChunks = VEGS_PLACE_CHUNKS;  // target chunk count: warps for the placement
    const int C = (int)(n_kept > kChunks * 128 ? (n_kept + kChunks - 1) / kChunks : 128);
    const int n_chunks = n_kept > 0 ? (int)((n_kept + C - 1) / C) : 0;
#ifndef VEGS_PLACE_GROUP
#define VEGS_PLACE_GROUP 64
#endif
    const int G = VEGS_PLACE_GROUP, n_groups = (n_chunks + G - 1) / G;  // chunks per scan group
    size_t t_depth = 0, t_scan = 0, t_tiles = 0;
    {
        cub::DoubleBuffer<uint32_t> dk(nullptr, nullptr), dv(nullptr, nullptr);
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_depth, dk, dv, n_sort, 0, 32, s));
        uint32_t *u = nullptr;
        int32_t *v = nullptr;
        VEGS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, u, v, n_tiles, s));
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_tiles, u, u, v, v, n_tiles, 0, 16, s));
    }
    size_t t_max = t_depth > t_scan ? t_depth : t_scan;
    t_max = t_max > t_tiles ? t_max : t_tiles;
    const size_t b_n = align_up(sizeof(uint32_t) * (n + 1)), b_t = align_up(sizeof(uint32_t) * n_tiles);
    const size_t b_cnt = align_up(sizeof(uint32_t) * (size_t)n_chunks * n_cells);
    size_t b_grp = align_up(sizeof(uint32_t) * (size_t)n_groups * n_cells);
    if (two) {  // reused for the tile difference array
        const size_t b_diff = align_up(sizeof(int) * (size_t)(tiles_x + 1) * (tiles_y + 1));
        b_grp = b_grp > b_diff ? b_grp : b_diff;
    }
    const size_t b_blk = two ? 3 * align_up(sizeof(uint32_t) * n_blk) : 0;
    const size_t b_coarse = align_up(sizeof(uint32_t) * (size_t)(coarse_cap > 0 ? coarse_cap : 1));
    const size_t b_rect = cull_record ? align_up(sizeof(int4) * n) : 0;
    const size_t need = 4 * b_n + b_cnt + b_grp + 4 * b_t + align_up(t_max) + b_rect + b_blk + (two ? b_coarse : 0);
    if (!ws) {
        *ws_bytes = need;
        return VEGS_OK;
    }
    if (*ws_bytes < need) return VEGS_ERR_CAPACITY;
    char *w = (char *)ws;
    int4 *brect = (int4 *)w; w += b_rect;
    uint32_t *dk0 = (uint32_t *)w; w += b_n;
    uint32_t *dk1 = (uint32_t *)w; w += b_n;
    uint32_t *id0 = (uint32_t *)w; w += b_n;
    uint32_t *id1 = (uint32_t *)w; w += b_n;
    uint32_t *counts = (uint32_t *)w; w += b_cnt;
    uint32_t *gsum = (uint32_t *)w; w += b_grp;
    uint32_t *total = (uint32_t *)w; w += b_t;
    uint32_t *tkey0 = (uint32_t *)w; w += b_t;
    uint32_t *tkey1 = (uint32_t *)w; w += b_t;
    int32_t *tval = (int32_t *)w; w += b_t;
    uint32_t *ctotal = nullptr, *coarse = nullptr;
    int32_t *cstart = nullptr, *cend = nullptr;
    if (two) {
        const size_t b1 = align_up(sizeof(uint32_t) * n_blk);
        ctotal = (uint32_t *)w; w += b1;
        cstart = (int32_t *)w; w += b1;
        cend = (int32_t *)w; w += b1;
        coarse = (uint32_t *)w; w += b_coarse;
    }
    void *tmp = w;
    const size_t tb0 = align_up(t_max);

    if (n_inst == 0 || n_kept == 0) {  // (device counts: a zero kept capacity -- the first, overflowing step)
        VEGS_CUDA(cudaMemsetAsync(tile_start, 0, sizeof(int32_t) * n_tiles, s));
        VEGS_CUDA(cudaMemsetAsync(tile_end, 0, sizeof(int32_t) * n_tiles, s));
    } else {
        // 1. stable depth order of the kept splats (as in bin_sort_impl)
        if (counts_dev) {
            const int64_t m = n > n_sort ? n : n_sort;
            depth_key32_compact_kernel<<<(int)((m + 255) / 256), 256, 0, s>>>(depth_key, kept_idx, n, n_sort,
                                                                              n_kept_dev, dk0, id0);
        } else {
            depth_key32_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(depth_key, n, dk0, id0);
        }
        VEGS_CHECK_LAUNCH();
        cub::DoubleBuffer<uint32_t> dk(dk0, dk1), dv(id0, id1);
        size_t tb = tb0;
        const char *ss_env = getenv("VEGS_SMALL_SORT");  // "0": always the device-wide sort (tests)
        if (n_sort <= kSmallSort && !(ss_env && ss_env[0] == '0')) {  // one CTA (config-4 sized views)
            const int smem = (int)(2 * sizeof(uint32_t) * kSmallSort);
            VEGS_CUDA(cudaFuncSetAttribute(small_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            small_sort_kernel<<<1, kSmallSortT, smem, s>>>(dk0, id0, (int)n_sort, dk1, id1);
            VEGS_CHECK_LAUNCH();
            dk.selector = 1;
            dv.selector = 1;
        } else {
            VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, n_sort, 0, 32, s));
        }
        depth_ties_kernel<<<(int)((n_kept + 255) / 256), 256, 0, s>>>(dk.Current(), depth_key, n_kept, dv.Current(),
                                                                     n_kept_dev);
        VEGS_CHECK_LAUNCH();
        const uint32_t *ids = dv.Current();
        const int4 *bin_rect = (const int4 *)rect;
        if (cull_record) {  // the tight binning rects (all n splats: culled ones are never read)
            bin_rect_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(cull_record, rs, (const int4 *)rect, n, brect);
            VEGS_CHECK_LAUNCH();
            bin_rect = brect;
        }
        // 2. per-chunk cell counts -> first slot of every chunk in every cell, cell ranges
        //    (cells: the tiles, or with two levels the 4x4-tile blocks)
        const size_t diff_bytes = sizeof(int) * (size_t)(cells_x + 1) * (cells_y + 1);
        uint32_t *ctot = two ? ctotal : total;
        int32_t *c_start = two ? cstart : tile_start, *c_end = two ? cend : tile_end;
        chunk_count_kernel<<<n_chunks, 256, diff_bytes, s>>>(ids, bin_rect, n_kept, C, cells_x, cells_y, counts,
                                                             n_kept_dev, cell_shift);
        VEGS_CHECK_LAUNCH();
        const int64_t ng = (int64_t)n_groups * n_cells;
        chunk_group_sum_kernel<<<(int)((ng + 255) / 256), 256, 0, s>>>(counts, n_chunks, n_cells, G, gsum);
        VEGS_CHECK_LAUNCH();
        tile_group_scan_kernel<<<(n_cells + 255) / 256, 256, 0, s>>>(gsum, n_groups, n_cells, ctot);
        VEGS_CHECK_LAUNCH();
        tb = tb0;
        VEGS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, ctot, c_start, n_cells, s));
        chunk_offsets_kernel<<<(int)((ng + 255) / 256), 256, 0, s>>>(counts, gsum, c_start, ctot, n_chunks,
                                                                     n_cells, G, c_end);
        VEGS_CHECK_LAUNCH();
        // 3. placement, one warp per chunk and band of cell rows
        uint32_t *dst = two ? coarse : sorted_gauss;
        if (n_cells <= 4096 && !two)
            place_kernel<8><<<n_chunks, 32 * 8, sizeof(uint32_t) * n_cells, s>>>(ids, bin_rect, n_kept, C, cells_x,
                                                                               cells_y, counts, dst, n_kept_dev,
                                                                               cell_shift);
        else if (!two)
            place_kernel<4><<<n_chunks, 32 * 4, sizeof(uint32_t) * n_cells, s>>>(ids, bin_rect, n_kept, C, cells_x,
                                                                               cells_y, counts, dst, n_kept_dev,
                                                                               cell_shift);
        else  // level 1 (a few block rows per band)
            place_kernel<VEGS_L1_BANDS><<<n_chunks, 32 * VEGS_L1_BANDS, sizeof(uint32_t) * n_cells, s>>>(
                ids, bin_rect, n_kept, C, cells_x, cells_y, counts, dst, n_kept_dev, cell_shift);
        VEGS_CHECK_LAUNCH();
        if (two) {  // 4. level 2: per block, its tiles' counts, the tile ranges, the runs
            int *tdiff = (int *)gsum;  // the level-1 group sums are consumed: reuse for the tile difference array
            VEGS_CUDA(cudaMemsetAsync(tdiff, 0, sizeof(int) * (size_t)(tiles_x + 1) * (tiles_y + 1), s));
            int diff_blocks = (int)((n_kept + 1023) / 1024);
            diff_blocks = diff_blocks < 148 * 2 ? diff_blocks : 148 * 2;
            const size_t tdiff_bytes = sizeof(int) * (size_t)(tiles_x + 1) * (tiles_y + 1);
            tile_diff_kernel<<<diff_blocks, 256, tdiff_bytes, s>>>(ids, bin_rect, n_kept, tiles_x, tiles_y, tdiff,
                                                                  n_kept_dev);
            VEGS_CHECK_LAUNCH();
            tile_total_kernel<<<1, 1024, tdiff_bytes, s>>>(tdiff, tiles_x, tiles_y, total);
            VEGS_CHECK_LAUNCH();
            tb = tb0;
            VEGS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, total, tile_start, n_tiles, s));
            block_place_kernel<<<n_blk, VEGS_BP_T, 0, s>>>(coarse, cstart, cend, bin_rect, tiles_x, tiles_y, bx, tile_start,
                                                     tile_end, sorted_gauss);
            VEGS_CHECK_LAUNCH();
        }
        if ((inst_pid || order) && !counts_dev && !cull_record) {
            placed_extras_kernel<<<(int)((n_inst + 255) / 256), 256, 0, s>>>(
                sorted_gauss, (const int4 *)rect, offsets, kept_idx, tile_end, n_inst, n_tiles, tiles_x, inst_pid,
                order);
            VEGS_CHECK_LAUNCH();
        }
    }
    // 4. optional launch order for the compositing kernels: heaviest tiles first
    if (tile_order) {
        tile_weight_kernel<<<(n_tiles + 255) / 256, 256, 0, s>>>(tile_start, tile_end, n_tiles, tkey0, tval);
        VEGS_CHECK_LAUNCH();
        size_t tb = tb0;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, tkey0, tkey1, tval, tile_order, n_tiles, 0, 16, s));
    }
    return VEGS_OK;
}

extern "C" int vegs_bin_sort(const uint32_t *tiles, const uint64_t *depth_key, const int32_t *rect,
                             const int64_t *offsets, const int64_t *kept_idx, int64_t n, int64_t n_kept,
                             int64_t n_inst, int32_t width, int32_t height, int32_t tile_size,
                             uint32_t *sorted_gauss, uint32_t *inst_pid, int64_t *order,
                             int32_t *tile_start, int32_t *tile_end, int32_t *tile_order,
                             const float *cull_record, int32_t n_channels, void *ws, size_t *ws_bytes, void *stream) {
    if (!ws_bytes || tile_size != kTile || width < 1 || height < 1) return VEGS_ERR_ARG;
    if (cull_record && ((n_channels != 3 && n_channels != 11) || inst_pid || order)) return VEGS_ERR_ARG;
    // instance positions are int32 (tile ranges, out_last): at most 2^31 - 1 instances per view
    if (n_inst > (int64_t)INT32_MAX || n >= (int64_t(1) << 32)) return VEGS_ERR_ARG;
    if (ws && (n > 0) && (!tiles || !depth_key || !rect || !offsets || !kept_idx)) return VEGS_ERR_ARG;
    if (ws && (!tile_start || !tile_end || (n_inst > 0 && !sorted_gauss))) return VEGS_ERR_ARG;
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int n_tiles = tiles_x * tiles_y;
    cudaStream_t s = (cudaStream_t)stream;
    const char *radix_env = getenv("VEGS_BIN_RADIX");  // test switch: set and not "0"
    const bool force_radix = radix_env && radix_env[0] && radix_env[0] != '0';
    if ((tiles_x + 1) * (tiles_y + 1) <= kMaxPlaceTiles && !force_radix)
        return bin_place_impl(depth_key, rect, offsets, kept_idx, n, n_kept, n_inst, tiles_x, tiles_y, sorted_gauss,
                              inst_pid, order, tile_start, tile_end, tile_order, ws, ws_bytes, s, nullptr,
                              cull_record, cull_record ? rec_stride(n_channels) : 0);
    if (n_tiles <= 65536)
        return bin_sort_impl<uint16_t>(tiles, depth_key, rect, offsets, kept_idx, n, n_kept, n_inst, tiles_x,
                                       n_tiles, sorted_gauss, inst_pid, order, tile_start, tile_end, tile_order, ws,
                                       ws_bytes, s);
    return bin_sort_impl<uint32_t>(tiles, depth_key, rect, offsets, kept_idx, n, n_kept, n_inst, tiles_x, n_tiles,
                                   sorted_gauss, inst_pid, order, tile_start, tile_end, tile_order, ws, ws_bytes, s);
}

extern "C" int vegs_bin_count_dev(uint32_t *tiles, int64_t n, int64_t *offsets, int64_t *kept_idx, int64_t *counts,
                                  int64_t inst_capacity, int64_t kept_capacity, int64_t *step_state, int32_t *poison,
                                  void *ws, size_t *ws_bytes, void *stream) {
    if (!ws) return vegs_bin_count(tiles, n, offsets, kept_idx, counts, ws, ws_bytes, stream);
    if (!step_state || !poison || inst_capacity < 0 || kept_capacity < 0) return VEGS_ERR_ARG;
    const int rc = vegs_bin_count(tiles, n, offsets, kept_idx, counts, ws, ws_bytes, stream);
    if (rc != VEGS_OK) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    capacity_check_kernel<<<1, 1, 0, s>>>(counts, inst_capacity, kept_capacity, step_state, poison);
    VEGS_CHECK_LAUNCH();
    capacity_empty_kernel<<<(int)((n + 1 + 255) / 256), 256, 0, s>>>(poison, tiles, n, offsets, kept_idx);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" int vegs_bin_sort_dev(const uint64_t *depth_key, const int32_t *rect, const int64_t *offsets,
                                 const int64_t *kept_idx, int64_t n, const int64_t *counts, int64_t kept_capacity,
                                 int64_t inst_capacity,
                                 int32_t width, int32_t height, int32_t tile_size, uint32_t *sorted_gauss,
                                 int32_t *tile_start, int32_t *tile_end, int32_t *tile_order,
                                 const float *cull_record, int32_t n_channels, void *ws, size_t *ws_bytes,
                                 void *stream) {
    if (!ws_bytes || tile_size != kTile || width < 1 || height < 1 || !counts || inst_capacity < 0) return VEGS_ERR_ARG;
    if (cull_record && n_channels != 3 && n_channels != 11) return VEGS_ERR_ARG;
    if (n >= (int64_t(1) << 31)) return VEGS_ERR_ARG;
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    if ((tiles_x + 1) * (tiles_y + 1) > kMaxPlaceTiles) return VEGS_ERR_ARG;  // radix path needs host counts
    if (ws && (n > 0) && (!depth_key || !rect)) return VEGS_ERR_ARG;
    if (ws && (!tile_start || !tile_end || !sorted_gauss)) return VEGS_ERR_ARG;
    const int64_t kc = kept_capacity < n ? kept_capacity : n;
    return bin_place_impl(depth_key, rect, offsets, kept_idx, n, kc, 1, tiles_x, tiles_y, sorted_gauss, nullptr,
                          nullptr, tile_start, tile_end, tile_order, ws, ws_bytes, (cudaStream_t)stream, counts,
                          cull_record, cull_record ? rec_stride(n_channels) : 0, inst_capacity);
}
