// Tile binning: the device form of _build_instances (pipeline.py:163-194).
//
//   np.repeat over kept splats  ->  one exclusive scan of packed (kept, tiles) counters
//   np.lexsort((depth, tile))   ->  (1) stable radix sort of the kept splats' float64 depth
//                                   keys; (2) instances duplicated *in depth order*; (3) a
//                                   stable radix sort on the tile id alone (12-16 bits)
//   np.searchsorted ranges      ->  boundary scatter over the sorted tile ids
//
// Stability makes the result exactly lexsort's: equal tiles keep depth order, equal
// depths keep kept-index order (step 1 is stable on Gaussian index), and one splat never
// has two instances in a tile.  Sorting only the tile id (2 onesweep passes on 16-bit
// keys) instead of a (tile, depth-rank) key saves half the passes and a third of the
// bytes per pass.  Instance payloads are the duplicate-order index p (rows of one
// Gaussian are contiguous in p, which the deterministic backward reduction relies on).

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

__global__ void iota_kernel(uint32_t *out, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint32_t)i;
}

// depth rank of each kept splat + its tile count in depth order
__global__ void rank_kernel(const uint32_t *sorted_ids, const uint32_t *tiles, int64_t n_kept, uint32_t *rank,
                            uint32_t *count_d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n_kept) return;
    if (i == n_kept) {
        count_d[i] = 0u;
        return;
    }
    const uint32_t g = sorted_ids[i];
    rank[g] = (uint32_t)i;
    count_d[i] = tiles[g];
}

// One warp per Gaussian: lanes stride over the splat's tiles (row-major, pipeline.py:181-187),
// writing tile keys at depth-order positions and duplicate-order payloads.
template <typename TKey>
__global__ void duplicate_kernel(const uint32_t *tiles, const int32_t *rect, const int64_t *offsets,
                                 const uint32_t *rank, const uint32_t *offs_d, int64_t n, int tiles_x, TKey *keys,
                                 uint32_t *vals, uint32_t *inst_gauss) {
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= n) return;
    const uint32_t cnt = tiles[g];
    if (cnt == 0) return;
    const int x0 = rect[4 * g] / kTile, x1 = (rect[4 * g + 1] - 1) / kTile;
    const int y0 = rect[4 * g + 2] / kTile;
    const int nx = x1 - x0 + 1;
    const int64_t base_p = offsets[g];
    const int64_t base_d = offs_d[rank[g]];
    for (uint32_t j = lane; j < cnt; j += 32) {
        const int dy = (int)(j / nx), dx = (int)(j - dy * nx);
        keys[base_d + j] = (TKey)((y0 + dy) * tiles_x + (x0 + dx));
        vals[base_d + j] = (uint32_t)(base_p + j);
        inst_gauss[base_p + j] = (uint32_t)g;
    }
}

// For each sorted instance: Gaussian id, optional kept index (`order`), and the
// searchsorted tile ranges (empty tiles get start == end == insertion point).
template <typename TKey>
__global__ void finalize_kernel(const TKey *keys, const uint32_t *vals, const uint32_t *inst_gauss,
                                const int64_t *kept_idx, int64_t n_inst, int n_tiles, uint32_t *sorted_gauss,
                                int64_t *order, int32_t *tile_start, int32_t *tile_end) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_inst) return;
    const uint32_t gid = inst_gauss[vals[s]];
    sorted_gauss[s] = gid;
    if (order) order[s] = kept_idx[gid];
    const int tile = (int)keys[s];
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
                         int64_t *order, int32_t *tile_start, int32_t *tile_end, void *ws, size_t *ws_bytes,
                         cudaStream_t s) {
    const int tile_bits = bits_for(n_tiles);
    size_t t_depth = 0, t_scan = 0, t_inst = 0;
    {
        cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
        cub::DoubleBuffer<uint32_t> dv(nullptr, nullptr);
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_depth, dk, dv, (int64_t)n, 0, 64, s));
        uint32_t *dummy = nullptr;
        VEGS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, dummy, dummy, (int64_t)n_kept + 1, s));
        cub::DoubleBuffer<TKey> ik(nullptr, nullptr);
        cub::DoubleBuffer<uint32_t> iv(nullptr, nullptr);
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_inst, ik, iv, (int64_t)n_inst, 0, tile_bits, s));
    }
    const size_t b_dk = align_up(sizeof(uint64_t) * n), b_id = align_up(sizeof(uint32_t) * (n + 1));
    const size_t b_k = align_up(sizeof(TKey) * n_inst), b_v = align_up(sizeof(uint32_t) * n_inst);
    size_t t_max = t_depth > t_inst ? t_depth : t_inst;
    t_max = t_max > t_scan ? t_max : t_scan;
    const size_t b_tmp = align_up(t_max);
    const size_t need = 2 * b_dk + 5 * b_id + 2 * b_k + 2 * b_v + b_tmp;
    if (!ws) {
        *ws_bytes = need;
        return VEGS_OK;
    }
    if (*ws_bytes < need) return VEGS_ERR_CAPACITY;
    char *w = (char *)ws;
    uint64_t *dk0 = (uint64_t *)w; w += b_dk;
    uint64_t *dk1 = (uint64_t *)w; w += b_dk;
    uint32_t *id0 = (uint32_t *)w; w += b_id;
    uint32_t *id1 = (uint32_t *)w; w += b_id;
    uint32_t *rank = (uint32_t *)w; w += b_id;
    uint32_t *count_d = (uint32_t *)w; w += b_id;
    uint32_t *offs_d = (uint32_t *)w; w += b_id;
    TKey *k0 = (TKey *)w; w += b_k;
    TKey *k1 = (TKey *)w; w += b_k;
    uint32_t *v1 = (uint32_t *)w; w += b_v;
    uint32_t *inst_gauss = (uint32_t *)w; w += b_v;
    void *tmp = w;

    if (n_inst == 0) {
        VEGS_CUDA(cudaMemsetAsync(tile_start, 0, sizeof(int32_t) * n_tiles, s));
        VEGS_CUDA(cudaMemsetAsync(tile_end, 0, sizeof(int32_t) * n_tiles, s));
        return VEGS_OK;
    }
    // 1. stable depth order of the kept splats (culled ones carry the max key, sort last)
    VEGS_CUDA(cudaMemcpyAsync(dk0, depth_key, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, s));
    iota_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(id0, n);
    VEGS_CHECK_LAUNCH();
    {
        cub::DoubleBuffer<uint64_t> dk(dk0, dk1);
        cub::DoubleBuffer<uint32_t> dv(id0, id1);
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int64_t)n, 0, 64, s));
        rank_kernel<<<(int)((n_kept + 1 + 255) / 256), 256, 0, s>>>(dv.Current(), tiles, n_kept, rank, count_d);
        VEGS_CHECK_LAUNCH();
    }
    // 2. instance offsets in depth order, then duplication (tile keys in depth order)
    {
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, count_d, offs_d, (int64_t)n_kept + 1, s));
    }
    duplicate_kernel<TKey><<<(int)((n * 32 + 255) / 256), 256, 0, s>>>(tiles, rect, offsets, rank, offs_d, n,
                                                                       tiles_x, k0, inst_pid, inst_gauss);
    VEGS_CHECK_LAUNCH();
    // 3. stable sort on the tile id only
    cub::DoubleBuffer<TKey> ik(k0, k1);
    cub::DoubleBuffer<uint32_t> iv(inst_pid, v1);
    {
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, ik, iv, (int64_t)n_inst, 0, tile_bits, s));
    }
    if (iv.Current() != inst_pid)
        VEGS_CUDA(cudaMemcpyAsync(inst_pid, iv.Current(), sizeof(uint32_t) * n_inst, cudaMemcpyDeviceToDevice, s));
    // 4. gauss ids, kept-index order, tile ranges
    finalize_kernel<TKey><<<(int)((n_inst + 255) / 256), 256, 0, s>>>(ik.Current(), inst_pid, inst_gauss, kept_idx,
                                                                      n_inst, n_tiles, sorted_gauss, order,
                                                                      tile_start, tile_end);
    VEGS_CHECK_LAUNCH();
    return VEGS_OK;
}

extern "C" int vegs_bin_sort(const uint32_t *tiles, const uint64_t *depth_key, const int32_t *rect,
                             const int64_t *offsets, const int64_t *kept_idx, int64_t n, int64_t n_kept,
                             int64_t n_inst, int32_t width, int32_t height, int32_t tile_size,
                             uint32_t *sorted_gauss, uint32_t *inst_pid, int64_t *order,
                             int32_t *tile_start, int32_t *tile_end, void *ws, size_t *ws_bytes,
                             void *stream) {
    if (!ws_bytes || tile_size != kTile || width < 1 || height < 1) return VEGS_ERR_ARG;
    if (n_inst >= (int64_t(1) << 32) || n >= (int64_t(1) << 32)) return VEGS_ERR_ARG;
    if (ws && (n > 0) && (!tiles || !depth_key || !rect || !offsets || !kept_idx)) return VEGS_ERR_ARG;
    if (ws && (!tile_start || !tile_end || (n_inst > 0 && (!sorted_gauss || !inst_pid)))) return VEGS_ERR_ARG;
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int n_tiles = tiles_x * tiles_y;
    cudaStream_t s = (cudaStream_t)stream;
    if (n_tiles <= 65536)
        return bin_sort_impl<uint16_t>(tiles, depth_key, rect, offsets, kept_idx, n, n_kept, n_inst, tiles_x,
                                       n_tiles, sorted_gauss, inst_pid, order, tile_start, tile_end, ws, ws_bytes, s);
    return bin_sort_impl<uint32_t>(tiles, depth_key, rect, offsets, kept_idx, n, n_kept, n_inst, tiles_x, n_tiles,
                                   sorted_gauss, inst_pid, order, tile_start, tile_end, ws, ws_bytes, s);
}
