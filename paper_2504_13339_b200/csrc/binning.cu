// Tile binning: the device form of _build_instances (pipeline.py:163-194).
//
//   np.repeat over kept splats  ->  one exclusive scan of packed (kept, tiles) counters
//   np.lexsort((depth, tile))   ->  stable radix sort of the kept float64 depths (rank),
//                                   then one radix sort of key = tile << rank_bits | rank
//   np.searchsorted ranges      ->  boundary scatter over the sorted keys
//
// key order equals lexsort order exactly: tiles compare first, equal tiles compare by
// depth, equal depths by kept index (the stable rank) -- the same tie-break lexsort
// applies to the repeat-ordered instance list.  Keys are 32-bit whenever
// tile_bits + rank_bits <= 32 (configs 0-2), else 64-bit.

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

__global__ void rank_kernel(const uint32_t *sorted_ids, int64_t n_kept, uint32_t *rank) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_kept) rank[sorted_ids[i]] = (uint32_t)i;
}

// One warp per Gaussian: lanes stride over the splat's tiles (row-major, pipeline.py:181-187).
template <typename Key>
__global__ void duplicate_kernel(const uint32_t *tiles, const int32_t *rect, const int64_t *offsets,
                                 const uint32_t *rank, int64_t n, int tiles_x, int rank_bits,
                                 Key *keys, uint32_t *vals, uint32_t *inst_gauss) {
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= n) return;
    const uint32_t cnt = tiles[g];
    if (cnt == 0) return;
    const int x0 = rect[4 * g] / kTile, x1 = (rect[4 * g + 1] - 1) / kTile;
    const int y0 = rect[4 * g + 2] / kTile;
    const int nx = x1 - x0 + 1;
    const int64_t base = offsets[g];
    const Key r = (Key)rank[g];
    for (uint32_t j = lane; j < cnt; j += 32) {
        const int dy = (int)(j / nx), dx = (int)(j - dy * nx);
        const Key tile = (Key)((y0 + dy) * tiles_x + (x0 + dx));
        const int64_t p = base + j;
        keys[p] = (tile << rank_bits) | r;
        vals[p] = (uint32_t)p;
        inst_gauss[p] = (uint32_t)g;
    }
}

// For each sorted instance: Gaussian id, optional kept index (`order`), and the
// searchsorted tile ranges (empty tiles get start == end == insertion point).
template <typename Key>
__global__ void finalize_kernel(const Key *keys, const uint32_t *vals, const uint32_t *inst_gauss,
                                const int64_t *kept_idx, int64_t n_inst, int rank_bits, int n_tiles,
                                uint32_t *sorted_gauss, int64_t *order, int32_t *tile_start,
                                int32_t *tile_end) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_inst) return;
    const uint32_t gid = inst_gauss[vals[s]];
    sorted_gauss[s] = gid;
    if (order) order[s] = kept_idx[gid];
    const int tile = (int)(keys[s] >> rank_bits);
    const int prev = s > 0 ? (int)(keys[s - 1] >> rank_bits) : -1;
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

template <typename Key>
static int bin_sort_impl(const uint32_t *tiles, const uint64_t *depth_key, const int32_t *rect,
                         const int64_t *offsets, const int64_t *kept_idx, int64_t n, int64_t n_kept,
                         int64_t n_inst, int tiles_x, int n_tiles, int key_bits,
                         uint32_t *sorted_gauss, uint32_t *inst_pid, int64_t *order, int32_t *tile_start,
                         int32_t *tile_end, void *ws, size_t *ws_bytes, cudaStream_t s) {
    // workspace: depth sort (keys u64 x2, ids u32 x2, rank u32), instance keys x2, vals alt,
    // inst_gauss, cub temp (max of both sorts)
    size_t t_depth = 0, t_inst = 0;
    {
        cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
        cub::DoubleBuffer<uint32_t> dv(nullptr, nullptr);
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_depth, dk, dv, (int64_t)n, 0, 64, s));
        cub::DoubleBuffer<Key> ik(nullptr, nullptr);
        cub::DoubleBuffer<uint32_t> iv(nullptr, nullptr);
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_inst, ik, iv, (int64_t)n_inst, 0, key_bits, s));
    }
    const size_t b_dk = align_up(sizeof(uint64_t) * n), b_id = align_up(sizeof(uint32_t) * n);
    const size_t b_k = align_up(sizeof(Key) * n_inst), b_v = align_up(sizeof(uint32_t) * n_inst);
    const size_t b_tmp = align_up(t_depth > t_inst ? t_depth : t_inst);
    const size_t need = 2 * b_dk + 3 * b_id + 2 * b_k + 2 * b_v + b_tmp;
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
    Key *k0 = (Key *)w; w += b_k;
    Key *k1 = (Key *)w; w += b_k;
    uint32_t *v1 = (uint32_t *)w; w += b_v;
    uint32_t *inst_gauss = (uint32_t *)w; w += b_v;
    void *tmp = w;

    if (n_inst == 0) {
        VEGS_CUDA(cudaMemsetAsync(tile_start, 0, sizeof(int32_t) * n_tiles, s));
        VEGS_CUDA(cudaMemsetAsync(tile_end, 0, sizeof(int32_t) * n_tiles, s));
        return VEGS_OK;
    }
    // 1. stable depth rank of the kept splats (culled ones carry the max key)
    VEGS_CUDA(cudaMemcpyAsync(dk0, depth_key, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, s));
    iota_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(id0, n);
    VEGS_CHECK_LAUNCH();
    {
        cub::DoubleBuffer<uint64_t> dk(dk0, dk1);
        cub::DoubleBuffer<uint32_t> dv(id0, id1);
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int64_t)n, 0, 64, s));
        rank_kernel<<<(int)((n_kept + 255) / 256), 256, 0, s>>>(dv.Current(), n_kept, rank);
        VEGS_CHECK_LAUNCH();
    }
    // 2. duplicate into tiles
    const int rank_bits = key_bits - bits_for(n_tiles);
    duplicate_kernel<Key><<<(int)((n * 32 + 255) / 256), 256, 0, s>>>(
        tiles, rect, offsets, rank, n, tiles_x, rank_bits, k0, inst_pid, inst_gauss);
    VEGS_CHECK_LAUNCH();
    // 3. sort (tile, rank) keys carrying the duplicate-order index
    cub::DoubleBuffer<Key> ik(k0, k1);
    cub::DoubleBuffer<uint32_t> iv(inst_pid, v1);
    {
        size_t tb = b_tmp;
        VEGS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, ik, iv, (int64_t)n_inst, 0, key_bits, s));
    }
    if (iv.Current() != inst_pid)
        VEGS_CUDA(cudaMemcpyAsync(inst_pid, iv.Current(), sizeof(uint32_t) * n_inst,
                                  cudaMemcpyDeviceToDevice, s));
    // 4. gauss ids, kept-index order, tile ranges
    finalize_kernel<Key><<<(int)((n_inst + 255) / 256), 256, 0, s>>>(
        ik.Current(), inst_pid, inst_gauss, kept_idx, n_inst, rank_bits, n_tiles,
        sorted_gauss, order, tile_start, tile_end);
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
    const int key_bits = bits_for(n_tiles) + bits_for(n_kept > 1 ? n_kept : 2);
    cudaStream_t s = (cudaStream_t)stream;
    if (key_bits <= 32)
        return bin_sort_impl<uint32_t>(tiles, depth_key, rect, offsets, kept_idx, n, n_kept, n_inst, tiles_x,
                                       n_tiles, key_bits, sorted_gauss, inst_pid, order, tile_start,
                                       tile_end, ws, ws_bytes, s);
    return bin_sort_impl<uint64_t>(tiles, depth_key, rect, offsets, kept_idx, n, n_kept, n_inst, tiles_x,
                                   n_tiles, key_bits, sorted_gauss, inst_pid, order, tile_start, tile_end,
                                   ws, ws_bytes, s);
}
