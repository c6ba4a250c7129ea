// binning.cu -- K3-K5: tile binning, exact max-alpha culling, stable sort,
// tile ranges.  bin_and_sort, forward.py:184-255; _cull_pairs, forward.py:112-159.
//
// The reference orders pairs by (tile, stable depth rank, row).  Instead of one
// 64-bit (tile<<32 | depth) radix sort over all P pairs (44 significant bits =
// 6 onesweep passes over 12 B/pair), the rows are first sorted once by depth
// (M keys, 32 bits) and the pairs are EMITTED in depth-rank order; a stable
// radix sort on the tile id alone (ceil(log2(n_tiles)) bits: 2 passes over
// 8 B/pair at 1280x720) then yields exactly the reference order.
#include <cub/cub.cuh>

#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

struct TileGeom {
    int32_t width, height, tiles_x, tiles_y;
};

// Candidate tile rectangle of one row; returns false when the cutoff box
// misses the image (forward.py:204-216).
template <typename T>
__device__ __forceinline__ bool tile_rect(const T rec[12], const TileGeom &g, int &tx0, int &tx1,
                                          int &ty0, int &ty1)
{
    const T u = rec[R_MX], v = rec[R_MY], r = rec[R_RAD];
    const T Wm1 = (T)(g.width - 1), Hm1 = (T)(g.height - 1);
    if (!((u + r >= (T)0) && (u - r <= Wm1) && (v + r >= (T)0) && (v - r <= Hm1))) return false;
    const T ts = (T)kTile;
    auto clampi = [](T f, int hi) -> int { return f < (T)0 ? 0 : (f > (T)hi ? hi : (int)f); };
    tx0 = clampi(rfloor((u - r) / ts), g.tiles_x - 1);
    tx1 = clampi(rfloor((u + r) / ts), g.tiles_x - 1);
    ty0 = clampi(rfloor((v - r) / ts), g.tiles_y - 1);
    ty1 = clampi(rfloor((v + r) / ts), g.tiles_y - 1);
    return true;
}

// Exact min of the Mahalanobis form over the tile's pixel-centre rectangle
// (edges with the clamped stationary point, which covers the corners);
// keep iff qmin <= q_cut.  Same float operations as the numba kernel.
// boc = b / c and boa = b / a are per-row constants of the numba loop
// (forward.py:131-147), computed once per row by the caller.
template <typename T>
__device__ __forceinline__ bool cull_keep(const T rec[12], T boc, T boa, int tx, int ty,
                                          const TileGeom &g)
{
    const T mx = rec[R_MX], my = rec[R_MY], a = rec[R_A], b = rec[R_B], c = rec[R_C];
    const T x0 = (T)(tx * kTile), y0 = (T)(ty * kTile);
    const T x1 = (T)min(tx * kTile + kTile - 1, g.width - 1);
    const T y1 = (T)min(ty * kTile + kTile - 1, g.height - 1);
    if (x0 <= mx && mx <= x1 && y0 <= my && my <= y1) return true;
    T qmin = (T)INFINITY;
    const T two = (T)2;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const T xe = e ? x1 : x0;
        T yv = my - boc * (xe - mx);
        if (yv < y0) yv = y0;
        else if (yv > y1) yv = y1;
        const T dx = xe - mx, dy = yv - my;
        const T q = a * dx * dx + two * b * dx * dy + c * dy * dy;
        if (q < qmin) qmin = q;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const T ye = e ? y1 : y0;
        T xv = mx - boa * (ye - my);
        if (xv < x0) xv = x0;
        else if (xv > x1) xv = x1;
        const T dx = xv - mx, dy = ye - my;
        const T q = a * dx * dx + two * b * dx * dy + c * dy * dy;
        if (q < qmin) qmin = q;
    }
    return qmin <= rec[R_QC];
}

// Pass 1: kept-tile count per row, in depth-rank order.  For rows with at most
// 64 candidate tiles (all but the largest splats) the kept set is also stored
// as a bitmask so the emit pass does not repeat the exact cull tests.
constexpr uint64_t kNoMask = ~0ull;

template <typename T>
__global__ void __launch_bounds__(256) count_kernel(int64_t m, const T *__restrict__ records,
                                                    const uint8_t *__restrict__ valid,
                                                    const uint32_t *__restrict__ order,
                                                    TileGeom g, int cull,
                                                    uint32_t *__restrict__ counts,
                                                    uint64_t *__restrict__ masks)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const uint32_t row = order[r];
    uint32_t cnt = 0;
    uint64_t mask = 0;
    if (valid[row]) {
        T rec[12];
        load_record(records, row, rec);
        int tx0, tx1, ty0, ty1;
        if (tile_rect(rec, g, tx0, tx1, ty0, ty1)) {
            const int nx = tx1 - tx0 + 1, ncand = nx * (ty1 - ty0 + 1);
            if (!cull) {
                cnt = (uint32_t)ncand;
                mask = kNoMask;
            } else {
                const T boc = rec[R_B] / rec[R_C], boa = rec[R_B] / rec[R_A];
                int i = 0;
                for (int ty = ty0; ty <= ty1; ++ty)
                    for (int tx = tx0; tx <= tx1; ++tx, ++i) {
                        const bool k = cull_keep(rec, boc, boa, tx, ty, g);
                        cnt += k;
                        if (k && i < 64) mask |= 1ull << i;
                    }
                if (ncand > 64) mask = kNoMask;
            }
        }
    }
    counts[r] = cnt;
    masks[r] = mask;
}

// Pass 2: emit (tile, row) pairs at the scanned offsets, still in depth order.
template <typename T>
__global__ void __launch_bounds__(256) emit_kernel(int64_t m, const T *__restrict__ records,
                                                   const uint8_t *__restrict__ valid,
                                                   const uint32_t *__restrict__ order,
                                                   const uint32_t *__restrict__ offs, TileGeom g,
                                                   int cull, const uint64_t *__restrict__ masks,
                                                   uint32_t *__restrict__ keys,
                                                   uint32_t *__restrict__ vals,
                                                   const int64_t *__restrict__ status)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= m) return;
    if (status && status[1]) return;  // pair capacity overflow: emit nothing
    uint32_t o = offs[r];
    const uint32_t end = offs[r + 1];
    if (o == end) return;
    const uint32_t row = order[r];
    T rec[12];
    load_record(records, row, rec);
    int tx0, tx1, ty0, ty1;
    tile_rect(rec, g, tx0, tx1, ty0, ty1);
    const int nx = tx1 - tx0 + 1;
    const uint64_t mask = masks[r];
    if (mask != kNoMask) {
        uint64_t bits = mask;
        while (bits) {
            const int i = __ffsll((long long)bits) - 1;
            bits &= bits - 1;
            const int ty = ty0 + i / nx, tx = tx0 + i - (i / nx) * nx;
            keys[o] = (uint32_t)(ty * g.tiles_x + tx);
            vals[o] = row;
            ++o;
        }
        return;
    }
    const T boc = rec[R_B] / rec[R_C], boa = rec[R_B] / rec[R_A];
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            if (cull && !cull_keep(rec, boc, boa, tx, ty, g)) continue;
            keys[o] = (uint32_t)(ty * g.tiles_x + tx);
            vals[o] = row;
            ++o;
        }
}

// status[0] = P, status[1] = overflow (P > capacity)
__global__ void status_kernel(const uint32_t *__restrict__ total, int64_t cap,
                              int64_t *__restrict__ status)
{
    const int64_t P = *total;
    status[0] = P;
    status[1] = P > cap;
}

// sentinel keys past P sort behind every real tile
__global__ void pad_kernel(uint32_t *__restrict__ keys, uint32_t *__restrict__ vals, int64_t cap,
                           int n_tiles, const int64_t *__restrict__ status)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cap) return;
    if (status[1] || i >= status[0]) {
        keys[i] = (uint32_t)n_tiles;
        vals[i] = 0;
    }
}

// CSR offsets[t] = lower_bound(sorted tile ids, t); with a device status the
// count P is read there (and an overflow yields all-empty tiles)
__global__ void ranges_kernel(const uint32_t *__restrict__ tiles, int64_t P, int n_tiles,
                              int32_t *__restrict__ offsets, const int64_t *__restrict__ status)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > n_tiles) return;
    if (status) {
        if (status[1]) { offsets[t] = 0; return; }
        P = status[0];
    }
    int64_t lo = 0, hi = P;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (tiles[mid] < (uint32_t)t) lo = mid + 1;
        else hi = mid;
    }
    offsets[t] = (int32_t)lo;
}

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct BinLayout {
    size_t keys_sorted, order, counts, offs, masks, pkeys, pvals, total, temp, temp_bytes, bytes;
};

static BinLayout bin_layout(int64_t m, int64_t cap)
{
    BinLayout L;
    size_t o = 0;
    const int64_t mm = m > 0 ? m : 1, cc = cap > 0 ? cap : 1;
    L.keys_sorted = o; o += align256(8 * mm);
    L.order = o; o += align256(4 * mm);
    L.counts = o; o += align256(4 * (mm + 1));
    L.offs = o; o += align256(4 * (mm + 1));
    L.masks = o; o += align256(8 * mm);
    L.pkeys = o; o += align256(4 * cc);
    L.pvals = o; o += align256(4 * cc);
    L.total = o; o += 256;
    size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)mm);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)mm);
    cub::DeviceRadixSort::SortPairs(nullptr, t3, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)cc);
    cub::DeviceScan::ExclusiveSum(nullptr, t4, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (int)(mm + 1));
    L.temp_bytes = std::max(std::max(t1, t2), std::max(t3, t4));
    L.temp = o; o += align256(L.temp_bytes);
    L.bytes = o;
    return L;
}

}  // namespace sb

using namespace sb;

extern "C" size_t sb_bin_workspace_bytes(int64_t m, int64_t pair_capacity, int32_t width,
                                         int32_t height)
{
    (void)width; (void)height;
    return bin_layout(m, pair_capacity).bytes;
}

extern "C" int32_t sb_bin(int32_t dtype, int64_t m, const void *records, const uint8_t *valid,
                          void *depth_key, uint32_t *depth_val, int32_t width, int32_t height,
                          int32_t tile_size, int32_t cull, int64_t pair_capacity,
                          int32_t *pair_gaussian, int32_t *pair_tile, int32_t *offsets,
                          int64_t *n_pairs, void *workspace, size_t workspace_bytes,
                          int64_t *d_status, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(tile_size == kTile, "tile_size %d unsupported (only %d)", tile_size, kTile);
    SB_REQUIRE(width > 0 && height > 0, "bad image size %dx%d", width, height);
    SB_REQUIRE(m >= 0 && m < 0x7FFFFFFF, "bad row count");
    SB_REQUIRE(n_pairs != nullptr, "n_pairs is NULL");
    const BinLayout L = bin_layout(m, pair_capacity);
    SB_REQUIRE(workspace_bytes >= L.bytes, "workspace too small: %zu < %zu", workspace_bytes, L.bytes);
    cudaStream_t st = as_stream(stream);
    TileGeom g{width, height, (width + kTile - 1) / kTile, (height + kTile - 1) / kTile};
    const int n_tiles = g.tiles_x * g.tiles_y;
    char *ws = (char *)workspace;
    uint32_t *order = (uint32_t *)(ws + L.order);
    uint32_t *counts = (uint32_t *)(ws + L.counts);
    uint32_t *offs = (uint32_t *)(ws + L.offs);
    uint64_t *masks = (uint64_t *)(ws + L.masks);
    uint32_t *pkeys = (uint32_t *)(ws + L.pkeys);
    uint32_t *pvals = (uint32_t *)(ws + L.pvals);
    void *temp = ws + L.temp;
    size_t temp_bytes = L.temp_bytes;

    if (m == 0) {
        SB_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (n_tiles + 1), st));
        *n_pairs = 0;
        return SB_OK;
    }
    // 1. stable depth sort of the rows (forward.py:248-249); invalid rows last
    if (dtype == SB_F32)
        SB_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, (const uint32_t *)depth_key,
                                                (uint32_t *)(ws + L.keys_sorted), depth_val, order,
                                                (int)m, 0, 32, st));
    else
        SB_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, (const uint64_t *)depth_key,
                                                (uint64_t *)(ws + L.keys_sorted), depth_val, order,
                                                (int)m, 0, 64, st));
    // 2. kept-tile counts in depth order, 3. scan
    const unsigned gm = grid_for(m, 256);
    if (dtype == SB_F32)
        count_kernel<float><<<gm, 256, 0, st>>>(m, (const float *)records, valid, order, g, cull, counts, masks);
    else
        count_kernel<double><<<gm, 256, 0, st>>>(m, (const double *)records, valid, order, g, cull, counts, masks);
    SB_CUDA(cudaGetLastError());
    SB_CUDA(cudaMemsetAsync(counts + m, 0, sizeof(uint32_t), st));
    SB_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offs, (int)(m + 1), st));
    if (d_status != nullptr) {
        // sync-free: P stays on the device; the sort runs over the full
        // capacity with sentinel keys past P; on overflow nothing is emitted,
        // every tile range is empty and d_status[1] = 1 tells the caller (and
        // the step's update kernels) to discard this iteration.
        int bits = 1;
        while ((1 << bits) < n_tiles + 1) ++bits;
        status_kernel<<<1, 1, 0, st>>>(offs + m, pair_capacity, d_status);
        if (dtype == SB_F32)
            emit_kernel<float><<<gm, 256, 0, st>>>(m, (const float *)records, valid, order, offs, g, cull, masks, pkeys, pvals, d_status);
        else
            emit_kernel<double><<<gm, 256, 0, st>>>(m, (const double *)records, valid, order, offs, g, cull, masks, pkeys, pvals, d_status);
        pad_kernel<<<grid_for(pair_capacity, 256), 256, 0, st>>>(pkeys, pvals, pair_capacity, n_tiles, d_status);
        SB_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, pkeys, (uint32_t *)pair_tile, pvals,
                                                (uint32_t *)pair_gaussian, (int)pair_capacity, 0, bits, st));
        ranges_kernel<<<grid_for(n_tiles + 1, 256), 256, 0, st>>>((const uint32_t *)pair_tile, 0,
                                                                   n_tiles, offsets, d_status);
        *n_pairs = -1;
        return check_launch("ranges_kernel");
    }
    uint32_t total = 0;
    SB_CUDA(cudaMemcpyAsync(&total, offs + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    *n_pairs = total;
    SB_REQUIRE(total < 0x7FFFFFFFu, "pair count overflow");
    if ((int64_t)total > pair_capacity) {
        set_error("pair capacity %lld < %u", (long long)pair_capacity, total);
        return SB_ERR_CAPACITY;
    }
    if (total == 0) {
        SB_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (n_tiles + 1), st));
        return SB_OK;
    }
    // 4. emit in depth order
    if (dtype == SB_F32)
        emit_kernel<float><<<gm, 256, 0, st>>>(m, (const float *)records, valid, order, offs, g, cull, masks, pkeys, pvals, nullptr);
    else
        emit_kernel<double><<<gm, 256, 0, st>>>(m, (const double *)records, valid, order, offs, g, cull, masks, pkeys, pvals, nullptr);
    SB_CUDA(cudaGetLastError());
    // 5. stable sort by tile id only
    int bits = 1;
    while ((1 << bits) < n_tiles) ++bits;
    SB_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, pkeys, (uint32_t *)pair_tile, pvals,
                                            (uint32_t *)pair_gaussian, (int)total, 0, bits, st));
    // 6. CSR ranges
    ranges_kernel<<<grid_for(n_tiles + 1, 256), 256, 0, st>>>((const uint32_t *)pair_tile, total,
                                                               n_tiles, offsets, nullptr);
    return check_launch("ranges_kernel");
}
