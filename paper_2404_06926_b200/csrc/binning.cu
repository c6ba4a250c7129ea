// binning.cu -- K3-K5: tile binning, exact max-alpha culling, stable sort,
// tile ranges.  bin_and_sort, forward.py:184-255; _cull_pairs, forward.py:112-159.
//
// The reference orders pairs by (tile, stable depth rank, row).  Instead of one
// 64-bit (tile<<32 | depth) radix sort over all P pairs (44 significant bits =
// 6 onesweep passes over 12 B/pair), the rows are sorted once by depth (M
// keys) and the pairs are then placed by a ONE-pass stable counting sort on
// the tile id, so each pair is written to HBM exactly once (4 B):
//
//   1. stable depth sort of the rows -> order[rank] = row        (CUB, M keys)
//   2. count (+3. histogram, same kernel): per row (depth-rank order) the
//      exact kept-tile count and the kept set -- a 64-bit mask over its
//      candidate rectangle, or, for the rare rows with more than 64
//      candidates, an explicit tile list in a side buffer; the ranks are cut
//      into chunks of R = 2048 and each chunk's tile histogram is kept in
//      shared memory and stored tile-major: hist[t * C + c]
//   4. exclusive scan of hist (T*C entries, L2-resident): hist[t * C + c] is
//      now where chunk c's first pair of tile t goes; hist[t * C] is the CSR
//      offset of tile t, hist[T * C] = P
//   5. place: one CTA per chunk walks its pair stream in windows of 2048
//      pairs (8 consecutive pairs per thread); a block-wide stable radix
//      sort
//      of the window by tile id (on-chip) gives each pair its rank inside its
//      tile's run, and a per-tile cursor in shared memory (seeded from step 4)
//      its global slot.
//
// Chunks are placed in rank order, windows in rank order inside a chunk and
// the window sort is stable, so every tile list comes out in depth-rank order
// -- exactly the reference order, deterministic, no pair-sized sort passes.
//
// For the deterministic backward (blend_bwd.cu) the passes also leave a map
// from pairs to a rank-major index: rank_of[row] = r (count), rank_e0[r] =
// the exclusive prefix of the kept counts in rank order (place: per-chunk
// totals + the in-chunk prefix), so the j-th kept tile of rank r (tiles
// ascending) is pair e = rank_e0[r] + j; the backward stores each replayed
// pair's partial adjoints at e, and every row's partials are contiguous, in
// ascending tile order -- the reference's merge order (backward.py:92-98) --
// reduced with no float atomics (gather_short_kernel below).
#include <cub/cub.cuh>

#include <mutex>

#include "abi_util.cuh"
#include "common.cuh"

namespace sb {
constexpr uint32_t kNoRow = 0xFFFFFFFFu;   // padding rank of a bounded sort
}

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
__device__ __forceinline__ bool cull_keep_f(T mx, T my, T a, T b, T c, T qc, T boc, T boa,
                                            int tx, int ty, const TileGeom &g)
{
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
    return qmin <= qc;
}

template <typename T>
__device__ __forceinline__ bool cull_keep(const T rec[12], T boc, T boa, int tx, int ty,
                                          const TileGeom &g)
{
    return cull_keep_f(rec[R_MX], rec[R_MY], rec[R_A], rec[R_B], rec[R_C], rec[R_QC], boc, boa,
                       tx, ty, g);
}

// ---------------------------------------------------------------------------
constexpr int kBinThreads = 256;
constexpr int kRowsPerThread = 4;                        // rows per thread per chunk
constexpr int kChunkRows = kBinThreads * kRowsPerThread; // R
constexpr int kMaxTiles = 32768;                         // 16-bit tile keys, smem cursors
constexpr int kMaxCoarse = 4096;                         // coarse depth-limit cells
constexpr uint32_t kBig = kGeoBig;                       // geo flag: explicit tile list

// geo word of a row: first candidate tile (16 bits) | (nx - 1) << 16, or kBig
// (then the mask word holds the row's offset in the explicit tile list)
__device__ __forceinline__ uint32_t geo_word(int tbase, int nx) { return (uint32_t)tbase | (uint32_t)(nx - 1) << 16; }

// tile of candidate bit i (i < 64) of a masked row; (i + 0.5) / nx is exact
// enough in float for i < 64 to give floor(i / nx) without an integer divide
__device__ __forceinline__ int bit_tile(uint32_t geo, int i, float inv_nx, int tiles_x)
{
    const int nx = (int)((geo >> 16) & 0x7F) + 1;
    const int dy = (int)(((float)i + 0.5f) * inv_nx);
    return (int)(geo & 0xFFFF) + dy * tiles_x + (i - dy * nx);
}

__device__ __forceinline__ float geo_inv_nx(uint32_t geo) { return __frcp_rn((float)(((geo >> 16) & 0x7F) + 1)); }

// Invalid rows carry the all-ones depth key and sort behind every valid row:
// a chunk whose first rank is invalid is entirely invalid (with the engine's
// depth-limit drop in sb_preprocess_fwd that is most chunks).
template <typename T>
__device__ __forceinline__ bool rank_invalid(const void *keys_sorted, int64_t r)
{
    if (sizeof(T) == 4) return __ldg(reinterpret_cast<const uint32_t *>(keys_sorted) + r) == 0xFFFFFFFFu;
    return __ldg(reinterpret_cast<const unsigned long long *>(keys_sorted) + r) == 0xFFFFFFFFFFFFFFFFull;
}

// Passes 2+3: kept-tile count and kept set per row (depth-rank order) and the
// chunk's tile histogram, in one kernel: one CTA per chunk, 8 warps, each
// warp takes 32 rows at a time and spreads their candidate tiles evenly over
// its lanes (a row's exact cull tests are the expensive, variable part), so a
// warp runs ceil(candidates / 32) uniform iterations instead of the longest
// row's count.  Rows with more than 64 candidates (the explicit-list rows) are
// walked afterwards by the whole warp, one row at a time.
constexpr int kCountWarps = 32;
constexpr int kCountThreads = 32 * kCountWarps;
constexpr int kSmallChunk = 256;                 // rows per chunk for small maps
constexpr int64_t kSmallMapRows = 262144;        // up to here: 256-row chunks

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// CW: warps per CTA = rows per chunk / 32 (32 for 1024-row chunks, 8 for the
// 256-row chunks of small maps, which would otherwise leave most SMs idle)
template <typename T, int CW = kCountWarps>
__global__ void __launch_bounds__(32 * CW) count_hist_kernel(
    int64_t m, const T *__restrict__ records, const uint8_t *__restrict__ valid,
    const uint32_t *__restrict__ order, TileGeom g, int cull, int n_chunks,
    uint32_t *__restrict__ counts, uint64_t *__restrict__ masks, uint32_t *__restrict__ geo,
    uint16_t *__restrict__ big, int64_t big_cap, unsigned long long *__restrict__ big_total,
    uint32_t *__restrict__ hist, const float *__restrict__ dlim, int coarse,
    const void *__restrict__ keys_sorted, uint32_t *__restrict__ chunk_tot,
    uint32_t *__restrict__ rank_of, uint8_t *__restrict__ rank_hit)
{
    extern __shared__ uint32_t h[];
    __shared__ uint32_t smask[CW][32][2];
    constexpr int kThr = 32 * CW, kChunk = 32 * CW;
    // dlim (nullable): per-tile depth limit; a pair behind its tile's limit is
    // neither culled nor counted, so the tile's list ends there
    auto within = [&](T depth, int t) -> bool { return !dlim || depth <= (T)__ldg(dlim + t); };
    const int n_tiles = g.tiles_x * g.tiles_y;
    // counts and the histogram are zeroed by the caller (two coalesced
    // memsets): a chunk of invalid rows writes nothing, a valid chunk only
    // its non-zero tile counts -- the scattered zero stores of ~3/4 of the
    // chunks (depth-limited steady state) left warps stalled draining them
    if (keys_sorted && rank_invalid<T>(keys_sorted, (int64_t)blockIdx.x * kChunk)) {
        if (threadIdx.x == 0) chunk_tot[blockIdx.x] = 0;
        return;
    }
    // coarse grid (4x4 tiles) of the limits' maxima: rows behind every limit
    // under their rectangle skip the candidate loop altogether
    const int cgx = (g.tiles_x + 3) >> 2;
    uint32_t *cmax = h + n_tiles;   // [coarse cells], float bits (limits are >= 0)
    for (int t = threadIdx.x; t < n_tiles; t += kThr) h[t] = 0;
    if (coarse)
        for (int k = threadIdx.x; k < coarse; k += kThr) cmax[k] = 0;
    __syncthreads();
    if (coarse) {
        for (int t = threadIdx.x; t < n_tiles; t += kThr) {
            const int ty = t / g.tiles_x, tx = t - ty * g.tiles_x;
            atomicMax(cmax + (ty >> 2) * cgx + (tx >> 2), __float_as_uint(__ldg(dlim + t)));
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kWarpRows = kChunk / CW;   // 32: one row per lane
    const int64_t wbase = (int64_t)blockIdx.x * kChunk + (int64_t)warp * kWarpRows;

    for (int bt = 0; bt < kWarpRows; bt += 32) {
        const int64_t r = wbase + bt + lane;
        T mx = 0, my = 0, a = 1, b = 0, c = 1, qc = 0, boc = 0, boa = 0, dep = 0;
        int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;
        bool have = false;
        uint32_t row = 0;
        if (r < m) {
            row = order[r];
            rank_hit[r] = 0;                 // set by the deterministic backward
            if (row != kNoRow && valid[row]) {
                rank_of[row] = (uint32_t)r;
                T rec[12];
                load_record(records, row, rec);
                have = tile_rect(rec, g, tx0, tx1, ty0, ty1);
                mx = rec[R_MX]; my = rec[R_MY]; a = rec[R_A]; b = rec[R_B]; c = rec[R_C];
                qc = rec[R_QC];
                dep = rec[R_DEP];
                if (have && coarse) {
                    float lim = 0.f;
                    for (int cy = ty0 >> 2; cy <= ty1 >> 2; ++cy)
                        for (int cx = tx0 >> 2; cx <= tx1 >> 2; ++cx)
                            lim = fmaxf(lim, __uint_as_float(cmax[cy * cgx + cx]));
                    if (dep > (T)lim) have = false;   // behind every limit: no pairs
                }
                if (have) { boc = b / c; boa = b / a; }
            }
        }
        const int nx = tx1 - tx0 + 1;
        const int ncand = have ? nx * (ty1 - ty0 + 1) : 0;
        const bool is_big = ncand > 64;
        // warp-exclusive offsets of the small rows' candidates
        const int mine = is_big ? 0 : ncand;
        int incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        const int excl = incl - mine;
        const int total = shfl(incl, 31);
        smask[warp][lane][0] = 0;
        smask[warp][lane][1] = 0;
        __syncwarp();
        for (int k0 = 0; k0 < total; k0 += 32) {
            const int k = k0 + lane;
            // owner: last lane whose first candidate is <= k
            int o = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                const int cand = o + step;
                const int v = shfl(excl, cand & 31);
                if (cand < 32 && v <= k) o = cand;
            }
            const int oe = shfl(excl, o), onx = shfl(nx, o), otx0 = shfl(tx0, o),
                      oty0 = shfl(ty0, o);
            const T omx = shfl(mx, o), omy = shfl(my, o), oa = shfl(a, o), ob = shfl(b, o),
                    oc = shfl(c, o), oqc = shfl(qc, o), oboc = shfl(boc, o), oboa = shfl(boa, o),
                    odep = shfl(dep, o);
            if (k < total) {
                const int i = k - oe;
                const int dy = (int)(((float)i + 0.5f) * __frcp_rn((float)onx));
                const int tx = otx0 + i - dy * onx, ty = oty0 + dy;
                if (within(odep, ty * g.tiles_x + tx) &&
                    (!cull || cull_keep_f(omx, omy, oa, ob, oc, oqc, oboc, oboa, tx, ty, g))) {
                    atomicOr(&smask[warp][o][i >> 5], 1u << (i & 31));
                    atomicAdd(&h[ty * g.tiles_x + tx], 1u);
                }
            }
        }
        __syncwarp();
        // big rows (> 64 candidates: an explicit tile list in big[]), one at a
        // time by the whole warp, 32 candidates per trip: a count pass sizes
        // the row's slice of big[], a second pass writes its tiles in
        // candidate (row-major) order.  One lane walking a near, image-sized
        // footprint serially held its warp for thousands of tests (the grown
        // 4M-row map of config 4: 983 us per launch)
        uint32_t cnt = 0;
        uint64_t mask = 0;
        for (unsigned todo = __ballot_sync(0xffffffffu, is_big); todo; todo &= todo - 1) {
            const int o = __ffs(todo) - 1;
            const int onc = shfl(ncand, o), onx = shfl(nx, o), otx0 = shfl(tx0, o),
                      oty0 = shfl(ty0, o);
            const T omx = shfl(mx, o), omy = shfl(my, o), oa = shfl(a, o), ob = shfl(b, o),
                    oc = shfl(c, o), oqc = shfl(qc, o), oboc = shfl(boc, o), oboa = shfl(boa, o),
                    odep = shfl(dep, o);
            auto keep_at = [&](int k, int &t) -> bool {
                if (k >= onc) return false;
                const int dy = k / onx;
                const int tx = otx0 + k - dy * onx, ty = oty0 + dy;
                t = ty * g.tiles_x + tx;
                return within(odep, t) &&
                       (!cull || cull_keep_f(omx, omy, oa, ob, oc, oqc, oboc, oboa, tx, ty, g));
            };
            uint32_t rc = 0;
            for (int k0 = 0; k0 < onc; k0 += 32) {
                int t;
                rc += (uint32_t)__popc(__ballot_sync(0xffffffffu, keep_at(k0 + lane, t)));
            }
            unsigned long long off = 0ull;
            if (lane == o && rc) off = atomicAdd(big_total, (unsigned long long)rc);
            off = __shfl_sync(0xffffffffu, off, o);
            // beyond the capacity P > capacity too: the step is discarded
            const bool fits = rc && (int64_t)(off + rc) <= big_cap;
            uint64_t kk = off;
            for (int k0 = 0; k0 < onc; k0 += 32) {
                int t = 0;
                const bool kp = keep_at(k0 + lane, t);
                const unsigned bal = __ballot_sync(0xffffffffu, kp);
                if (kp) {
                    atomicAdd(&h[t], 1u);
                    if (fits) big[kk + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)t;
                }
                kk += (uint64_t)__popc(bal);
            }
            if (lane == o) { cnt = rc; mask = off; }
        }
        if (r >= m) continue;
        uint32_t gw = kBig;
        if (!is_big) {
            mask = (uint64_t)smask[warp][lane][0] | (uint64_t)smask[warp][lane][1] << 32;
            cnt = (uint32_t)__popcll(mask);
            gw = ncand ? geo_word(ty0 * g.tiles_x + tx0, nx) : 0u;
        }
        counts[r] = cnt;
        masks[r] = mask;
        geo[r] = gw;
    }
    __syncthreads();
    __shared__ uint32_t s_tot;
    if (threadIdx.x == 0) s_tot = 0;
    uint32_t mine_tot = 0;
    for (int t = threadIdx.x; t < n_tiles; t += kThr)
        if (h[t]) {
            hist[(int64_t)t * n_chunks + blockIdx.x] = h[t];
            mine_tot += h[t];
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine_tot += __shfl_xor_sync(0xffffffffu, mine_tot, o);
    __syncthreads();
    if (lane == 0 && mine_tot) atomicAdd(&s_tot, mine_tot);   // integer: order-free
    __syncthreads();
    if (threadIdx.x == 0) chunk_tot[blockIdx.x] = s_tot;   // pairs of this chunk
}

// Pass 4b: CSR offsets and the device status from the scanned histogram, in
// one CTA.  status[0] = P, status[1] = overflow (P > capacity): every range
// empty; or-ed with the caller's halt flag (an earlier invalid iteration).
__global__ void __launch_bounds__(1024) tile_offsets_kernel(
    const uint32_t *__restrict__ hoff, int n_chunks, int n_tiles, int64_t cap,
    int32_t *__restrict__ offsets, int64_t *__restrict__ status, const int *__restrict__ sort_over,
    const int64_t *__restrict__ halt)
{
    const int64_t P = hoff[(int64_t)n_tiles * n_chunks];
    const bool over = P > cap || (sort_over && *sort_over);
    for (int t = threadIdx.x; t < n_tiles; t += 1024)
        offsets[t] = over ? 0 : (int32_t)hoff[(int64_t)t * n_chunks];
    if (threadIdx.x == 0) {
        offsets[n_tiles] = over ? 0 : (int32_t)P;
        if (status) {
            status[0] = P;
            status[1] = over || (halt && *halt);
        }
    }
}

struct MaxOp {
    __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};

// Pass 5: place one chunk's pairs.  One window: generate ITEMS consecutive
// pairs per thread (blocked), stable-sort them by tile on chip, and write
// each to its tile's cursor + its rank in the tile's run.  1024-thread CTAs
// (one row per thread) use 4-bit radix digits so the sort's counters fit
// the static shared memory.
template <int THREADS, int ITEMS>
struct PlaceSort {
    using Sort = cub::BlockRadixSort<uint16_t, THREADS, ITEMS, uint32_t, THREADS >= 1024 ? 4 : 6>;
};

template <int THREADS, int ITEMS, int CH>
__device__ __forceinline__ void place_window(
    uint32_t w0, uint32_t total, const uint32_t *__restrict__ lo_s,
    const uint32_t *__restrict__ s_row, const uint64_t *__restrict__ s_mask,
    const uint32_t *__restrict__ s_geo, const uint16_t *__restrict__ big, int tiles_x,
    int key_bits, uint32_t *__restrict__ cursor,
    typename PlaceSort<THREADS, ITEMS>::Sort::TempStorage &sort_tmp,
    uint16_t *__restrict__ skey, typename cub::BlockScan<int, THREADS>::TempStorage &run_tmp,
    int32_t *__restrict__ pair_gaussian, int32_t *__restrict__ pair_tile)
{
    using Sort = typename PlaceSort<THREADS, ITEMS>::Sort;
    using RunScan = cub::BlockScan<int, THREADS>;
    constexpr int W = THREADS * ITEMS;
    const uint16_t pad = (uint16_t)((1u << key_bits) - 1u);
    const uint32_t wend = min(total, w0 + (uint32_t)W);
    const uint32_t e0 = w0 + threadIdx.x * ITEMS;
    uint16_t key[ITEMS];
    uint32_t val[ITEMS];
    // the row holding pair e0: last q with lo_s[q] <= e0
    int q = 0;
    if (e0 < wend) {
        int a = 0, b = CH;           // lo_s[a] <= e0 < lo_s[b]
        while (b - a > 1) {
            const int mid = (a + b) >> 1;
            if (lo_s[mid] <= e0) a = mid;
            else b = mid;
        }
        q = a;
    }
    // running state of row q: remaining kept bits / list position
    uint64_t rem = 0;
    uint32_t gw = 0, row = 0, j = 0;
    float inv = 1.f;
    int cur = -1;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const uint32_t e = e0 + i;
        key[i] = pad;
        val[i] = 0;
        if (e < wend) {
            while (lo_s[q + 1] <= e) ++q;
            if (q != cur) {
                cur = q;
                row = s_row[q];
                gw = s_geo[q];
                rem = s_mask[q];
                j = e - lo_s[q];
                if (gw != kBig) {
                    inv = geo_inv_nx(gw);
                    for (uint32_t s = 0; s < j; ++s) rem &= rem - 1;
                }
            }
            uint32_t tile;
            if (gw == kBig) {
                tile = big[rem + j];
                ++j;
            } else {
                const int bit = __ffsll((long long)rem) - 1;
                rem &= rem - 1;
                tile = (uint32_t)bit_tile(gw, bit, inv, tiles_x);
            }
            key[i] = (uint16_t)tile;
            val[i] = row;
        }
    }
    Sort(sort_tmp).Sort(key, val, 0, key_bits);   // stable; blocked arrangement
    __syncthreads();
    const int base = threadIdx.x * ITEMS;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) skey[base + i] = key[i];
    __syncthreads();
    int start[ITEMS];
    const uint16_t *tk = key;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const uint16_t prev = i ? tk[i - 1] : (base ? skey[base - 1] : (uint16_t)0xFFFFu);
        start[i] = (base + i == 0 || prev != tk[i]) ? base + i : 0;
    }
    RunScan(run_tmp).InclusiveScan(start, start, MaxOp());
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        if (tk[i] == pad) continue;
        // in range by construction: the scanned histogram bounds every
        // chunk's run of every tile (a capacity overflow never gets here)
        const uint32_t pos = cursor[tk[i]] + (uint32_t)(base + i - start[i]);
        pair_gaussian[pos] = (int32_t)val[i];
        if (pair_tile) pair_tile[pos] = tk[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        if (tk[i] == pad) continue;
        const uint16_t next = i + 1 < ITEMS ? tk[i + 1]
                              : (base + ITEMS < W ? skey[base + ITEMS] : pad);
        if (next != tk[i]) cursor[tk[i]] += (uint32_t)(base + i - start[i] + 1);
    }
    __syncthreads();
}


// sum of chunk_tot[0, c): chunk c's first rank-major pair index.  Block-wide
// (every thread of the THREADS-CTA calls it and gets the result).
template <int THREADS = kBinThreads>
__device__ __forceinline__ uint32_t chunk_pair_base(int c, const uint32_t *__restrict__ chunk_tot)
{
    __shared__ uint32_t s_part[THREADS / 32];
    uint32_t v = 0;
    for (int k = threadIdx.x; k < c; k += THREADS) v += __ldg(chunk_tot + k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
    __syncthreads();
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) t += s_part[w];
    __syncthreads();
    return t;
}

// One CTA per chunk of CH = THREADS x RPT ranks (256 x 4 for maps above
// kSmallMapRows, 256 x 1 below).
template <int THREADS, int RPT>
__global__ void __launch_bounds__(THREADS, THREADS >= 1024 ? 1 : 3) place_kernel(
    int64_t m, const uint32_t *__restrict__ order, const uint32_t *__restrict__ counts,
    const uint64_t *__restrict__ masks, const uint32_t *__restrict__ geo,
    const uint16_t *__restrict__ big, const uint32_t *__restrict__ hoff, int tiles_x, int n_tiles,
    int n_chunks, int key_bits, const int32_t *__restrict__ offsets,
    int32_t *__restrict__ pair_gaussian, int32_t *__restrict__ pair_tile,
    const uint32_t *__restrict__ chunk_tot, uint8_t *__restrict__ pvalid,
    uint32_t *__restrict__ rank_e0)
{
    using RowScan = cub::BlockScan<uint32_t, THREADS>;
    using RunScan = cub::BlockScan<int, THREADS>;
    constexpr int CH = THREADS * RPT;              // ranks per chunk
    constexpr int kItems = 2048 / THREADS;         // pairs per thread per window (full lists: 240 -> 223 us vs 4096-pair windows)
    constexpr int kSmall = kItems >= 4 ? kItems / 4 : 1;   // the last, short window
    constexpr int W = THREADS * kItems;            // pairs per window
    __shared__ union {
        typename PlaceSort<THREADS, kItems>::Sort::TempStorage sort;
        typename PlaceSort<THREADS, kSmall>::Sort::TempStorage sort_small;
        uint16_t key[W];
    } u;
    __shared__ union {
        typename RowScan::TempStorage rows;
        typename RunScan::TempStorage runs;
    } sc;
    __shared__ uint32_t lo_s[CH + 1];        // chunk-local pair offset of each rank
    // dynamic: the chunk's rows staged (mask, row, geometry per rank: the
    // pair walk's per-row reads hit shared memory), then the next slot of
    // every tile
    extern __shared__ uint64_t dyn_smem[];
    uint64_t *s_mask = dyn_smem;
    uint32_t *s_row = reinterpret_cast<uint32_t *>(s_mask + CH);
    uint32_t *s_geo = s_row + CH;
    uint32_t *cursor = s_geo + CH;

    // a capacity overflow empties every range (tile_offsets_kernel): nothing
    // is placed
    if (offsets[n_tiles] == 0) return;
    const int c = blockIdx.x;
    if (__ldg(chunk_tot + c) == 0) return;   // no kept pair in the chunk
    const int64_t r0 = (int64_t)c * CH;
    {
        uint32_t cnt[RPT], lo[RPT];
        const int64_t rb = r0 + (int64_t)threadIdx.x * RPT;
#pragma unroll
        for (int i = 0; i < RPT; ++i) cnt[i] = rb + i < m ? counts[rb + i] : 0u;
        uint32_t tot;
        RowScan(sc.rows).ExclusiveSum(cnt, lo, tot);
#pragma unroll
        for (int i = 0; i < RPT; ++i) lo_s[threadIdx.x * RPT + i] = lo[i];
        if (threadIdx.x == 0) lo_s[CH] = tot;
    }
    __syncthreads();
    const uint32_t total = lo_s[CH];
    if (total == 0) return;   // every row of the chunk dropped (depth limits) or empty
    // this chunk's first rank-major pair index; each rank's first index and
    // the chunk's cleared replayed flags for the deterministic backward
    const uint32_t cb = chunk_pair_base<THREADS>(c, chunk_tot);
    {
        // the rows with kept pairs, staged: every load issued before the
        // shared-memory stores (the staging is on the chunk's critical path)
        constexpr int kQ = (CH + THREADS - 1) / THREADS;
        uint32_t vr[kQ], vg[kQ];
        uint64_t vm[kQ];
        bool need[kQ];
#pragma unroll
        for (int k = 0; k < kQ; ++k) {
            const int q = threadIdx.x + k * THREADS;
            need[k] = q < CH && r0 + q < m && lo_s[q + 1] != lo_s[q];
            if (need[k]) {
                vr[k] = __ldg(order + r0 + q);
                vg[k] = __ldg(geo + r0 + q);
                vm[k] = __ldg(masks + r0 + q);
            }
        }
#pragma unroll
        for (int k = 0; k < kQ; ++k) {
            const int q = threadIdx.x + k * THREADS;
            if (q < CH && r0 + q < m) rank_e0[r0 + q] = cb + lo_s[q];
            if (need[k]) {
                s_row[q] = vr[k];
                s_geo[q] = vg[k];
                s_mask[q] = vm[k];
            }
        }
    }
    for (uint32_t i = threadIdx.x; i < total; i += THREADS) pvalid[cb + i] = 0;
    // a pair's slot: the scanned histogram entry (the tile's CSR offset +
    // its pairs in earlier chunks) + its rank in this chunk (8 loads in
    // flight per thread: the strided histogram reads are L2 round trips)
    for (int t0 = threadIdx.x; t0 < n_tiles; t0 += 8 * THREADS) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int t = t0 + k * THREADS;
            v[k] = t < n_tiles ? __ldg(hoff + (int64_t)t * n_chunks + c) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int t = t0 + k * THREADS;
            if (t < n_tiles) cursor[t] = v[k];
        }
    }
    __syncthreads();

    for (uint32_t w0 = 0; w0 < total;) {
        if (total - w0 <= (uint32_t)(THREADS * kSmall)) {
            place_window<THREADS, kSmall, CH>(w0, total, lo_s, s_row, s_mask, s_geo, big,
                                              tiles_x, key_bits, cursor, u.sort_small, u.key,
                                              sc.runs, pair_gaussian, pair_tile);
            w0 += THREADS * kSmall;
        } else {
            place_window<THREADS, kItems, CH>(w0, total, lo_s, s_row, s_mask, s_geo, big,
                                              tiles_x, key_bits, cursor, u.sort, u.key, sc.runs,
                                              pair_gaussian, pair_tile);
            w0 += W;
        }
    }
}

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct BinLayout {
    size_t keys_sorted, order, counts, masks, geo, big, big_total, hist, temp, temp_bytes, bytes;
    size_t pvalid;                  // per rank-major pair index: replayed [cap]
    size_t chunk_tot;               // per chunk: pair total
    size_t rank_e0, rank_hit;       // per rank: first rank-major pair index, replayed flag
    size_t rank_of;                 // per map row: its depth rank
    size_t keys_c, vals_c, n_sel;   // bounded sort: compacted keys / rows, selected count
    int n_chunks, n_tiles;
    int chunk;                      // rows per chunk: 1024, or 256 for small maps
    int64_t big_cap;
};

// Bounded sort (sb_bin's sort_capacity): the rows with a valid depth key, in
// row order (CUB's select is stable), are gathered into sort_capacity slots
// and only those are sorted; the slots past the selected count hold invalid
// keys and kNoRow.  The stable depth order of the selected rows is exactly
// the full sort's order of its valid prefix (invalid keys sort last there).
template <typename K>
__global__ void key_flags_kernel(int64_t m, const K *__restrict__ keys, uint8_t *__restrict__ flags)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) flags[i] = keys[i] != ~(K)0;
}

// Pads the compacted keys / rows past the selected count up to the bound;
// more selected rows than the bound sets *sort_over (tile_offsets_kernel
// turns it into an empty, invalid step).
template <typename K>
__global__ void pad_bounded_kernel(int64_t cap, const int *__restrict__ n_sel,
                                   K *__restrict__ keys_c, uint32_t *__restrict__ vals_c,
                                   int *__restrict__ sort_over)
{
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n = *n_sel;
    if (j == 0) *sort_over = n > cap;
    if (j >= cap || j < n) return;
    keys_c[j] = ~(K)0;
    vals_c[j] = kNoRow;
}

static BinLayout bin_layout_compute(int64_t m, int64_t cap, int32_t width, int32_t height);

// The layout is a pure function of (m, cap, width, height), but computing it
// asks CUB for its temporary-storage sizes (device-attribute queries: tens of
// microseconds of host time).  The host path of an sb_bin call (and of the
// backward's merge, which views the same workspace) would pay that on every
// eager launch, e.g. every frame of the render path; a small memo keeps it
// to the first call per shape.
static BinLayout bin_layout(int64_t m, int64_t cap, int32_t width, int32_t height)
{
    struct Entry {
        int64_t m, cap;
        int32_t w, h;
        BinLayout L;
    };
    static std::mutex mu;
    static Entry memo[16];
    static int n_memo = 0, next = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        for (int i = 0; i < n_memo; ++i)
            if (memo[i].m == m && memo[i].cap == cap && memo[i].w == width && memo[i].h == height)
                return memo[i].L;
    }
    const BinLayout L = bin_layout_compute(m, cap, width, height);
    std::lock_guard<std::mutex> lock(mu);
    memo[next] = Entry{m, cap, width, height, L};
    next = (next + 1) % 16;
    n_memo = n_memo < 16 ? n_memo + 1 : 16;
    return L;
}

static BinLayout bin_layout_compute(int64_t m, int64_t cap, int32_t width, int32_t height)
{
    BinLayout L;
    size_t o = 0;
    const int64_t mm = m > 0 ? m : 1;
    L.n_tiles = ((width + kTile - 1) / kTile) * ((height + kTile - 1) / kTile);
    // small maps get 256-row chunks: 10-100 chunks of 1024 rows would leave
    // most of the 148 SMs idle in the count and placement passes
    L.chunk = mm <= kSmallMapRows ? kSmallChunk : kChunkRows;
    L.n_chunks = (int)((mm + L.chunk - 1) / L.chunk);
    L.big_cap = cap > 0 ? cap : 1;
    const int64_t nh = (int64_t)L.n_tiles * L.n_chunks + 1;
    L.keys_sorted = o; o += align256(8 * mm);
    L.order = o; o += align256(4 * mm);
    L.counts = o; o += align256(4 * mm);
    L.masks = o; o += align256(8 * mm);
    L.geo = o; o += align256(4 * mm);
    L.big = o; o += align256(2 * L.big_cap);
    L.big_total = o; o += 256;
    L.hist = o; o += align256(4 * nh);
    L.keys_c = o; o += align256(8 * mm);
    L.vals_c = o; o += align256(4 * mm);
    L.n_sel = o; o += 256;
    L.pvalid = o; o += align256(L.big_cap);
    L.chunk_tot = o; o += align256(4 * (size_t)L.n_chunks);
    L.rank_e0 = o; o += align256(4 * mm);
    L.rank_hit = o; o += align256(mm);
    L.rank_of = o; o += align256(4 * mm);
    size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)mm);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)mm);
    cub::DeviceScan::ExclusiveSum(nullptr, t3, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (int)nh);
    size_t t5 = 0;
    cub::DeviceSelect::Flagged(nullptr, t4, (const uint32_t *)nullptr, (const uint8_t *)nullptr,
                               (uint32_t *)nullptr, (int *)nullptr, (int)mm);
    cub::DeviceSelect::Flagged(nullptr, t5, (const unsigned long long *)nullptr,
                               (const uint8_t *)nullptr, (unsigned long long *)nullptr,
                               (int *)nullptr, (int)mm);
    t4 = std::max(t4, t5);
    L.temp_bytes = std::max(std::max(t1, t2), std::max(t3, t4));
    L.temp = o; o += align256(L.temp_bytes);
    L.bytes = o;
    return L;
}

// The same workspace viewed for fewer sorted ranks (a bounded sort): fewer
// chunks, so a smaller tile histogram inside the same allocation.
static BinLayout bin_layout_ranks(const BinLayout &L, int64_t ms)
{
    BinLayout R = L;
    R.n_chunks = (int)((ms + R.chunk - 1) / R.chunk);
    return R;
}

// place_kernel's dynamic shared memory: the staged rows (16 B each) and a
// cursor per tile
static inline size_t place_smem(int n_tiles, int chunk)
{
    return (size_t)16 * chunk + sizeof(uint32_t) * (size_t)n_tiles;
}

// Opt the histogram/place kernels in to the dynamic shared memory of the
// largest supported tile grid (static + dynamic above 48 KB needs the
// attribute); the launch size, not this limit, sets the occupancy.  Done once
// per process, before any graph capture can see it.
static int32_t opt_in_smem()
{
    static bool done = false;
    if (!done) {
        const int bytes = (int)sizeof(uint32_t) * kMaxTiles;
        const int cbytes = bytes + (int)sizeof(uint32_t) * kMaxCoarse;
        SB_CUDA(cudaFuncSetAttribute(count_hist_kernel<float, kCountWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize, cbytes));
        SB_CUDA(cudaFuncSetAttribute(count_hist_kernel<double, kCountWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize, cbytes));
        SB_CUDA(cudaFuncSetAttribute(count_hist_kernel<float, kSmallChunk / 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, cbytes));
        SB_CUDA(cudaFuncSetAttribute(count_hist_kernel<double, kSmallChunk / 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, cbytes));
            SB_CUDA(cudaFuncSetAttribute(place_kernel<kBinThreads, kRowsPerThread>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)place_smem(kMaxTiles, kChunkRows)));
        SB_CUDA(cudaFuncSetAttribute(place_kernel<kSmallChunk, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)place_smem(kMaxTiles, kSmallChunk)));
        done = true;
    }
    return SB_OK;
}

template <typename T>
static int32_t bin_passes(int64_t m, const T *records, const uint8_t *valid, const uint32_t *order,
                          const TileGeom &g, int cull, const BinLayout &L, char *ws,
                          int64_t cap, int32_t *pair_gaussian, int32_t *pair_tile,
                          int32_t *offsets, int64_t *d_status, const float *dlim,
                          int64_t *n_pairs, const int *sort_over, const int64_t *halt,
                          cudaStream_t st)
{
    uint32_t *counts = (uint32_t *)(ws + L.counts);
    uint64_t *masks = (uint64_t *)(ws + L.masks);
    uint32_t *geo = (uint32_t *)(ws + L.geo);
    uint16_t *big = (uint16_t *)(ws + L.big);
    unsigned long long *big_total = (unsigned long long *)(ws + L.big_total);
    uint32_t *hist = (uint32_t *)(ws + L.hist);
    uint32_t *chunk_tot = (uint32_t *)(ws + L.chunk_tot);
    uint8_t *pvalid = (uint8_t *)(ws + L.pvalid);
    const int64_t nh = (int64_t)L.n_tiles * L.n_chunks + 1;
    const size_t dyn = sizeof(uint32_t) * L.n_tiles;
    const int32_t rc = opt_in_smem();
    if (rc != SB_OK) return rc;

    SB_CUDA(cudaMemsetAsync(big_total, 0, sizeof(unsigned long long), st));
    SB_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * nh, st));
    SB_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * m, st));
    const int cells = ((g.tiles_x + 3) >> 2) * ((g.tiles_y + 3) >> 2);
    const int coarse = dlim && cells <= kMaxCoarse ? cells : 0;
    if (L.chunk == kChunkRows)
        count_hist_kernel<T, kCountWarps><<<L.n_chunks, kCountThreads, dyn + sizeof(uint32_t) * coarse, st>>>(
            m, records, valid, order, g, cull, L.n_chunks, counts, masks, geo, big, L.big_cap,
            big_total, hist, dlim, coarse, ws + L.keys_sorted, chunk_tot,
            (uint32_t *)(ws + L.rank_of), (uint8_t *)(ws + L.rank_hit));
    else
        count_hist_kernel<T, kSmallChunk / 32><<<L.n_chunks, kSmallChunk, dyn + sizeof(uint32_t) * coarse, st>>>(
            m, records, valid, order, g, cull, L.n_chunks, counts, masks, geo, big, L.big_cap,
            big_total, hist, dlim, coarse, ws + L.keys_sorted, chunk_tot,
            (uint32_t *)(ws + L.rank_of), (uint8_t *)(ws + L.rank_hit));
    SB_CUDA(cudaGetLastError());
    SB_CUDA(cudaMemsetAsync(hist + nh - 1, 0, sizeof(uint32_t), st));
    size_t tb = L.temp_bytes;
    SB_CUDA(cub::DeviceScan::ExclusiveSum(ws + L.temp, tb, hist, hist, (int)nh, st));
    tile_offsets_kernel<<<1, 1024, 0, st>>>(hist, L.n_chunks, L.n_tiles, cap, offsets, d_status,
                                            sort_over, halt);
    SB_CUDA(cudaGetLastError());
    if (d_status == nullptr) {
        uint32_t total = 0;
        SB_CUDA(cudaMemcpyAsync(&total, hist + nh - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        SB_CUDA(cudaStreamSynchronize(st));
        *n_pairs = total;
        SB_REQUIRE(total < 0x7FFFFFFFu, "pair count overflow");
        if ((int64_t)total > cap) {
            set_error("pair capacity %lld < %u", (long long)cap, total);
            return SB_ERR_CAPACITY;
        }
        if (total == 0) return SB_OK;
    } else {
        *n_pairs = -1;
    }
    int bits = 1;
    while ((1 << bits) <= L.n_tiles) ++bits;   // pad key (2^bits - 1) >= n_tiles
#define PLACE_ARGS                                                                             \
    m, order, counts, masks, geo, big, hist, g.tiles_x, L.n_tiles, L.n_chunks, bits, offsets,  \
        pair_gaussian, pair_tile, chunk_tot, pvalid, (uint32_t *)(ws + L.rank_e0)
    const size_t psm = place_smem(L.n_tiles, L.chunk);
    if (L.chunk == kChunkRows) {
        // 256-thread CTAs (4 ranks per thread): measured against 1024-thread
        // CTAs for the heavy chunks only (two launches split by chunk_tot)
        // and for all chunks -- config 3: 851 / 849 / 854 it/s, its full
        // lists 682 / 653 / 655, the config-4 stream 284 / 278 / 284
        place_kernel<kBinThreads, kRowsPerThread><<<L.n_chunks, kBinThreads, psm, st>>>(
            PLACE_ARGS);
    } else {
        place_kernel<kSmallChunk, 1><<<L.n_chunks, kSmallChunk, psm, st>>>(PLACE_ARGS);
    }
#undef PLACE_ARGS
    return check_launch("place_kernel");
}

// The deterministic backward's reduction (sb_blend_bwd_det, blend_bwd.cu):
// the backward blend stored one partial adjoint record (kPartialReals reals)
// per replayed (tile, row) pair at the pair's rank-major index e and set
// pvalid[e], so each rank's pairs are contiguous, in ascending tile order.
// One CTA per chunk of depth ranks, one rank per thread: a rank with at most
// kGatherSerial kept pairs adds its replayed records in order -- the
// reference's merge order (backward.py:92-98); the rare long ranks (large
// splats over many tiles, e.g. the sky shell, clustered in depth) are queued
// for a persistent grid of warps that load 128 records at a time and add
// them in the same sequential order.  So every row's
// adjoints are the sum, from zero, of its replayed (tile, row) records in
// ascending tile order: independent of scheduling, of the serial/queued
// split and of how many unreplayed pairs the lists hold (depth-limited vs
// full lists) -- no float atomics, bitwise reproducible.  Rows with no kept
// pair are not touched (the caller zeroes the adjoint buffers).
constexpr uint32_t kGatherSerial = (uint32_t)kGatherQueueDiv;

__device__ __forceinline__ void load_partial(const float *__restrict__ p, float a[9])
{
    const float4 *q = reinterpret_cast<const float4 *>(p);
    const float4 x = __ldg(q), y = __ldg(q + 1), z = __ldg(q + 2);
    a[0] = x.x; a[1] = x.y; a[2] = x.z; a[3] = x.w;
    a[4] = y.x; a[5] = y.y; a[6] = y.z; a[7] = y.w; a[8] = z.x;
}

__device__ __forceinline__ void load_partial(const double *__restrict__ p, double a[9])
{
    const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double2 v = __ldg(q + k);
        a[2 * k] = v.x;
        a[2 * k + 1] = v.y;
    }
    a[8] = __ldg(p + 8);
}

template <typename T>
__device__ __forceinline__ void store_adjoints(uint32_t row, const T a[9], T *__restrict__ d_mean,
                                               T *__restrict__ d_conic, T *__restrict__ d_op,
                                               T *__restrict__ d_col)
{
    d_mean[2 * (int64_t)row] = a[0];
    d_mean[2 * (int64_t)row + 1] = a[1];
    d_conic[3 * (int64_t)row] = a[2];
    d_conic[3 * (int64_t)row + 1] = a[3];
    d_conic[3 * (int64_t)row + 2] = a[4];
    d_op[row] = a[5];
    d_col[3 * (int64_t)row] = a[6];
    d_col[3 * (int64_t)row + 1] = a[7];
    d_col[3 * (int64_t)row + 2] = a[8];
}

// A merged row is reached when its adjoints are not all zero: its flag byte
// (nullable) names it for the chain rule, which then reads no other row's
// adjoints.
template <typename T>
__device__ __forceinline__ void reach_mark(uint8_t *__restrict__ row_flag, uint32_t row,
                                           const T a[9])
{
    if (!row_flag) return;
    bool nz = false;
#pragma unroll
    for (int v = 0; v < 9; ++v) nz |= a[v] != (T)0;
    if (nz) row_flag[row] = 1;
}

// one rank per thread
template <typename T>
__global__ void __launch_bounds__(kBinThreads) gather_short_kernel(
    int64_t m, const uint32_t *__restrict__ order, const uint32_t *__restrict__ counts,
    const uint32_t *__restrict__ rank_e0, const uint8_t *__restrict__ pvalid,
    const T *__restrict__ partial, T *__restrict__ d_mean, T *__restrict__ d_conic,
    T *__restrict__ d_op, T *__restrict__ d_col, uint4 *__restrict__ queue,
    uint32_t *__restrict__ queue_n, const uint32_t *__restrict__ chunk_tot, int chunk,
    const uint8_t *__restrict__ rank_hit, uint8_t *__restrict__ row_flag)
{
    const int64_t r0 = (int64_t)blockIdx.x * kBinThreads, r = r0 + threadIdx.x;
    // the binning chunk of these ranks had no kept pair (the invalid rows
    // sorted behind the valid ones): one load for the whole CTA
    if (__ldg(chunk_tot + r0 / chunk) == 0) return;
    if (r >= m || !__ldg(rank_hit + r)) return;   // no replayed pair: not reached
    const uint32_t cnt = __ldg(counts + r);
    const uint32_t row = __ldg(order + r), e0 = __ldg(rank_e0 + r);
    // long ranks -> the global queue (warp-aggregated append; the queue
    // order does not affect any sum)
    const bool is_long = cnt > kGatherSerial;
    const unsigned am = __activemask();
    const unsigned lm = __ballot_sync(am, is_long);
    if (is_long) {
        const int lane = threadIdx.x & 31, leader = __ffs(lm) - 1;
        uint32_t qb = 0;
        if (lane == leader) qb = atomicAdd(queue_n, (uint32_t)__popc(lm));
        qb = __shfl_sync(lm, qb, leader);
        queue[qb + __popc(lm & ((1u << lane) - 1u))] = make_uint4(row, e0, cnt, 0u);
        return;
    }
    T a[9];
#pragma unroll
    for (int v = 0; v < 9; ++v) a[v] = (T)0;
    // batches of 8 flags, then their records 4 at a time (loads in flight),
    // added in pair order
    for (uint32_t j0 = 0; j0 < cnt; j0 += 8) {
        bool ok[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) ok[u] = j0 + u < cnt && __ldg(pvalid + e0 + j0 + u);
#pragma unroll
        for (int h = 0; h < 8; h += 4) {
            T p[4][9];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (ok[h + u]) load_partial(partial + (int64_t)(e0 + j0 + h + u) * kPartialReals, p[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (!ok[h + u]) continue;
#pragma unroll
                for (int v = 0; v < 9; ++v) a[v] += p[u][v];
            }
        }
    }
    store_adjoints(row, a, d_mean, d_conic, d_op, d_col);
    reach_mark(row_flag, row, a);
}

// Long ranks: one warp per queued rank.  The warp loads 32 x kLongDepth
// records at a time (the next group's loads issued before this group is
// summed), transposes each batch of 32 through shared memory, and lanes 0-8
// add value v of the records strictly in pair order -- the same sequential
// sum as the short path.  Unreplayed pairs and the tail past the count
// contribute +0, a bitwise no-op: a running sum that starts at +0 is never
// -0.  (The previous half-warp form paid a dependent flag -> record load per
// 16 records; a row over most of a 1280x720 image took ~240 us alone.)
constexpr int kLongDepth = 4;

template <typename T>
__device__ __forceinline__ void long_group(const uint8_t *__restrict__ pvalid,
                                           const T *__restrict__ partial, uint32_t e0,
                                           uint32_t cnt, uint32_t j0, int lane,
                                           T p[kLongDepth][9], bool ok[kLongDepth])
{
#pragma unroll
    for (int d = 0; d < kLongDepth; ++d) {
        const uint32_t j = j0 + d * 32 + lane;
        const bool in = j < cnt;
        ok[d] = in && __ldg(pvalid + e0 + j);
        if (in) {
            load_partial(partial + (int64_t)(e0 + j) * kPartialReals, p[d]);
        } else {
#pragma unroll
            for (int v = 0; v < 9; ++v) p[d][v] = (T)0;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kBinThreads) gather_long_kernel(
    const uint8_t *__restrict__ pvalid, const T *__restrict__ partial, T *__restrict__ d_mean,
    T *__restrict__ d_conic, T *__restrict__ d_op, T *__restrict__ d_col,
    const uint4 *__restrict__ queue, const uint32_t *__restrict__ queue_n,
    uint8_t *__restrict__ row_flag)
{
    constexpr int kWarps = kBinThreads / 32;
    __shared__ T s[kWarps][9][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t nq = *queue_n;
    const uint32_t nw = gridDim.x * kWarps;
    for (uint32_t k = blockIdx.x * kWarps + w; k < nq; k += nw) {
        const uint4 q = queue[k];                  // row, e0, cnt (warp-uniform)
        T acc = (T)0;                              // lane v < 9: value v's sum
        T p[kLongDepth][9];
        bool ok[kLongDepth];
        long_group(pvalid, partial, q.y, q.z, 0u, lane, p, ok);
        for (uint32_t j0 = 0; j0 < q.z; j0 += 32 * kLongDepth) {
            const uint32_t jn = j0 + 32 * kLongDepth;
            T pn[kLongDepth][9];
            bool okn[kLongDepth];
            if (jn < q.z) long_group(pvalid, partial, q.y, q.z, jn, lane, pn, okn);
#pragma unroll
            for (int d = 0; d < kLongDepth; ++d) {
                __syncwarp();
#pragma unroll
                for (int v = 0; v < 9; ++v) s[w][v][lane] = ok[d] ? p[d][v] : (T)0;
                __syncwarp();
                if (lane < 9) {
#pragma unroll 8
                    for (int i = 0; i < 32; ++i) acc += s[w][lane][i];
                }
            }
            if (jn < q.z) {
#pragma unroll
                for (int d = 0; d < kLongDepth; ++d) {
                    ok[d] = okn[d];
#pragma unroll
                    for (int v = 0; v < 9; ++v) p[d][v] = pn[d][v];
                }
            }
        }
        T a[9];
#pragma unroll
        for (int v = 0; v < 9; ++v) a[v] = __shfl_sync(0xffffffffu, acc, v);
        if (lane == 0) {
            store_adjoints(q.x, a, d_mean, d_conic, d_op, d_col);
            reach_mark(row_flag, q.x, a);
        }
    }
}

// The deterministic backward's maps in an sb_bin workspace (same m, pair
// capacity, image size as the sb_bin call).
BinMaps bin_maps(int64_t m, int64_t pair_capacity, int32_t width, int32_t height,
                 const void *bin_workspace)
{
    const BinLayout L = bin_layout(m, pair_capacity, width, height);
    char *ws = (char *)bin_workspace;
    BinMaps M;
    M.rank_of = (const uint32_t *)(ws + L.rank_of);
    M.geo = (const uint32_t *)(ws + L.geo);
    M.counts = (const uint32_t *)(ws + L.counts);
    M.rank_e0 = (const uint32_t *)(ws + L.rank_e0);
    M.masks = (const uint64_t *)(ws + L.masks);
    M.big = (const uint16_t *)(ws + L.big);
    M.pvalid = (uint8_t *)(ws + L.pvalid);
    M.rank_hit = (uint8_t *)(ws + L.rank_hit);
    return M;
}

// Host side of the gather over the workspace of the sb_bin call that made
// the pairs (same m, pair capacity, image size and sort capacity).  queue
// holds at least pair_capacity / kGatherSerial + 1 entries (16 B); queue_n
// is one uint32 (zeroed here).
int32_t launch_gather_adjoints(int32_t dtype, int64_t m, int64_t pair_capacity, int32_t width,
                               int32_t height, int64_t sort_capacity, const void *bin_workspace,
                               const void *partial, void *d_mean, void *d_conic, void *d_op,
                               void *d_col, void *queue, uint32_t *queue_n,
                               uint8_t *reached_rows, cudaStream_t st)
{
    if (m == 0) return SB_OK;
    const BinLayout L = bin_layout(m, pair_capacity, width, height);
    const int64_t ms = sort_capacity > 0 && sort_capacity < m ? sort_capacity : m;
    const char *ws = (const char *)bin_workspace;
    SB_CUDA(cudaMemsetAsync(queue_n, 0, sizeof(uint32_t), st));
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
#define GATHER_SHORT(T)                                                                        \
    gather_short_kernel<T><<<grid_for(ms, kBinThreads), kBinThreads, 0, st>>>(                 \
        ms, (const uint32_t *)(ws + L.order), (const uint32_t *)(ws + L.counts),                \
        (const uint32_t *)(ws + L.rank_e0), (const uint8_t *)(ws + L.pvalid),                  \
        (const T *)partial, (T *)d_mean, (T *)d_conic, (T *)d_op, (T *)d_col, (uint4 *)queue,  \
        queue_n, (const uint32_t *)(ws + L.chunk_tot), L.chunk,                                \
        (const uint8_t *)(ws + L.rank_hit), reached_rows)
#define GATHER_LONG(T)                                                                         \
    gather_long_kernel<T><<<8 * sms, kBinThreads, 0, st>>>(                                    \
        (const uint8_t *)(ws + L.pvalid), (const T *)partial, (T *)d_mean, (T *)d_conic,       \
        (T *)d_op, (T *)d_col, (const uint4 *)queue, queue_n, reached_rows)
    if (dtype == SB_F32) GATHER_SHORT(float);
    else GATHER_SHORT(double);
    SB_CUDA(cudaGetLastError());
    if (dtype == SB_F32) GATHER_LONG(float);
    else GATHER_LONG(double);
#undef GATHER_SHORT
#undef GATHER_LONG
    return check_launch("gather_long_kernel");
}

}  // namespace sb

using namespace sb;

extern "C" size_t sb_bin_workspace_bytes(int64_t m, int64_t pair_capacity, int32_t width,
                                         int32_t height)
{
    return bin_layout(m, pair_capacity, width, height).bytes;
}

extern "C" int32_t sb_bin(int32_t dtype, int64_t m, const void *records, const uint8_t *valid,
                          void *depth_key, uint32_t *depth_val, int32_t width, int32_t height,
                          int32_t tile_size, int32_t cull, int64_t pair_capacity,
                          int32_t *pair_gaussian, int32_t *pair_tile, int32_t *offsets,
                          int64_t *n_pairs, void *workspace, size_t workspace_bytes,
                          int64_t *d_status, const float *tile_depth_limit,
                          int64_t sort_capacity, const int64_t *halt, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(tile_size == kTile, "tile_size %d unsupported (only %d)", tile_size, kTile);
    SB_REQUIRE(width > 0 && height > 0, "bad image size %dx%d", width, height);
    SB_REQUIRE(m >= 0 && m < 0x7FFFFFFF, "bad row count");
    SB_REQUIRE(n_pairs != nullptr, "n_pairs is NULL");
    const BinLayout L = bin_layout(m, pair_capacity, width, height);
    SB_REQUIRE(L.n_tiles <= kMaxTiles, "%d tiles > %d supported", L.n_tiles, kMaxTiles);
    SB_REQUIRE((int64_t)L.n_tiles * L.n_chunks < 0x7FFFFFFF, "tile histogram too large");
    SB_REQUIRE(workspace_bytes >= L.bytes, "workspace too small: %zu < %zu", workspace_bytes, L.bytes);
    SB_REQUIRE(tile_depth_limit == nullptr || d_status != nullptr,
               "tile depth limits need the device status");
    cudaStream_t st = as_stream(stream);
    TileGeom g{width, height, (width + kTile - 1) / kTile, (height + kTile - 1) / kTile};
    char *ws = (char *)workspace;
    uint32_t *order = (uint32_t *)(ws + L.order);
    size_t temp_bytes = L.temp_bytes;

    if (m == 0) {
        SB_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (L.n_tiles + 1), st));
        if (d_status) SB_CUDA(cudaMemsetAsync(d_status, 0, 2 * sizeof(int64_t), st));
        if (d_status && halt)
            SB_CUDA(cudaMemcpyAsync(d_status + 1, halt, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
        *n_pairs = d_status ? -1 : 0;
        return SB_OK;
    }
    // 1. stable depth sort of the rows (forward.py:248-249); invalid rows last
    const int *sort_over = nullptr;
    const void *skeys = depth_key;
    const uint32_t *svals = depth_val;
    int64_t ms = m;
    if (sort_capacity > 0 && sort_capacity < m) {
        // bounded: sort only the rows with a valid key (those can have pairs)
        SB_REQUIRE(d_status != nullptr, "a bounded sort needs the device status");
        int *n_sel = (int *)(ws + L.n_sel);
        sort_over = n_sel + 1;
        const unsigned gg = (unsigned)((sort_capacity + 255) / 256);
        const unsigned gm = (unsigned)((m + 255) / 256);
        uint8_t *flags = (uint8_t *)(ws + L.counts);   // scratch until count_hist writes counts
        // the keys and the rows with a valid key, each compacted in order
        // (CUB's select is stable, so the two stay paired)
        if (dtype == SB_F32) {
            key_flags_kernel<uint32_t><<<gm, 256, 0, st>>>(m, (const uint32_t *)depth_key, flags);
            SB_CUDA(cub::DeviceSelect::Flagged(ws + L.temp, temp_bytes, (const uint32_t *)depth_key,
                                               flags, (uint32_t *)(ws + L.keys_c), n_sel, (int)m, st));
        } else {
            key_flags_kernel<unsigned long long><<<gm, 256, 0, st>>>(
                m, (const unsigned long long *)depth_key, flags);
            SB_CUDA(cub::DeviceSelect::Flagged(ws + L.temp, temp_bytes,
                                               (const unsigned long long *)depth_key, flags,
                                               (unsigned long long *)(ws + L.keys_c), n_sel,
                                               (int)m, st));
        }
        temp_bytes = L.temp_bytes;
        SB_CUDA(cub::DeviceSelect::Flagged(ws + L.temp, temp_bytes, depth_val, flags,
                                           (uint32_t *)(ws + L.vals_c), n_sel, (int)m, st));
        if (dtype == SB_F32)
            pad_bounded_kernel<uint32_t><<<gg, 256, 0, st>>>(
                sort_capacity, n_sel, (uint32_t *)(ws + L.keys_c), (uint32_t *)(ws + L.vals_c),
                n_sel + 1);
        else
            pad_bounded_kernel<unsigned long long><<<gg, 256, 0, st>>>(
                sort_capacity, n_sel, (unsigned long long *)(ws + L.keys_c),
                (uint32_t *)(ws + L.vals_c), n_sel + 1);
        SB_CUDA(cudaGetLastError());
        skeys = ws + L.keys_c;
        svals = (const uint32_t *)(ws + L.vals_c);
        ms = sort_capacity;
        temp_bytes = L.temp_bytes;
    }
    if (dtype == SB_F32)
        SB_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.temp, temp_bytes, (const uint32_t *)skeys,
                                                (uint32_t *)(ws + L.keys_sorted), svals, order,
                                                (int)ms, 0, 32, st));
    else
        SB_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.temp, temp_bytes, (const uint64_t *)skeys,
                                                (uint64_t *)(ws + L.keys_sorted), svals, order,
                                                (int)ms, 0, 64, st));
    // 2-4. count + tile histogram, scan, place (over the sorted ranks)
    const BinLayout Ls = ms == m ? L : bin_layout_ranks(L, ms);
    if (dtype == SB_F32)
        return bin_passes<float>(ms, (const float *)records, valid, order, g, cull, Ls, ws,
                                 pair_capacity, pair_gaussian, pair_tile, offsets, d_status,
                                 tile_depth_limit, n_pairs, sort_over, halt, st);
    return bin_passes<double>(ms, (const double *)records, valid, order, g, cull, Ls, ws,
                              pair_capacity, pair_gaussian, pair_tile, offsets, d_status,
                              tile_depth_limit, n_pairs, sort_over, halt, st);
}
