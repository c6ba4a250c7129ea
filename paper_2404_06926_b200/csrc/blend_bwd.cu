// blend_bwd.cu -- K8 backward blend (a6 _backward_tiles, backward.py:91-213).
//
// One CTA per 16x16 tile; PPT pixels per thread set its width: 1 -> 256
// threads, eight warps of 8x4 pixels (393 us at config 3), 2 -> 128
// threads that each own two pixels of a column of an 8x8 warp block (400
// us; but 6 % more it/s in the full-list config-4 stream), 4 -> 64 threads
// (640 us: a tile's serial replay per warp gets too long).  The step picks 1
// or 2 on the device from its replay total (kBwdHeavyPerTile).  The tile is
// replayed front to back only up to the forward's recorded last contributor
// (P_proc in SURVEY §8), each warp only to its own pixels' bound.  Per
// Gaussian, a thread adds its pixels' 9 screen-space adjoints, the warp
// reduces them with a 12-shuffle transpose-reduce into a per-warp shared slot
// (plain stores -- shared-memory float atomics compile to CAS loops), the
// warps' slots are summed once per batch.  Then either (sb_blend_bwd) one
// global float atomic per (tile, Gaussian, value) -- fast, but the summation
// order over tiles varies run to run -- or (sb_blend_bwd_det, the engine's
// path) the 9 sums are stored as the pair's partial record at its
// rank-major index e = rank_e0[rank] + (the tile's index among the row's kept
// tiles) -- sb_bin's maps, BinMaps in common.cuh; a row's pairs are
// contiguous there, tiles ascending -- and the pair and its rank are flagged
// replayed; launch_gather_adjoints (binning.cu) then adds every row's records
// in ascending tile order: the reference's merge order (backward.py:92-98),
// bitwise reproducible.
//
// The outputs are gradients, checked against the oracle within a tolerance,
// so this file is compiled with FMA contraction and recomputes alpha with the
// hardware exp and reciprocal; the forward's exact arithmetic fixes the
// rendered image and the replay bound.
#include "blend_common.cuh"

namespace sb {

constexpr int kBatch = 128;             // records per shared-memory batch (float)
// Gaussians per replay-loop trip: 3 at one pixel per thread (391.7 vs 398
// us for 2, 436 for 4 at config 3), 2 at two pixels per thread (the
// config-4 stream: 288 vs 281 it/s)
template <int PPT>
constexpr int kUnroll = PPT == 1 ? 3 : 2;

// The backward's exp: a 2-ulp hardware exp (ex2.approx) in float.  The
// backward's alphas feed gradients compared within a tolerance, and its
// replay is bounded by the forward's recorded last contributor, so it does
// not need the forward's correctly rounded exp (which is ~40 issue slots).
__device__ __forceinline__ float bwd_exp(float x) { return __expf(x); }
__device__ __forceinline__ double bwd_exp(double x) { return exp(x); }

// approximate reciprocal (1 ulp): only gradients depend on it
__device__ __forceinline__ float rrcp(float x) { return __fdividef(1.0f, x); }
__device__ __forceinline__ double rrcp(double x) { return 1.0 / x; }

// Reduce 9 per-lane values across the warp with 12 shuffles instead of 45:
// at each butterfly level a lane keeps half of its values and receives the
// partner's copy of that half (a transpose-reduce).  Afterwards lane l holds
// the full sum of value reduce9_slot(l) (-1: odd lanes and padding slots).
__device__ __forceinline__ int reduce9_slot(int lane)
{
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    int local;
    if (b3) local = b2 ? -1 : 3 + (int)b1;
    else local = (2 * (int)b2 + (int)b1) <= 2 ? 2 * (int)b2 + (int)b1 : -1;
    if (lane & 1) return -1;
    if (b4) return (local >= 0 && local <= 3) ? 5 + local : -1;
    return (local >= 0 && local <= 4) ? local : -1;
}

template <typename T>
__device__ __forceinline__ T warp_reduce9(const T g[9])
{
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    const T z = (T)0;
    T a[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const T lo = g[i], hi = i < 4 ? g[5 + i] : z;
        a[i] = (b4 ? hi : lo) + __shfl_xor_sync(full, b4 ? lo : hi, 16);
    }
    T b[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const T lo = a[i], hi = i < 2 ? a[3 + i] : z;
        b[i] = (b3 ? hi : lo) + __shfl_xor_sync(full, b3 ? lo : hi, 8);
    }
    T c[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const T lo = b[i], hi = i < 1 ? b[2] : z;
        c[i] = (b2 ? hi : lo) + __shfl_xor_sync(full, b2 ? lo : hi, 4);
    }
    T d = (b1 ? c[1] : c[0]) + __shfl_xor_sync(full, b1 ? c[0] : c[1], 2);
    d += __shfl_xor_sync(full, d, 1);
    return d;
}

// Per-pixel backward state
template <typename T>
struct BwdPix {
    T Tr, P0, P1, P2, dc0, dc1, dc2, cf0, cf1, cf2;
    int end;
    bool done;
};

// One pixel's replay step; adds its adjoints into g[9] when it contributes.
template <typename T>
__device__ __forceinline__ bool bwd_pixel(BwdPix<T> &st, const SmemSplat<T> &s, T fpx, T fpy,
                                          int list_pos, int early, T thresh, T g[9])
{
    const T one = (T)1, half = one / (T)2, two = one + one;
    const T clamp = (T)kAlphaClamp;
    if (st.done || list_pos >= st.end || fpy < s.by0 || fpy > s.by1) return false;
    const T dy = fpy - s.my;
    const T dx = fpx - s.mx;
    T q, gauss, alpha_raw;
    if constexpr (sizeof(T) == 4) {
        // bit for bit the forward's step alpha (blend_common.cuh step_q)
        q = step_q(s, dx, dy);
        if (q > s.qc) return false;
        gauss = step_gauss(q);
        alpha_raw = __fmul_rn(s.opa, gauss);
    } else {
        q = s.a * dx * dx + two * s.b * dy * dx + s.c * dy * dy;
        if (q > s.qc) return false;
        gauss = bwd_exp(-(half * q));
        alpha_raw = s.opa * gauss;
    }
    T alpha = alpha_raw;
    if (alpha > clamp) alpha = clamp;
    if (alpha < (T)kAlphaCutoff) return false;
    const T Tr = st.Tr;
    const T w = sizeof(T) == 4 ? (T)__fmul_rn((float)alpha, (float)Tr) : alpha * Tr;
    const T p0 = st.P0 + w * s.c0;
    const T p1 = st.P1 + w * s.c1;
    const T p2 = st.P2 + w * s.c2;
    g[6] += w * st.dc0;
    g[7] += w * st.dc1;
    g[8] += w * st.dc2;
    if (alpha_raw < clamp) {
        const T inv_rest = rrcp(one - alpha);   // 1 / (1 - alpha) to within 1 ulp (float)
        const T dalpha = (st.dc0 * (s.c0 * Tr - (st.cf0 - p0) * inv_rest)
                          + st.dc1 * (s.c1 * Tr - (st.cf1 - p1) * inv_rest)
                          + st.dc2 * (s.c2 * Tr - (st.cf2 - p2) * inv_rest));
        g[5] += dalpha * gauss;
        const T dq = -(half * gauss * (dalpha * s.opa));
        g[0] += -(two * dq * (s.a * dx + s.b * dy));
        g[1] += -(two * dq * (s.b * dx + s.c * dy));
        g[2] += dq * dx * dx;
        g[3] += dq * dx * dy;
        g[4] += dq * dy * dy;
    }
    st.P0 = p0; st.P1 = p1; st.P2 = p2;
    // the forward's transmittance update, bit for bit
    st.Tr = sizeof(T) == 4 ? (T)__fmul_rn((float)Tr, __fsub_rn(1.0f, (float)alpha))
                           : Tr * (one - alpha);
    if (early && st.Tr < thresh) st.done = true;
    return true;
}

template <typename T>
__device__ __forceinline__ void bwd_init(BwdPix<T> &st, int px, int py, int width, int height,
                                         const T *__restrict__ dC_img,
                                         const T *__restrict__ cfinal,
                                         const int32_t *__restrict__ last_img, int list_len,
                                         int early, T thresh)
{
    st.Tr = (T)1;
    st.P0 = st.P1 = st.P2 = (T)0;
    st.dc0 = st.dc1 = st.dc2 = st.cf0 = st.cf1 = st.cf2 = (T)0;
    st.end = 0;
    if (px < width && py < height) {
        const int64_t pix = (int64_t)py * width + px;
        st.dc0 = dC_img[3 * pix]; st.dc1 = dC_img[3 * pix + 1]; st.dc2 = dC_img[3 * pix + 2];
        st.cf0 = cfinal[3 * pix]; st.cf1 = cfinal[3 * pix + 1]; st.cf2 = cfinal[3 * pix + 2];
        st.end = last_img ? last_img[pix] : list_len;
    }
    st.done = st.end == 0 || (early && (T)1 < thresh);
}

// the pair's partial record (9 sums, padded): three 16-byte stores for float
__device__ __forceinline__ void store_partial(float *__restrict__ p, const float a[9])
{
    float4 *q = reinterpret_cast<float4 *>(p);
    q[0] = make_float4(a[0], a[1], a[2], a[3]);
    q[1] = make_float4(a[4], a[5], a[6], a[7]);
    q[2] = make_float4(a[8], 0.f, 0.f, 0.f);
}

__device__ __forceinline__ void store_partial(double *__restrict__ p, const double a[9])
{
    double2 *q = reinterpret_cast<double2 *>(p);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = make_double2(a[2 * k], a[2 * k + 1]);
    q[4] = make_double2(a[8], 0.0);
    q[5] = make_double2(0.0, 0.0);
}

// DET: partial records at the pairs' rank-major indices + replayed flags
// (BinMaps) instead of float atomics into the adjoint rows.
//
// PPT pixels per thread: 2 -> 4 warps per tile, each owning an 8x8 block
// (pixels at rows y and y + 4 of its column); 4 -> 2 warps per tile, each
// owning a 16x8 half (four consecutive rows of its column).  More pixels
// per thread amortise the per-Gaussian work of a warp (the staged record
// read, the column box test, the vote and the 9-value reduction) over more
// pixels, and fewer warps share a batch barrier.
template <int PPT>
struct BwdShape {
    static constexpr int kThreads = kTilePx / PPT;
    static constexpr int kWarps = kThreads / 32;
};

template <typename T, bool DET, int PPT>
__global__ void __launch_bounds__(BwdShape<PPT>::kThreads) blend_bwd_kernel(
    const T *__restrict__ records, const int32_t *__restrict__ pair_gaussian,
    const int32_t *__restrict__ offsets, int width, int height, int tiles_x, int early,
    T thresh, const T *__restrict__ dC_img, const T *__restrict__ cfinal,
    const int32_t *__restrict__ last_img, T *__restrict__ d_mean, T *__restrict__ d_conic,
    T *__restrict__ d_op, T *__restrict__ d_col, const int32_t *__restrict__ order,
    T *__restrict__ partial, BinMaps maps, const int32_t *__restrict__ shape_sel, int shape_id)
{
    // two shapes are launched back to back; the step's replay total picks one
    if (shape_sel && *shape_sel != shape_id) return;
    constexpr int kT = BwdShape<PPT>::kThreads;
    constexpr int kWarps = BwdShape<PPT>::kWarps;
    // records per batch: 128 for float; half that for double so the
    // per-warp partial sums still fit the 48 KB of static shared memory
    constexpr int kB = sizeof(T) == 4 ? kBatch : kBatch / 2;
    __shared__ SmemSplat<T> sm[kB];
    __shared__ int32_t srow[kB];
    __shared__ uint32_t se[DET ? kB : 1];   // DET: each staged pair's rank-major index
    __shared__ T acc[kWarps][kB][9];   // per-warp partial sums: plain stores, no smem atomics
    __shared__ int s_end;
    const int warp = threadIdx.x >> 5;
    const int slot = reduce9_slot(threadIdx.x & 31);
    const int tile = order ? order[blockIdx.x] : blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    // compact pixel blocks per warp: a splat's footprint touches fewer
    // warps, and fewer lanes idle inside a touched warp
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    int lx, ly0, dyp;
    if (PPT == 1) {
        lx = ((wq & 1) << 3) + (lane & 7);
        ly0 = ((wq >> 1) << 2) + (lane >> 3);
        dyp = 0;
    } else if (PPT == 2) {
        lx = ((wq & 1) << 3) + (lane & 7);
        ly0 = ((wq >> 1) << 3) + (lane >> 3);
        dyp = 4;
    } else {
        lx = lane & 15;
        ly0 = (wq << 3) + ((lane >> 4) << 2);
        dyp = 1;
    }
    const int px = tx * kTile + lx;
    const T fpx = (T)px;
    T fpy[PPT];
    const int lo = offsets[tile], hi = offsets[tile + 1];

    BwdPix<T> P[PPT];
    int my_end = 0;
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
        const int py = ty * kTile + ly0 + i * dyp;
        fpy[i] = (T)py;
        bwd_init(P[i], px, py, width, height, dC_img, cfinal, last_img, hi - lo, early, thresh);
        my_end = max(my_end, P[i].end);
    }
    if (threadIdx.x == 0) s_end = 0;
    __syncthreads();
    if (my_end > 0) atomicMax(&s_end, my_end);
    __syncthreads();
    const int end = lo + s_end;
    // this warp's own replay bound: past it none of its pixels contributes
    const int wend = lo + (int)__reduce_max_sync(0xffffffffu, (unsigned)my_end);

    for (int base = lo; base < end; base += kB) {
        for (int i = threadIdx.x; i < kB; i += kT) {
            const int k = base + i;
            if (k < end) {
                T rec[12];
                const int row = pair_gaussian[k];
                if (DET) {   // where the pair's partial goes (loads overlap the record's)
                    const uint32_t r = __ldg(maps.rank_of + row);
                    se[i] = __ldg(maps.rank_e0 + r) + kept_index(maps, r, tx, ty, tiles_x);
                    maps.rank_hit[r] = 1;
                }
                load_record(records, row, rec);
                stage(sm[i], rec);
                srow[i] = row;
            }
#pragma unroll
            for (int w = 0; w < kWarps; ++w)
#pragma unroll
                for (int v = 0; v < 9; ++v) acc[w][i][v] = (T)0;
        }
        __syncthreads();
        const int nb = min(kB, end - base);
        const int wnb = min(nb, wend - base);
        // kU Gaussians per trip: their pixel replays stay in list order, and
        // each one's warp reduction can overlap the next one's math
        constexpr int kU = kUnroll<PPT>;
        for (int j = 0; j < wnb; j += kU) {
            bool all_done = true;
#pragma unroll
            for (int i = 0; i < PPT; ++i) all_done &= P[i].done;
            if (__all_sync(0xffffffffu, all_done)) break;  // warp-uniform
            T g[kU][9];
            bool c[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
#pragma unroll
                for (int v = 0; v < 9; ++v) g[u][v] = (T)0;
                c[u] = false;
                if (j + u < wnb) {
                    const SmemSplat<T> su = sm[j + u];
                    if (!(fpx < su.bx0 || fpx > su.bx1)) {
#pragma unroll
                        for (int i = 0; i < PPT; ++i)
                            c[u] |= bwd_pixel(P[i], su, fpx, fpy[i], base + j + u - lo, early,
                                              thresh, g[u]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (__ballot_sync(0xffffffffu, c[u])) {
                    const T red = warp_reduce9(g[u]);
                    if (slot >= 0) acc[warp][j + u][slot] = red;
                }
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nb; i += kT) {
            const int row = srow[i];
            T a[9];
            bool nz = false;
#pragma unroll
            for (int v = 0; v < 9; ++v) {
                T sum = acc[0][i][v];
#pragma unroll
                for (int w = 1; w < kWarps; ++w) sum += acc[w][i][v];
                a[v] = sum;
                nz |= sum != (T)0;
            }
            if (DET) {
                const uint32_t e = se[i];
                store_partial(partial + (int64_t)e * kPartialReals, a);
                maps.pvalid[e] = 1;
            } else if (nz) {
                atomicAdd(d_mean + 2 * row, a[0]);
                atomicAdd(d_mean + 2 * row + 1, a[1]);
                atomicAdd(d_conic + 3 * row, a[2]);
                atomicAdd(d_conic + 3 * row + 1, a[3]);
                atomicAdd(d_conic + 3 * row + 2, a[4]);
                atomicAdd(d_op + row, a[5]);
                atomicAdd(d_col + 3 * row, a[6]);
                atomicAdd(d_col + 3 * row + 1, a[7]);
                atomicAdd(d_col + 3 * row + 2, a[8]);
            }
        }
        __syncthreads();
    }
}

// The launch shape.  Short replays (a keyframe stepped repeatedly: depth-
// limited lists, ~120 replayed pairs per tile at config 3) favour one pixel
// per thread (more warps on a tile's serial replay: 393 vs 400 us); long
// ones (full lists, ~400 per tile in the config-4 stream) two (each warp's
// reduction amortised over 64 pixels: the stream 268 -> 284 it/s).  With a
// tile schedule the choice is made on the device from the forward's replay
// lengths (tile_order_kernel's total) and both shapes are launched, one
// leaving at once.
constexpr int kBwdHeavyPerTile = 256;     // replayed pairs per tile, on average
constexpr int kPPTLight = 1, kPPTHeavy = 2;

}  // namespace sb

using namespace sb;

extern "C" int32_t sb_blend_bwd(int32_t dtype, const void *records, const int32_t *pair_gaussian,
                                const int32_t *offsets, int32_t width, int32_t height,
                                int32_t tile_size, int32_t early_termination,
                                double term_threshold, const void *d_color_image,
                                const void *c_final, const int32_t *last, void *d_mean2d,
                                void *d_conic, void *d_opacity, void *d_color,
                                const int32_t *tile_sched_in, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(tile_size == kTile, "tile_size %d unsupported (only %d)", tile_size, kTile);
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    cudaStream_t st = as_stream(stream);
#define BWD_ARGS(T)                                                                            \
    (const T *)records, pair_gaussian, offsets, width, height, tiles_x, early_termination,      \
        (T)term_threshold, (const T *)d_color_image, (const T *)c_final, last, (T *)d_mean2d,   \
        (T *)d_conic, (T *)d_opacity, (T *)d_color, order, nullptr, BinMaps{}, nullptr, 0
    const int n_tiles = tiles_x * tiles_y;
    const int32_t *order = nullptr;
    if (tile_sched_in && last) {   // heavy-first by the forward's replay lengths
        int32_t *sched = const_cast<int32_t *>(tile_sched_in);
        tile_order_kernel<<<1, kSchedThreads, 0, st>>>(nullptr, sched + n_tiles, n_tiles,
                                                       sched + 2 * n_tiles);
        order = sched + 2 * n_tiles;
    }
    constexpr int kTh = BwdShape<kPPTHeavy>::kThreads;
    if (dtype == SB_F32) blend_bwd_kernel<float, false, kPPTHeavy><<<tiles_x * tiles_y, kTh, 0, st>>>(BWD_ARGS(float));
    else blend_bwd_kernel<double, false, kPPTHeavy><<<tiles_x * tiles_y, kTh, 0, st>>>(BWD_ARGS(double));
#undef BWD_ARGS
    return check_launch("blend_bwd_kernel");
}

static inline size_t bwd_a256(size_t x) { return (x + 255) & ~size_t(255); }

extern "C" size_t sb_blend_bwd_workspace_bytes(int32_t dtype, int64_t pair_capacity,
                                               int32_t width, int32_t height)
{
    const size_t rs = dtype == SB_F64 ? 8 : 4;
    const int64_t n_tiles = (int64_t)((width + kTile - 1) / kTile) * ((height + kTile - 1) / kTile);
    const int64_t cap = pair_capacity > 0 ? pair_capacity : 1;
    (void)n_tiles;
    return bwd_a256((size_t)kPartialReals * rs * (size_t)cap) +
           bwd_a256(16 * (size_t)(cap / kGatherQueueDiv + 1)) + 256;
}

struct BwdWs {
    void *partial, *queue;
    uint32_t *queue_n;
};

static BwdWs bwd_ws(int32_t dtype, int64_t pair_capacity, void *workspace)
{
    const size_t rs = dtype == SB_F64 ? 8 : 4;
    char *ws = (char *)workspace;
    const int64_t cap = pair_capacity > 0 ? pair_capacity : 1;
    BwdWs w;
    w.partial = ws;            // one record per rank-major pair index
    size_t off = bwd_a256((size_t)kPartialReals * rs * (size_t)cap);
    w.queue = ws + off;        // long ranks of the gather (launch_gather_adjoints)
    off += bwd_a256(16 * (size_t)(cap / kGatherQueueDiv + 1));
    w.queue_n = (uint32_t *)(ws + off);
    return w;
}

extern "C" int32_t sb_blend_bwd_partials(int32_t dtype, const void *records,
                                         const int32_t *pair_gaussian, const int32_t *offsets,
                                         int32_t width, int32_t height, int32_t tile_size,
                                         int32_t early_termination, double term_threshold,
                                         const void *d_color_image, const void *c_final,
                                         const int32_t *last, const int32_t *tile_sched_in,
                                         int64_t m, int64_t pair_capacity,
                                         void *bin_workspace, void *workspace,
                                         size_t workspace_bytes, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(tile_size == kTile, "tile_size %d unsupported (only %d)", tile_size, kTile);
    SB_REQUIRE(bin_workspace != nullptr, "bin_workspace is NULL (the sb_bin workspace of the pairs)");
    SB_REQUIRE(workspace != nullptr &&
                   workspace_bytes >= sb_blend_bwd_workspace_bytes(dtype, pair_capacity, width, height),
               "blend_bwd workspace too small");
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int n_tiles = tiles_x * tiles_y;
    cudaStream_t st = as_stream(stream);
    const BwdWs w = bwd_ws(dtype, pair_capacity, workspace);
    const BinMaps maps = bin_maps(m, pair_capacity, width, height, bin_workspace);
    const int32_t *order = nullptr;
    int32_t *sel = nullptr;
    if (tile_sched_in && last) {   // heavy-first by the forward's replay lengths
        int32_t *sched = const_cast<int32_t *>(tile_sched_in);
        sel = reinterpret_cast<int32_t *>(w.queue_n + 1);   // in the workspace's tail
        tile_order_kernel<<<1, kSchedThreads, 0, st>>>(nullptr, sched + n_tiles, n_tiles,
                                                       sched + 2 * n_tiles, sel,
                                                       (long long)kBwdHeavyPerTile * n_tiles);
        order = sched + 2 * n_tiles;
    }
#define BWD_ARGS(T, ID)                                                                        \
    (const T *)records, pair_gaussian, offsets, width, height, tiles_x, early_termination,      \
        (T)term_threshold, (const T *)d_color_image, (const T *)c_final, last, nullptr,         \
        nullptr, nullptr, nullptr, order, (T *)w.partial, maps, sel, ID
    constexpr int kTl = BwdShape<kPPTLight>::kThreads, kTh = BwdShape<kPPTHeavy>::kThreads;
    if (dtype == SB_F32) {
        if (sel) blend_bwd_kernel<float, true, kPPTLight><<<n_tiles, kTl, 0, st>>>(BWD_ARGS(float, 0));
        blend_bwd_kernel<float, true, kPPTHeavy><<<n_tiles, kTh, 0, st>>>(BWD_ARGS(float, 1));
    } else {
        if (sel) blend_bwd_kernel<double, true, kPPTLight><<<n_tiles, kTl, 0, st>>>(BWD_ARGS(double, 0));
        blend_bwd_kernel<double, true, kPPTHeavy><<<n_tiles, kTh, 0, st>>>(BWD_ARGS(double, 1));
    }
#undef BWD_ARGS
    return check_launch("blend_bwd_kernel");
}

extern "C" int32_t sb_gather_adjoints(int32_t dtype, int64_t m, int64_t pair_capacity,
                                      int32_t width, int32_t height, int64_t sort_capacity,
                                      const void *bin_workspace, void *workspace,
                                      size_t workspace_bytes, void *d_mean2d, void *d_conic,
                                      void *d_opacity, void *d_color, uint8_t *reached_rows,
                                      void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(bin_workspace != nullptr, "bin_workspace is NULL (the sb_bin workspace of the pairs)");
    SB_REQUIRE(workspace != nullptr &&
                   workspace_bytes >= sb_blend_bwd_workspace_bytes(dtype, pair_capacity, width, height),
               "blend_bwd workspace too small");
    const BwdWs w = bwd_ws(dtype, pair_capacity, workspace);
    return launch_gather_adjoints(dtype, m, pair_capacity, width, height, sort_capacity,
                                  bin_workspace, w.partial, d_mean2d, d_conic, d_opacity, d_color,
                                  w.queue, w.queue_n, reached_rows, as_stream(stream));
}

extern "C" int32_t sb_blend_bwd_det(int32_t dtype, const void *records,
                                    const int32_t *pair_gaussian, const int32_t *offsets,
                                    int32_t width, int32_t height, int32_t tile_size,
                                    int32_t early_termination, double term_threshold,
                                    const void *d_color_image, const void *c_final,
                                    const int32_t *last, void *d_mean2d, void *d_conic,
                                    void *d_opacity, void *d_color, const int32_t *tile_sched_in,
                                    int64_t m, int64_t pair_capacity, int64_t sort_capacity,
                                    const void *bin_workspace, void *workspace,
                                    size_t workspace_bytes, void *stream)
{
    const int32_t rc = sb_blend_bwd_partials(
        dtype, records, pair_gaussian, offsets, width, height, tile_size, early_termination,
        term_threshold, d_color_image, c_final, last, tile_sched_in, m, pair_capacity,
        const_cast<void *>(bin_workspace), workspace, workspace_bytes, stream);
    if (rc != SB_OK) return rc;
    return sb_gather_adjoints(dtype, m, pair_capacity, width, height, sort_capacity,
                              bin_workspace, workspace, workspace_bytes, d_mean2d, d_conic,
                              d_opacity, d_color, nullptr, stream);
}
