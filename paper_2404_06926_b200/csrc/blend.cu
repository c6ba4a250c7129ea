// blend.cu -- K6 forward blend and K8 backward blend.
//
// a4 _composite_tiles, forward.py:261-342 (+ exposure epilogue, loss.py:31-36)
// a6 _backward_tiles,  backward.py:91-213
//
// One CTA per 16x16 tile.  The forward runs one thread per pixel (256); the
// backward runs 128 threads that each own two pixels of one column, rows y and
// y + 8, so its per-Gaussian overhead (shared-memory record read, box test,
// warp vote, reduction) is amortised over two pixels.  The tile's
// depth-ordered pair list is walked in batches of splat records staged in
// shared memory (one coalesced record load per thread), so each record is
// read from L2/HBM once per tile.  A pixel stops when T < 1e-4
// (checked BEFORE each Gaussian, like the reference: the Gaussian that drives T
// below the threshold is still composited); a warp skips work once all its
// pixels are done and the CTA leaves the list once all are
// (__syncthreads_count).
//
// The forward records, per pixel, 1 + the list position of its last
// contributor; the backward replays the tile only up to the max of that over
// the tile (P_proc in SURVEY §8), front to back, recomputing each alpha with
// a 2-ulp hardware exp (the gradients are tolerance-checked; the forward's
// correctly rounded exp is what fixes the rendered image and the replay
// bound).  Per
// Gaussian, a thread adds its two pixels' 9 screen-space adjoints, the warp
// reduces them with a 12-shuffle transpose-reduce into a per-warp shared slot
// (plain stores -- shared-memory float atomics compile to CAS loops), the 4
// warps' slots are summed once per batch, and one global atomic per (tile,
// Gaussian, value) follows.
#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

constexpr int kThreads = kTilePx / 2;  // 128 threads, two pixels each
constexpr int kBatch = kThreads;        // records per shared-memory batch

// exp(x) for the blend's range (x = -q/2 with 0 <= q <= q_cut + 1/64 <
// 2 ln 255 + 1/64, so -5.6 < x <= ~0): Cody-Waite reduction by ln 2 and a
// degree-12 Taylor polynomial in double (|r| <= 0.347: truncation 2e-16),
// then ONE rounding to float -- correctly rounded except with probability
// ~2^-28 per evaluation, like the (float)exp((double)x) of the oracle.
__device__ __forceinline__ float blend_exp(float xf)
{
    const double x = (double)xf;
    const double n = rint(x * 1.4426950408889634);
    const double r = __fma_rn(-n, 1.9082149292705877e-10, __fma_rn(-n, 0.6931471803691238, x));
    // Estrin's scheme: dependency depth 5 instead of Horner's 12 (the DFMA
    // latency chain, not the issue slots, was the cost); same accuracy class
    const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
    const double q0 = __fma_rn(r, 1.0, 1.0);                                          // 1 + r
    const double q1 = __fma_rn(r, 1.66666666666666666667e-01, 0.5);                   // 1/2! 1/3!
    const double q2 = __fma_rn(r, 8.33333333333333333333e-03, 4.16666666666666666667e-02);   // 1/4! 1/5!
    const double q3 = __fma_rn(r, 1.98412698412698412698e-04, 1.38888888888888888889e-03);   // 1/6! 1/7!
    const double q4 = __fma_rn(r, 2.75573192239858906526e-06, 2.48015873015873015873e-05);   // 1/8! 1/9!
    const double q5 = __fma_rn(r, 2.50521083854417187751e-08, 2.75573192239858906526e-07);   // 1/10! 1/11!
    const double s0 = __fma_rn(q1, r2, q0), s1 = __fma_rn(q3, r2, q2);
    const double s2 = __fma_rn(q5, r2, q4);
    const double t0 = __fma_rn(s1, r4, s0);
    const double t1 = __fma_rn(2.08767569878680989792e-09, r4, s2);                   // 1/12!
    const double p = __fma_rn(t1, r8, t0);
    const double scale = __longlong_as_double((long long)((int)n + 1023) << 52);
    return (float)(p * scale);
}
__device__ __forceinline__ double blend_exp(double x) { return exp(x); }

// The backward's exp: a 2-ulp hardware exp (ex2.approx) in float.  The
// backward's alphas feed gradients compared within a tolerance, and its
// replay is bounded by the forward's recorded last contributor, so it does
// not need the forward's correctly rounded exp (which is ~40 issue slots).
__device__ __forceinline__ float bwd_exp(float x) { return __expf(x); }
__device__ __forceinline__ double bwd_exp(double x) { return exp(x); }

// correctly rounded reciprocal: bitwise equal to 1 / x, cheaper than a divide
__device__ __forceinline__ float rrcp(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rrcp(double x) { return __drcp_rn(x); }

// 16 reals, 16-byte aligned: a thread copies a staged record into registers
// with four 128-bit shared loads per Gaussian
template <typename T>
struct __align__(16) SmemSplat {
    T mx, my, a, b, c, opa, qc, c0, c1, c2, dep;
    T bx0, bx1, by0, by1;  // pixel box [ceil(m - r), floor(m + r)] (forward.py:296-299)
    T pad;
};

template <typename T>
__device__ __forceinline__ void stage(SmemSplat<T> &s, const T rec[12])
{
    s.mx = rec[R_MX]; s.my = rec[R_MY];
    s.a = rec[R_A]; s.b = rec[R_B]; s.c = rec[R_C];
    s.opa = rec[R_OP];
    s.qc = rec[R_QC] + (T)1 / (T)64;  // q margin, forward.py:287
    s.c0 = rec[R_C0]; s.c1 = rec[R_C1]; s.c2 = rec[R_C2]; s.dep = rec[R_DEP];
    const T r = rec[R_RAD];
    s.bx0 = rceil(s.mx - r); s.bx1 = rfloor(s.mx + r);
    s.by0 = rceil(s.my - r); s.by1 = rfloor(s.my + r);
}

// Per-pixel forward state
template <typename T>
struct FwdPix {
    T Tr, C0, C1, C2, D;
    T ldep;   // depth of the last contributor
    int32_t nc, last;
    bool done;
};

template <typename T>
__device__ __forceinline__ void fwd_pixel(FwdPix<T> &st, const SmemSplat<T> &s, T fpx, T fpy,
                                          int list_pos, int early, T thresh)
{
    const T one = (T)1, half = one / (T)2, two = one + one;
    if (st.done || fpy < s.by0 || fpy > s.by1) return;
    const T dy = fpy - s.my;
    const T qy = s.c * dy * dy;
    const T bdy = two * s.b * dy;
    const T dx = fpx - s.mx;
    const T q = s.a * dx * dx + bdy * dx + qy;
    if (q > s.qc) return;
    T alpha = s.opa * blend_exp(-(half * q));
    if (alpha > (T)kAlphaClamp) alpha = (T)kAlphaClamp;
    if (alpha < (T)kAlphaCutoff) return;
    const T w = alpha * st.Tr;
    st.C0 += w * s.c0;
    st.C1 += w * s.c1;
    st.C2 += w * s.c2;
    st.D += w * s.dep;
    st.nc += 1;
    st.last = list_pos + 1;
    st.ldep = s.dep;
    st.Tr = st.Tr * (one - alpha);
    // termination is tested before the next Gaussian (forward.py:310)
    if (early && st.Tr < thresh) st.done = true;
}

// Forward: one pixel per thread (256 threads) -- the per-pixel dependency
// chain (exp, then the transmittance update) needs the extra warps to hide
// its latency; the backward amortises its heavier per-Gaussian reduction over
// two pixels per thread instead.
constexpr int kFwdThreads = kTilePx;

template <typename T, bool kExposure>
__global__ void __launch_bounds__(kFwdThreads) blend_fwd_kernel(
    const T *__restrict__ records, const int32_t *__restrict__ pair_gaussian,
    const int32_t *__restrict__ offsets, int width, int height, int tiles_x, int early,
    T thresh, const T *__restrict__ expo, T *__restrict__ out_c, T *__restrict__ out_d,
    T *__restrict__ out_t, T *__restrict__ out_o, int32_t *__restrict__ out_nc,
    int32_t *__restrict__ out_last, T *__restrict__ out_y, float *__restrict__ dlim,
    int64_t *__restrict__ status)
{
    __shared__ SmemSplat<T> sm[kFwdThreads];
    __shared__ float s_dep;
    const int tile = blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x >> 4;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const T fpx = (T)px, fpy = (T)py;
    const int lo = offsets[tile], hi = offsets[tile + 1];

    FwdPix<T> A;
    A.Tr = (T)1;
    A.C0 = A.C1 = A.C2 = A.D = (T)0;
    A.ldep = (T)0;
    A.nc = A.last = 0;
    A.done = !(px < width && py < height) || (early && (T)1 < thresh);

    for (int base = lo; base < hi; base += kFwdThreads) {
        if (__syncthreads_count(!A.done) == 0) break;
        const int k = base + threadIdx.x;
        if (k < hi) {
            T rec[12];
            load_record(records, pair_gaussian[k], rec);
            stage(sm[threadIdx.x], rec);
        }
        __syncthreads();
        const int nb = min(kFwdThreads, hi - base);
        for (int j = 0; j < nb && !A.done; ++j) {
            const SmemSplat<T> s = sm[j];
            if (fpx < s.bx0 || fpx > s.bx1) continue;
            fwd_pixel(A, s, fpx, fpy, base + j - lo, early, thresh);
        }
    }
    if (dlim) {
        // per-tile depth limit for the next iteration's binning: a tile whose
        // every pixel terminated needs its pairs only up to about the depth of
        // its deepest last contributor (25% margin); other tiles need them
        // all.  A tile that was limited this time and did not terminate
        // everywhere may have lost contributors: the iteration is flagged
        // (status[1]) and the caller re-runs it with full lists.
        if (threadIdx.x == 0) s_dep = 0.f;
        const int saturated = __syncthreads_and(A.done);
        if (A.last > 0) atomicMax(reinterpret_cast<int *>(&s_dep), __float_as_int((float)A.ldep));
        __syncthreads();
        if (threadIdx.x == 0) {
            const float old = dlim[tile];
            if (!saturated && old < INFINITY && status) status[1] = 1;
            dlim[tile] = saturated ? s_dep * 1.25f + 1e-3f : INFINITY;
        }
    }
    if (!(px < width && py < height)) return;
    const T one = (T)1;
    const int64_t pix = (int64_t)py * width + px;
    out_c[3 * pix] = A.C0;
    out_c[3 * pix + 1] = A.C1;
    out_c[3 * pix + 2] = A.C2;
    out_d[pix] = A.D;
    out_t[pix] = A.Tr;
    if (out_o) out_o[pix] = one - A.Tr;
    out_nc[pix] = A.nc;
    if (out_last) out_last[pix] = A.last;
    if (kExposure) {
        // Y = C M^T + b (loss.py:157-158, BLAS FMA chain)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            out_y[3 * pix + c] =
                rfma(A.C2, expo[4 * c + 2], rfma(A.C1, expo[4 * c + 1], A.C0 * expo[4 * c])) +
                expo[4 * c + 3];
    }
}

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
    const T qy = s.c * dy * dy;
    const T bdy = two * s.b * dy;
    const T dx = fpx - s.mx;
    const T q = s.a * dx * dx + bdy * dx + qy;
    if (q > s.qc) return false;
    const T gauss = bwd_exp(-(half * q));
    const T alpha_raw = s.opa * gauss;
    T alpha = alpha_raw;
    if (alpha > clamp) alpha = clamp;
    if (alpha < (T)kAlphaCutoff) return false;
    const T Tr = st.Tr;
    const T w = alpha * Tr;
    const T p0 = st.P0 + w * s.c0;
    const T p1 = st.P1 + w * s.c1;
    const T p2 = st.P2 + w * s.c2;
    g[6] += w * st.dc0;
    g[7] += w * st.dc1;
    g[8] += w * st.dc2;
    if (alpha_raw < clamp) {
        const T inv_rest = rrcp(one - alpha);   // == one / (one - alpha), bitwise
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
    st.Tr = Tr * (one - alpha);
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

template <typename T>
__global__ void __launch_bounds__(kThreads) blend_bwd_kernel(
    const T *__restrict__ records, const int32_t *__restrict__ pair_gaussian,
    const int32_t *__restrict__ offsets, int width, int height, int tiles_x, int early,
    T thresh, const T *__restrict__ dC_img, const T *__restrict__ cfinal,
    const int32_t *__restrict__ last_img, T *__restrict__ d_mean, T *__restrict__ d_conic,
    T *__restrict__ d_op, T *__restrict__ d_col)
{
    // records per batch: one per thread for float; half that for double so
    // the per-warp partial sums still fit the 48 KB of static shared memory
    constexpr int kB = sizeof(T) == 4 ? kBatch : kBatch / 2;
    constexpr int kWarps = kThreads / 32;
    __shared__ SmemSplat<T> sm[kB];
    __shared__ int32_t srow[kB];
    __shared__ T acc[kWarps][kB][9];   // per-warp partial sums: plain stores, no smem atomics
    __shared__ int s_end;
    const int warp = threadIdx.x >> 5;
    const int slot = reduce9_slot(threadIdx.x & 31);
    const int tile = blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x >> 4;
    const int px = tx * kTile + lx;
    const int py0 = ty * kTile + ly, py1 = py0 + 8;
    const T fpx = (T)px, fpy0 = (T)py0, fpy1 = (T)py1;
    const int lo = offsets[tile], hi = offsets[tile + 1];

    BwdPix<T> A, B;
    bwd_init(A, px, py0, width, height, dC_img, cfinal, last_img, hi - lo, early, thresh);
    bwd_init(B, px, py1, width, height, dC_img, cfinal, last_img, hi - lo, early, thresh);
    if (threadIdx.x == 0) s_end = 0;
    __syncthreads();
    const int my_end = max(A.end, B.end);
    if (my_end > 0) atomicMax(&s_end, my_end);
    __syncthreads();
    const int end = lo + s_end;
    // this warp's own replay bound: past it none of its pixels contributes
    const int wend = lo + (int)__reduce_max_sync(0xffffffffu, (unsigned)my_end);

    for (int base = lo; base < end; base += kB) {
        const int k = base + threadIdx.x;
        if (threadIdx.x < kB) {
            if (k < end) {
                T rec[12];
                const int row = pair_gaussian[k];
                load_record(records, row, rec);
                stage(sm[threadIdx.x], rec);
                srow[threadIdx.x] = row;
            }
#pragma unroll
            for (int w = 0; w < kWarps; ++w)
#pragma unroll
                for (int v = 0; v < 9; ++v) acc[w][threadIdx.x][v] = (T)0;
        }
        __syncthreads();
        const int nb = min(kB, end - base);
        const int wnb = min(nb, wend - base);
        for (int j = 0; j < wnb; ++j) {
            if (__all_sync(0xffffffffu, A.done && B.done)) break;  // warp-uniform
            const SmemSplat<T> s = sm[j];
            T g[9];
#pragma unroll
            for (int v = 0; v < 9; ++v) g[v] = (T)0;
            bool contrib = false;
            if (!(fpx < s.bx0 || fpx > s.bx1)) {
                contrib |= bwd_pixel(A, s, fpx, fpy0, base + j - lo, early, thresh, g);
                contrib |= bwd_pixel(B, s, fpx, fpy1, base + j - lo, early, thresh, g);
            }
            if (__ballot_sync(0xffffffffu, contrib)) {
                const T red = warp_reduce9(g);
                if (slot >= 0) acc[warp][j][slot] = red;
            }
        }
        __syncthreads();
        if (threadIdx.x < nb) {
            const int row = srow[threadIdx.x];
            T a[9];
            bool nz = false;
#pragma unroll
            for (int v = 0; v < 9; ++v) {
                T sum = acc[0][threadIdx.x][v];
#pragma unroll
                for (int w = 1; w < kWarps; ++w) sum += acc[w][threadIdx.x][v];
                a[v] = sum;
                nz |= sum != (T)0;
            }
            if (nz) {
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

}  // namespace sb

using namespace sb;

extern "C" int32_t sb_blend_fwd(int32_t dtype, const void *records, const int32_t *pair_gaussian,
                                const int32_t *offsets, int32_t width, int32_t height,
                                int32_t tile_size, int32_t early_termination,
                                double term_threshold, const void *exposure, void *out_color,
                                void *out_depth, void *out_transmittance, void *out_opacity,
                                int32_t *out_n_contrib, int32_t *out_last, void *out_y,
                                float *tile_depth_limit, int64_t *d_status, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(tile_size == kTile, "tile_size %d unsupported (only %d)", tile_size, kTile);
    SB_REQUIRE(width > 0 && height > 0, "bad image size");
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const bool ex = exposure != nullptr && out_y != nullptr;
    cudaStream_t st = as_stream(stream);
#define FWD_ARGS(T)                                                                            \
    (const T *)records, pair_gaussian, offsets, width, height, tiles_x, early_termination,      \
        (T)term_threshold, (const T *)exposure, (T *)out_color, (T *)out_depth,                 \
        (T *)out_transmittance, (T *)out_opacity, out_n_contrib, out_last, (T *)out_y,         \
        tile_depth_limit, d_status
    if (dtype == SB_F32) {
        if (ex) blend_fwd_kernel<float, true><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(float));
        else blend_fwd_kernel<float, false><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(float));
    } else {
        if (ex) blend_fwd_kernel<double, true><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(double));
        else blend_fwd_kernel<double, false><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(double));
    }
#undef FWD_ARGS
    return check_launch("blend_fwd_kernel");
}

extern "C" int32_t sb_blend_bwd(int32_t dtype, const void *records, const int32_t *pair_gaussian,
                                const int32_t *offsets, int32_t width, int32_t height,
                                int32_t tile_size, int32_t early_termination,
                                double term_threshold, const void *d_color_image,
                                const void *c_final, const int32_t *last, void *d_mean2d,
                                void *d_conic, void *d_opacity, void *d_color, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(tile_size == kTile, "tile_size %d unsupported (only %d)", tile_size, kTile);
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    cudaStream_t st = as_stream(stream);
#define BWD_ARGS(T)                                                                            \
    (const T *)records, pair_gaussian, offsets, width, height, tiles_x, early_termination,      \
        (T)term_threshold, (const T *)d_color_image, (const T *)c_final, last, (T *)d_mean2d,   \
        (T *)d_conic, (T *)d_opacity, (T *)d_color
    if (dtype == SB_F32) blend_bwd_kernel<float><<<tiles_x * tiles_y, kThreads, 0, st>>>(BWD_ARGS(float));
    else blend_bwd_kernel<double><<<tiles_x * tiles_y, kThreads, 0, st>>>(BWD_ARGS(double));
#undef BWD_ARGS
    return check_launch("blend_bwd_kernel");
}
