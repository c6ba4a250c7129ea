// blend.cu -- K6 forward blend (a4 _composite_tiles, forward.py:261-342, +
// exposure epilogue, loss.py:31-36).
//
// One CTA per 16x16 tile, one thread per pixel.  The tile's depth-ordered
// pair list is walked in batches of splat records staged in shared memory
// (one coalesced record load per thread), so each record is read from L2/HBM
// once per tile.  A pixel stops when T < 1e-4 (checked BEFORE each Gaussian,
// like the reference: the Gaussian that drives T below the threshold is still
// composited); the CTA leaves the list once all pixels are done
// (__syncthreads_count).  The forward records, per pixel, 1 + the list
// position of its last contributor: the backward (blend_bwd.cu) replays the
// tile only up to the max of that over the tile.
//
// Compiled with -fmad=false: every alpha, colour and transmittance is the
// reference's float operation sequence, exp correctly rounded.
#include "blend_common.cuh"

namespace sb {

// Per-pixel forward state
template <typename T>
struct FwdPix {
    T Tr, C0, C1, C2, D;
    T ldep;   // depth of the last contributor
    int32_t nc, last;
    bool done;
};

// FAST (float): the mapping step's forward -- alpha from step_q/step_gauss
// (the hardware exp; the exact operations the backward replays with), FMA
// accumulation -- whose outputs feed a tolerance-checked loss and gradients.
// Otherwise the render API's forward: the reference's float operation
// sequence with the correctly rounded exp (bit-identical to it).
template <typename T, bool FAST>
__device__ __forceinline__ void fwd_pixel(FwdPix<T> &st, const SmemSplat<T> &s, T fpx, T fpy,
                                          int list_pos, int early, T thresh,
                                          const double *__restrict__ tab)
{
    const T one = (T)1, half = one / (T)2, two = one + one;
    if (st.done || fpy < s.by0 || fpy > s.by1) return;
    if constexpr (FAST && sizeof(T) == 4) {
        const float q = step_q(s, fpx - s.mx, fpy - s.my);
        if (q > s.qc) return;
        float alpha = __fmul_rn(s.opa, step_gauss(q));
        if (alpha > (float)kAlphaClamp) alpha = (float)kAlphaClamp;
        if (alpha < (float)kAlphaCutoff) return;
        const float w = __fmul_rn(alpha, st.Tr);
        st.C0 = __fmaf_rn(w, s.c0, st.C0);
        st.C1 = __fmaf_rn(w, s.c1, st.C1);
        st.C2 = __fmaf_rn(w, s.c2, st.C2);
        st.D = __fmaf_rn(w, s.dep, st.D);
        st.nc += 1;
        st.last = list_pos + 1;
        st.ldep = s.dep;
        st.Tr = __fmul_rn(st.Tr, __fsub_rn(1.0f, alpha));
    } else {
        const T dy = fpy - s.my;
        const T qy = s.c * dy * dy;
        const T bdy = two * s.b * dy;
        const T dx = fpx - s.mx;
        const T q = s.a * dx * dx + bdy * dx + qy;
        if (q > s.qc) return;
        T alpha = s.opa * blend_exp(-(half * q), tab);
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
    }
    // termination is tested before the next Gaussian (forward.py:310)
    if (early && st.Tr < thresh) st.done = true;
}

// One pixel per thread (256 threads): the per-pixel dependency chain (exp,
// then the transmittance update) needs the warps to hide its latency; the
// backward amortises its heavier per-Gaussian reduction over two pixels per
// thread instead.
constexpr int kFwdThreads = kTilePx;

template <typename T, bool kExposure, bool FAST = false>
__global__ void __launch_bounds__(kFwdThreads) blend_fwd_kernel(
    const T *__restrict__ records, const int32_t *__restrict__ pair_gaussian,
    const int32_t *__restrict__ offsets, int width, int height, int tiles_x, int early,
    T thresh, const T *__restrict__ expo, T *__restrict__ out_c, T *__restrict__ out_d,
    T *__restrict__ out_t, T *__restrict__ out_o, int32_t *__restrict__ out_nc,
    int32_t *__restrict__ out_last, T *__restrict__ out_y, float *__restrict__ dlim,
    int64_t *__restrict__ status, float *__restrict__ coarse, const int32_t *__restrict__ order,
    int32_t *__restrict__ replay, int64_t *__restrict__ halt)
{
    // an iteration the binning already flagged (pair overflow, halt) halts
    // the engine: the iterations queued behind it become no-ops
    if (halt && status && blockIdx.x == 0 && threadIdx.x == 0 && status[1]) *halt = 1;
    __shared__ SmemSplat<T> sm[kFwdThreads];
    __shared__ float s_dep;
    __shared__ int s_replay;
    __shared__ double s_tab[32];
    if (threadIdx.x < 32) s_tab[threadIdx.x] = kExp2Tab[threadIdx.x];   // read after the loop's first barrier
    if (threadIdx.x == 0) s_replay = 0;
    const int tile = order ? order[blockIdx.x] : blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    // each warp owns a compact 8x4 block of the tile: a splat's footprint
    // touches fewer warps, and fewer lanes idle inside a touched warp
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int lx = ((wq & 1) << 3) + (lane & 7), ly = ((wq >> 1) << 2) + (lane >> 3);
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
            fwd_pixel<T, FAST>(A, s, fpx, fpy, base + j - lo, early, thresh, s_tab);
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
            if (!saturated && old < INFINITY && status) {
                status[1] = 1;
                if (halt) *halt = 1;   // the iterations behind this one become no-ops
            }
            const float lim = saturated ? s_dep * 1.25f + 1e-3f : INFINITY;
            dlim[tile] = lim;
            if (coarse)   // 4x4-tile maxima for the next sb_preprocess_fwd (caller-zeroed)
                atomicMax(reinterpret_cast<int *>(coarse) + (ty >> 2) * ((tiles_x + 3) >> 2) + (tx >> 2),
                          __float_as_int(lim));
        }
    }
    if (replay) {
        // the tile's replay length (the backward's cost estimate)
        __syncthreads();
        if (A.last > 0) atomicMax(&s_replay, A.last);
        __syncthreads();
        if (threadIdx.x == 0) replay[tile] = s_replay;
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

}  // namespace sb

using namespace sb;

extern "C" int32_t sb_blend_fwd(int32_t dtype, const void *records, const int32_t *pair_gaussian,
                                const int32_t *offsets, int32_t width, int32_t height,
                                int32_t tile_size, int32_t early_termination,
                                double term_threshold, const void *exposure, void *out_color,
                                void *out_depth, void *out_transmittance, void *out_opacity,
                                int32_t *out_n_contrib, int32_t *out_last, void *out_y,
                                float *tile_depth_limit, int64_t *d_status,
                                float *coarse_depth_limit, int32_t *tile_sched, int64_t *halt,
                                int32_t fast_exp, void *stream)
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
        tile_depth_limit, d_status, coarse_depth_limit, order, replay, halt
    const int n_tiles = tiles_x * tiles_y;
    int32_t *order = nullptr, *replay = nullptr;
    if (tile_sched) {
        // [forward order | replay lengths | backward order]: this call orders
        // its tiles by the replay lengths the previous call with the same
        // schedule recorded (the list lengths are a poor estimate: a long
        // unsaturated sky list is cheap), then records the new ones
        order = tile_sched;
        replay = tile_sched + n_tiles;
        tile_order_kernel<<<1, kSchedThreads, 0, st>>>(nullptr, replay, n_tiles, order);
    }
    if (dtype == SB_F32) {
        if (ex && fast_exp) blend_fwd_kernel<float, true, true><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(float));
        else if (ex) blend_fwd_kernel<float, true><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(float));
        else if (fast_exp) blend_fwd_kernel<float, false, true><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(float));
        else blend_fwd_kernel<float, false><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(float));
    } else {
        if (ex) blend_fwd_kernel<double, true><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(double));
        else blend_fwd_kernel<double, false><<<tiles_x * tiles_y, kFwdThreads, 0, st>>>(FWD_ARGS(double));
    }
#undef FWD_ARGS
    return check_launch("blend_fwd_kernel");
}
