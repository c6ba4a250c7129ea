// blend.cu -- K6 forward blend and K8 backward blend.
//
// a4 _composite_tiles, forward.py:261-342 (+ exposure epilogue, loss.py:31-36)
// a6 _backward_tiles,  backward.py:91-213
//
// One CTA per 16x16 tile, one thread per pixel.  The tile's depth-ordered pair
// list is walked in batches of 256 splat records staged in shared memory (one
// coalesced record load per thread), so each record is read from L2/HBM once
// per tile.  A pixel stops when T < 1e-4 (checked BEFORE each Gaussian, like
// the reference: the Gaussian that drives T below the threshold is still
// composited); a warp skips work once all its pixels are done and the CTA
// leaves the list once all 256 are (__syncthreads_count).
//
// The forward records, per pixel, 1 + the list position of its last
// contributor; the backward replays the tile only up to the max of that over
// the tile (P_proc in SURVEY §8), front to back with the same float operations
// as the forward, so its transmittance/prefix state is bit-identical.  Per
// Gaussian, the 9 screen-space adjoints of the 32 pixels of a warp are reduced
// with shuffles, combined across the CTA's 8 warps in shared memory, and
// pushed to global memory with one atomic per (tile, Gaussian, value).
#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

constexpr int kBatch = kTilePx;  // 256 records per shared-memory batch

template <typename T>
struct SmemSplat {
    T mx, my, a, b, c, opa, qc, c0, c1, c2, dep;
    T bx0, bx1, by0, by1;  // pixel box [ceil(m - r), floor(m + r)] (forward.py:296-299)
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

template <typename T, bool kExposure>
__global__ void __launch_bounds__(kTilePx) blend_fwd_kernel(
    const T *__restrict__ records, const int32_t *__restrict__ pair_gaussian,
    const int32_t *__restrict__ offsets, int width, int height, int tiles_x, int early,
    T thresh, const T *__restrict__ expo, T *__restrict__ out_c, T *__restrict__ out_d,
    T *__restrict__ out_t, T *__restrict__ out_o, int32_t *__restrict__ out_nc,
    int32_t *__restrict__ out_last, T *__restrict__ out_y)
{
    __shared__ SmemSplat<T> sm[kBatch];
    const int tile = blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x >> 4;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < width && py < height;
    const T fpx = (T)px, fpy = (T)py;
    const int lo = offsets[tile], hi = offsets[tile + 1];

    const T one = (T)1, half = one / (T)2, two = one + one;
    const T clamp = (T)kAlphaClamp, cutoff = (T)kAlphaCutoff;
    T Tr = one, C0 = (T)0, C1 = (T)0, C2 = (T)0, D = (T)0;
    int32_t nc = 0, last = 0;
    bool done = !inside || (early && Tr < thresh);

    for (int base = lo; base < hi; base += kBatch) {
        if (__syncthreads_count(!done) == 0) break;
        const int k = base + threadIdx.x;
        if (k < hi) {
            T rec[12];
            load_record(records, pair_gaussian[k], rec);
            stage(sm[threadIdx.x], rec);
        }
        __syncthreads();
        const int nb = min(kBatch, hi - base);
        for (int j = 0; j < nb && !done; ++j) {
            const SmemSplat<T> &s = sm[j];
            if (fpx < s.bx0 || fpx > s.bx1 || fpy < s.by0 || fpy > s.by1) continue;
            const T dy = fpy - s.my;
            const T qy = s.c * dy * dy;
            const T bdy = two * s.b * dy;
            const T dx = fpx - s.mx;
            const T q = s.a * dx * dx + bdy * dx + qy;
            if (q > s.qc) continue;
            T alpha = s.opa * rexp(-(half * q));
            if (alpha > clamp) alpha = clamp;
            if (alpha < cutoff) continue;
            const T w = alpha * Tr;
            C0 += w * s.c0;
            C1 += w * s.c1;
            C2 += w * s.c2;
            D += w * s.dep;
            nc += 1;
            last = base + j - lo + 1;
            Tr = Tr * (one - alpha);
            // termination is tested before the next Gaussian (forward.py:310)
            if (early && Tr < thresh) done = true;
        }
    }
    if (!inside) return;
    const int64_t pix = (int64_t)py * width + px;
    out_c[3 * pix] = C0;
    out_c[3 * pix + 1] = C1;
    out_c[3 * pix + 2] = C2;
    out_d[pix] = D;
    out_t[pix] = Tr;
    if (out_o) out_o[pix] = one - Tr;
    out_nc[pix] = nc;
    if (out_last) out_last[pix] = last;
    if (kExposure) {
        // Y = C M^T + b (loss.py:157-158, BLAS FMA chain)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            out_y[3 * pix + c] =
                rfma(C2, expo[4 * c + 2], rfma(C1, expo[4 * c + 1], C0 * expo[4 * c])) + expo[4 * c + 3];
    }
}

// Reduce 9 per-lane values across the warp with 12 shuffles instead of 45:
// at each butterfly level a lane keeps half of its values and receives the
// partner's copy of that half (a transpose-reduce).  Returns the index (0..8)
// of the fully reduced value this lane ends up holding, or -1 (odd lanes and
// padding slots).
template <typename T>
__device__ __forceinline__ int warp_reduce9(const T g[9], T &out)
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
    out = d;
    int local;
    if (b3) local = b2 ? -1 : 3 + (int)b1;
    else local = (2 * (int)b2 + (int)b1) <= 2 ? 2 * (int)b2 + (int)b1 : -1;
    if (lane & 1) return -1;
    if (b4) return (local >= 0 && local <= 3) ? 5 + local : -1;
    return (local >= 0 && local <= 4) ? local : -1;
}

template <typename T>
__global__ void __launch_bounds__(kTilePx) blend_bwd_kernel(
    const T *__restrict__ records, const int32_t *__restrict__ pair_gaussian,
    const int32_t *__restrict__ offsets, int width, int height, int tiles_x, int early,
    T thresh, const T *__restrict__ dC_img, const T *__restrict__ cfinal,
    const int32_t *__restrict__ last_img, T *__restrict__ d_mean, T *__restrict__ d_conic,
    T *__restrict__ d_op, T *__restrict__ d_col)
{
    constexpr int B = sizeof(T) == 4 ? kBatch : kBatch / 2;  // fits 48 KB static smem
    __shared__ SmemSplat<T> sm[B];
    __shared__ int32_t srow[B];
    __shared__ T acc[B][9];
    __shared__ int s_end;
    const int tile = blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x >> 4;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < width && py < height;
    const T fpx = (T)px, fpy = (T)py;
    const int lo = offsets[tile], hi = offsets[tile + 1];
    const T one = (T)1, half = one / (T)2, two = one + one;
    const T clamp = (T)kAlphaClamp, cutoff = (T)kAlphaCutoff;
    T dc0 = 0, dc1 = 0, dc2 = 0, cf0 = 0, cf1 = 0, cf2 = 0;
    int my_end = 0;
    if (inside) {
        const int64_t pix = (int64_t)py * width + px;
        dc0 = dC_img[3 * pix]; dc1 = dC_img[3 * pix + 1]; dc2 = dC_img[3 * pix + 2];
        cf0 = cfinal[3 * pix]; cf1 = cfinal[3 * pix + 1]; cf2 = cfinal[3 * pix + 2];
        my_end = last_img ? last_img[pix] : hi - lo;
    }
    if (threadIdx.x == 0) s_end = 0;
    __syncthreads();
    if (my_end > 0) atomicMax(&s_end, my_end);
    __syncthreads();
    const int end = lo + s_end;
    T Tr = one, P0 = 0, P1 = 0, P2 = 0;
    bool done = !inside || my_end == 0 || (early && Tr < thresh);

    for (int base = lo; base < end; base += B) {
        const int k = base + threadIdx.x;
        if (threadIdx.x < B) {
            if (k < end) {
                T rec[12];
                const int row = pair_gaussian[k];
                load_record(records, row, rec);
                stage(sm[threadIdx.x], rec);
                srow[threadIdx.x] = row;
            }
#pragma unroll
            for (int v = 0; v < 9; ++v) acc[threadIdx.x][v] = (T)0;
        }
        __syncthreads();
        const int nb = min(B, end - base);
        for (int j = 0; j < nb; ++j) {
            if (__all_sync(0xffffffffu, done)) break;  // warp-uniform
            const SmemSplat<T> &s = sm[j];
            T g[9];
            bool contrib = false;
            if (!done && base + j - lo < my_end && !(fpx < s.bx0 || fpx > s.bx1 || fpy < s.by0 || fpy > s.by1)) {
                {
                    const T dy = fpy - s.my;
                    const T qy = s.c * dy * dy;
                    const T bdy = two * s.b * dy;
                    const T dx = fpx - s.mx;
                    const T q = s.a * dx * dx + bdy * dx + qy;
                    if (q <= s.qc) {
                        const T gauss = rexp(-(half * q));
                        const T alpha_raw = s.opa * gauss;
                        T alpha = alpha_raw;
                        if (alpha > clamp) alpha = clamp;
                        if (alpha >= cutoff) {
                            contrib = true;
                            const T w = alpha * Tr;
                            const T p0 = P0 + w * s.c0;
                            const T p1 = P1 + w * s.c1;
                            const T p2 = P2 + w * s.c2;
                            g[6] = w * dc0; g[7] = w * dc1; g[8] = w * dc2;
                            if (alpha_raw < clamp) {
                                const T inv_rest = one / (one - alpha);
                                const T dalpha = (dc0 * (s.c0 * Tr - (cf0 - p0) * inv_rest)
                                                  + dc1 * (s.c1 * Tr - (cf1 - p1) * inv_rest)
                                                  + dc2 * (s.c2 * Tr - (cf2 - p2) * inv_rest));
                                g[5] = dalpha * gauss;
                                const T dq = -(half * gauss * (dalpha * s.opa));
                                g[0] = -(two * dq * (s.a * dx + s.b * dy));
                                g[1] = -(two * dq * (s.b * dx + s.c * dy));
                                g[2] = dq * dx * dx;
                                g[3] = dq * dx * dy;
                                g[4] = dq * dy * dy;
                            } else {
                                g[0] = g[1] = g[2] = g[3] = g[4] = g[5] = (T)0;
                            }
                            P0 = p0; P1 = p1; P2 = p2;
                            Tr = Tr * (one - alpha);
                            if (early && Tr < thresh) done = true;
                        }
                    }
                }
            }
            const unsigned any = __ballot_sync(0xffffffffu, contrib);
            if (any) {
                if (!contrib) {
#pragma unroll
                    for (int v = 0; v < 9; ++v) g[v] = (T)0;
                }
                T red;
                const int idx = warp_reduce9(g, red);
                if (idx >= 0) atomicAdd(&acc[j][idx], red);
            }
        }
        __syncthreads();
        if (threadIdx.x < nb) {
            const int row = srow[threadIdx.x];
            const T *a = acc[threadIdx.x];
            bool nz = false;
#pragma unroll
            for (int v = 0; v < 9; ++v) nz |= a[v] != (T)0;
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
                                void *stream)
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
        (T *)out_transmittance, (T *)out_opacity, out_n_contrib, out_last, (T *)out_y
    if (dtype == SB_F32) {
        if (ex) blend_fwd_kernel<float, true><<<tiles_x * tiles_y, kTilePx, 0, st>>>(FWD_ARGS(float));
        else blend_fwd_kernel<float, false><<<tiles_x * tiles_y, kTilePx, 0, st>>>(FWD_ARGS(float));
    } else {
        if (ex) blend_fwd_kernel<double, true><<<tiles_x * tiles_y, kTilePx, 0, st>>>(FWD_ARGS(double));
        else blend_fwd_kernel<double, false><<<tiles_x * tiles_y, kTilePx, 0, st>>>(FWD_ARGS(double));
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
    if (dtype == SB_F32) blend_bwd_kernel<float><<<tiles_x * tiles_y, kTilePx, 0, st>>>(BWD_ARGS(float));
    else blend_bwd_kernel<double><<<tiles_x * tiles_y, kTilePx, 0, st>>>(BWD_ARGS(double));
#undef BWD_ARGS
    return check_launch("blend_bwd_kernel");
}
