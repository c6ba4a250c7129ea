// loss.cu -- K7 fused L1 + D-SSIM loss and its gradient, + K11 exposure Adam.
//
// photometric_loss loss.py:143-177; ssim_forward 81-104; ssim_backward 107-134;
// _conv_valid / _conv_valid_adjoint 54-78; apply_exposure 31-36;
// ScalarAdam.step adam.py:125-140.
//
// Three passes over the image, each a 2D tile per CTA with its halo in shared
// memory:
//   A  (stats):  11x11 separable Gaussian statistics of Y and gt on the
//      reflect-padded image (rows then columns, the reference's summation
//      order), per-pixel SSIM and the three SSIM cotangent maps
//      (d mu_x, d sigma_xx, d sigma_xy), block-reduced SSIM and L1 sums;
//   B1 (adjoint): the transposed blur of those maps (columns then rows) on
//      the padded grid, combined as A + 2 xp B + yp C (loss.py:128-130);
//   B2 (fold):   folds the reflect padding back (np.add.at order), adds the L1
//      subgradient, maps dY through the exposure (d_rendered = dY M) and
//      block-reduces dM = sum dY (x) C, db = sum dY in double.
// A one-CTA tail reduces the per-block partials in a fixed order (no float
// atomics: bitwise reproducible) into the loss parts; the f64 exposure
// Adam (ScalarAdam) is a separate one-thread kernel.
#include "loss_common.cuh"

namespace sb {

// the SSIM cotangent terms are gradients (tolerance-checked): a fast
// division there; the SSIM value itself keeps IEEE division (loss.py:98-100)
__device__ __forceinline__ float grad_div(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double grad_div(double a, double b) { return a / b; }

// Pass A.  Both separable passes slide a register window: a thread owns a
// run of outputs along the pass direction and loads each input once, so the
// shared-memory traffic per output drops from 11 loads per quantity to about
// 1 + 10 / run.  Each output still accumulates its 11 taps in the
// reference's order (k[0] term first, separate multiply and add: loss.py's
// numpy conv), so the values are unchanged.
constexpr int kVRun = 4;                    // rows per thread, vertical pass
constexpr int kHRun = 4;                    // columns per thread, horizontal pass (2: 60.9 us, 4: 55.9, 8: 93.0)

// The tile and its halo are loaded for all three channels at once (float;
// one channel at a time in double, to stay within 48 KB): the reflected
// source rows and columns are computed once per CTA, and each pixel's
// rendered colour is read once for its three exposed channels.
constexpr int kStatsThreads = 128;   // the horizontal pass's 16 x 8 items, one per thread

template <typename T>
__global__ void __launch_bounds__(kStatsThreads) ssim_stats_kernel(int h, int w, const T *__restrict__ y,
                                                         const T *__restrict__ C,
                                                         const T *__restrict__ E,
                                                         const T *__restrict__ gt, LossK<T> K,
                                                         T *__restrict__ maps,
                                                         double *__restrict__ accum)
{
    constexpr int HH = kLH + 2 * kPad, WW = kLW + 2 * kPad;
    constexpr int kCh = sizeof(T) == 4 ? 3 : 1;      // channels staged at once
    static_assert(kLH % kVRun == 0 && kLW % kHRun == 0, "runs must tile the block");
    constexpr int kVItems = (kLH / kVRun) * WW;      // vertical-pass work items
    constexpr int kHItems = kLH * (kLW / kHRun);     // horizontal-pass work items
    __shared__ T xs_all[kCh][HH][WW], ys_all[kCh][HH][WW];
    __shared__ T V[5][kLH][WW];
    __shared__ int s_sr[HH], s_sc[WW];
    const int r0 = blockIdx.y * kLH, c0 = blockIdx.x * kLW;
    const int64_t hw = (int64_t)h * w;
    if (threadIdx.x < HH) s_sr[threadIdx.x] = reflect_idx(r0 + (int)threadIdx.x - kPad, h);
    else if (threadIdx.x >= 64 && threadIdx.x < 64 + WW)
        s_sc[threadIdx.x - 64] = reflect_idx(c0 + (int)threadIdx.x - 64 - kPad, w);
    __syncthreads();
    double l1 = 0, ssum3[3];
    for (int ch = 0; ch < 3; ++ch) {
        const int cs = kCh == 3 ? ch : 0;            // staged slot of this channel
        if (kCh == 3 ? ch == 0 : true) {
            // the halo load is the pass's latency: all of a thread's loads
            // (its share of the tile, every channel) issued before any use
            constexpr int kLIters = (HH * WW + kStatsThreads - 1) / kStatsThreads;
            T xv[kLIters][kCh], yv[kLIters][kCh];
#pragma unroll
            for (int it = 0; it < kLIters; ++it) {
                const int t = threadIdx.x + it * kStatsThreads;
                const int tt = t < HH * WW ? t : 0;
                const int rr = tt / WW, cc = tt - rr * WW;
                const int64_t pix = (int64_t)s_sr[rr] * w + s_sc[cc];
#pragma unroll
                for (int k = 0; k < kCh; ++k) {
                    const int c = kCh == 3 ? k : ch;
                    xv[it][k] = y_at(y, C, E, pix, c);
                    yv[it][k] = gt[3 * pix + c];
                }
            }
#pragma unroll
            for (int it = 0; it < kLIters; ++it) {
                const int t = threadIdx.x + it * kStatsThreads;
                if (t >= HH * WW) continue;
                const int rr = t / WW, cc = t - rr * WW;
#pragma unroll
                for (int k = 0; k < kCh; ++k) {
                    xs_all[k][rr][cc] = xv[it][k];
                    ys_all[k][rr][cc] = yv[it][k];
                }
            }
            __syncthreads();
        }
        T (*xs)[WW] = xs_all[cs];
        T (*ys)[WW] = ys_all[cs];
        // rows first (loss.py:58-60): tmp[r][c] = sum_a k[a] * xp[r+a][c]
        for (int t = threadIdx.x; t < kVItems; t += blockDim.x) {
            const int g = t / WW, cc = t - g * WW, rb = g * kVRun;
            T xv[kVRun + kWin - 1], yv[kVRun + kWin - 1];
#pragma unroll
            for (int i = 0; i < kVRun + kWin - 1; ++i) {
                xv[i] = xs[rb + i][cc];
                yv[i] = ys[rb + i][cc];
            }
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                T val[kVRun + kWin - 1];
#pragma unroll
                for (int i = 0; i < kVRun + kWin - 1; ++i)
                    val[i] = q == 0 ? xv[i] : q == 1 ? yv[i] : q == 2 ? xv[i] * xv[i]
                             : q == 3 ? yv[i] * yv[i] : xv[i] * yv[i];
#pragma unroll
                for (int o = 0; o < kVRun; ++o) {
                    T acc = 0;
#pragma unroll
                    for (int a = 0; a < kWin; ++a) acc += K.k[a] * val[o + a];
                    V[q][rb + o][cc] = acc;
                }
            }
        }
        __syncthreads();
        double ssum = 0;
        for (int t = threadIdx.x; t < kHItems; t += blockDim.x) {
            const int rr = t / (kLW / kHRun), cb = (t - rr * (kLW / kHRun)) * kHRun;
            T m[5][kHRun];
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                T val[kHRun + kWin - 1];
#pragma unroll
                for (int i = 0; i < kHRun + kWin - 1; ++i) val[i] = V[q][rr][cb + i];
#pragma unroll
                for (int o = 0; o < kHRun; ++o) {
                    T acc = 0;
#pragma unroll
                    for (int b = 0; b < kWin; ++b) acc += K.k[b] * val[o + b];
                    m[q][o] = acc;
                }
            }
#pragma unroll
            for (int o = 0; o < kHRun; ++o) {
                const int cc = cb + o;
                const int r = r0 + rr, c = c0 + cc;
                if (r >= h || c >= w) continue;
                const T mx = m[0][o], my = m[1][o];
                const T vxx = m[2][o] - mx * mx, vyy = m[3][o] - my * my, vxy = m[4][o] - mx * my;
                const T two = (T)2;
                const T a1 = two * mx * my + K.c1, a2 = two * vxy + K.c2;
                const T b1 = mx * mx + my * my + K.c1, b2 = vxx + vyy + K.c2;
                const T s = (a1 * a2) / (b1 * b2);
                ssum += (double)s;
                const T denom = b1 * b2;
                const T da1 = grad_div(K.coeff * a2, denom), da2 = grad_div(K.coeff * a1, denom);
                const T db1 = grad_div(-K.coeff * s, b1), db2 = grad_div(-K.coeff * s, b2);
                T dmx = two * my * da1 + two * mx * db1;
                const T dvxy = two * da2, dvxx = db2;
                dmx += (T)(-2) * mx * dvxx - my * dvxy;
                const int64_t pix = (int64_t)r * w + c;
                maps[(3 * ch + 0) * hw + pix] = dmx;
                maps[(3 * ch + 1) * hw + pix] = dvxx;
                maps[(3 * ch + 2) * hw + pix] = dvxy;
                const T diff = xs[rr + kPad][cc + kPad] - ys[rr + kPad][cc + kPad];
                l1 += fabs((double)diff);
            }
        }
        ssum3[ch] = ssum;
        __syncthreads();
    }
    // the four block sums at once: warp shuffles, one barrier, 4 lanes finish
    __shared__ double wred[kStatsThreads / 32][4];
    double part[4] = {ssum3[0], ssum3[1], ssum3[2], l1};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) wred[threadIdx.x >> 5][q] = part[q];
    }
    __syncthreads();
    // per-block partial sums, reduced in a fixed order by the tail (no
    // float atomics: the loss and dE are bitwise reproducible)
    if (threadIdx.x < 4) {
        double t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += wred[i][threadIdx.x];
        const int64_t nb = (int64_t)gridDim.x * gridDim.y;   // quantity-major partials
        accum[threadIdx.x * nb + (int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// E is 3x4 [M|b]; the d_rendered mapping needs M as matrix rows: E[4c + j]
// is M[c][j].  (In loss_grad_kernel E[j2], E[4+j2], E[8+j2] = M[0..2][j2].)

// The block partials of passes A (4 sums) and B2 (12 sums), stored
// quantity-major, reduced in a fixed order: one CTA per sum, thread t adds
// blocks t, t + 256, ... (coalesced, 16 loads in flight) into 4 chains, then
// fixed warp butterflies and a fixed sum over the warps -- deterministic,
// unlike float atomics.  The last CTA to finish (a ticket; which CTA that is
// does not change any value) turns the 16 sums into the loss parts
// (loss.py:170-172).
constexpr int kTailThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kTailThreads) loss_tail_kernel(
    int h, int w, LossK<T> K, const double *__restrict__ partA, int nA,
    const double *__restrict__ partC, int nC, double *__restrict__ accum,
    double *__restrict__ parts, double *__restrict__ d_exposure, unsigned *__restrict__ ticket)
{
    __shared__ double wsum[kTailThreads / 32];
    __shared__ bool last;
    const int q = blockIdx.x;
    const double *src = q < 4 ? partA + (int64_t)q * nA : partC + (int64_t)(q - 4) * nC;
    const int nb = q < 4 ? nA : nC;
    double t[4] = {0, 0, 0, 0};
    for (int b0 = 0; b0 < nb; b0 += kTailThreads * 16) {
        double x[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int b = b0 + kTailThreads * k + threadIdx.x;
            x[k] = b < nb ? __ldg(src + b) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) t[k & 3] += x[k];
    }
    double v = (t[0] + t[1]) + (t[2] + t[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0;
        for (int i = 0; i < kTailThreads / 32; ++i) tot += wsum[i];
        accum[q] = tot;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    const volatile double *sums = accum;
    const double npx = (double)h * w;
    const T l1 = (T)(sums[3] / (3.0 * npx));
    const T ssim = (T)((sums[0] / npx + sums[1] / npx + sums[2] / npx) / 3.0);
    const T dssim = ((T)1 - ssim) / (T)2;
    const T loss = K.one_m_lam * l1 + K.lam * dssim;
    parts[0] = loss; parts[1] = l1; parts[2] = dssim; parts[3] = ssim;
    for (int k = 0; k < 12; ++k) d_exposure[k] = (double)(T)sums[4 + k];
}

// K11: ScalarAdam.step in float64 (adam.py:134-140)
template <typename T>
__global__ void exposure_adam_kernel(double *__restrict__ E, T *__restrict__ E_real,
                                     const double *__restrict__ g, double *__restrict__ st,
                                     double lr, const int64_t *__restrict__ status)
{
    if (status && status[1]) return;
    const int q = threadIdx.x;
    double t = st[24] + 1.0;
    __syncthreads();
    if (q < 12) {
        const double b1 = 0.9, b2 = 0.999;
        const double m = b1 * st[q] + (1 - b1) * g[q];
        const double v = b2 * st[12 + q] + (1 - b2) * g[q] * g[q];
        st[q] = m;
        st[12 + q] = v;
        const double mh = m / (1 - pow(b1, t));
        const double vh = v / (1 - pow(b2, t));
        E[q] = E[q] - lr * mh / (sqrt(vh) + 1e-15);
        if (E_real) E_real[q] = (T)E[q];
    }
    __syncthreads();
    if (q == 0) st[24] = t;
}

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <typename T>
static LossK<T> make_loss_k(int h, int w, double lam)
{
    LossK<T> K;
    double kd[kWin], s = 0;
    for (int i = 0; i < kWin; ++i) {
        const double x = (double)(i - kPad);
        kd[i] = std::exp(-(x * x) / (2.0 * 1.5 * 1.5));
        s += kd[i];
    }
    for (int i = 0; i < kWin; ++i) K.k[i] = (T)(kd[i] / s);
    K.c1 = (T)(0.01 * 0.01);
    K.c2 = (T)(0.03 * 0.03);
    const T lamT = (T)lam;
    K.lam = lamT;
    K.one_m_lam = (T)1 - lamT;
    // coeff = f(-float(lam)/2) / f(3 h w) (loss.py:114, 170)
    const T num = (T)(-(double)lamT / 2.0);
    const T den = (T)(3.0 * h * w);
    K.coeff = num / den;
    K.n3 = (T)((double)h * w * 3);
    return K;
}

}  // namespace sb

using namespace sb;

// workspace: [16 final sums | pass-A block partials (4 per block) | pass-B2
// block partials (12 per block) | 9 cotangent maps | padded adjoint image]
struct LossLayout {
    dim3 gA, gB;
    unsigned gC;
    int nA, nC;
    size_t partA, partC, maps, vp, bytes;
};

static LossLayout loss_layout(int32_t width, int32_t height)
{
    LossLayout L;
    const int h = height, w = width;
    L.gA = dim3((w + kLW - 1) / kLW, (h + kLH - 1) / kLH);
    L.gB = dim3((w + 2 * kPad + kLW - 1) / kLW, (h + 2 * kPad + kLH - 1) / kLH);
    L.gC = grid_for((int64_t)h * w, 256);
    L.nA = (int)(L.gA.x * L.gA.y);
    L.nC = (int)L.gC;
    const size_t hw = (size_t)w * h;
    const size_t hwp = (size_t)(w + 2 * kPad) * (h + 2 * kPad);
    size_t o = align256(17 * sizeof(double));
    L.partA = o; o += align256(4 * (size_t)L.nA * sizeof(double));
    L.partC = o; o += align256(12 * (size_t)L.nC * sizeof(double));
    L.maps = o; o += align256(9 * hw * sizeof(double));
    L.vp = o; o += align256(3 * hwp * sizeof(double));
    L.bytes = o;
    return L;
}

extern "C" size_t sb_loss_workspace_bytes(int32_t width, int32_t height)
{
    return loss_layout(width, height).bytes;
}

extern "C" int32_t sb_loss_fused(int32_t dtype, int32_t width, int32_t height,
                                 const void *rendered, const void *y, const void *ground_truth,
                                 const void *exposure, double lam, void *d_rendered,
                                 double *d_exposure, double *parts, void *workspace,
                                 size_t workspace_bytes, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(width >= 6 && height >= 6, "loss needs H, W >= 6 (got %dx%d)", width, height);
    SB_REQUIRE(exposure != nullptr, "exposure is NULL (pass identity)");
    SB_REQUIRE(workspace_bytes >= sb_loss_workspace_bytes(width, height), "loss workspace too small");
    cudaStream_t st = as_stream(stream);
    const int h = height, w = width;
    const LossLayout L = loss_layout(width, height);
    char *ws = (char *)workspace;
    double *accum = (double *)ws;                 // [16] final sums + the tail's ticket
    unsigned *ticket = (unsigned *)(accum + 16);
    double *partA = (double *)(ws + L.partA), *partC = (double *)(ws + L.partC);
    void *maps = ws + L.maps;
    void *vp = ws + L.vp;
    SB_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st));
#define LOSS_LAUNCH(T)                                                                         \
    {                                                                                          \
        const LossK<T> K = make_loss_k<T>(h, w, lam);                                          \
        ssim_stats_kernel<T><<<L.gA, kStatsThreads, 0, st>>>(h, w, (const T *)y, (const T *)rendered,    \
                                                (const T *)exposure, (const T *)ground_truth, K, \
                                                (T *)maps, partA);                             \
        SB_CUDA(launch_loss_bwd<T>(L.gB, L.gC, st, h, w, (const T *)y, (const T *)rendered,    \
                                   (const T *)exposure, (const T *)ground_truth, K,             \
                                   (T *)maps, (T *)vp, (T *)d_rendered, partC));                \
        loss_tail_kernel<T><<<16, kTailThreads, 0, st>>>(h, w, K, partA, L.nA, partC, L.nC,   \
                                                         accum, parts, d_exposure, ticket);    \
    }
    if (dtype == SB_F32) LOSS_LAUNCH(float)
    else LOSS_LAUNCH(double)
#undef LOSS_LAUNCH
    return check_launch("loss kernels");
}

extern "C" int32_t sb_exposure_adam(int32_t dtype, double *exposure, void *exposure_real,
                                    const double *d_exposure, double *state, double lr,
                                    const int64_t *d_status, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    cudaStream_t st = as_stream(stream);
    if (dtype == SB_F32)
        exposure_adam_kernel<float><<<1, 32, 0, st>>>(exposure, (float *)exposure_real, d_exposure, state, lr, d_status);
    else
        exposure_adam_kernel<double><<<1, 32, 0, st>>>(exposure, (double *)exposure_real, d_exposure, state, lr, d_status);
    return check_launch("exposure_adam_kernel");
}

// apply_exposure (loss.py:31-36) as a standalone op: out = C M^T + b
namespace sb {
template <typename T>
__global__ void apply_exposure_kernel(int64_t npx, const T *__restrict__ C, const T *__restrict__ E,
                                      T *__restrict__ out)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= npx) return;
#pragma unroll
    for (int c = 0; c < 3; ++c) out[3 * p + c] = y_at<T>(nullptr, C, E, p, c);
}

// psnr_8bit (metrics.py:16-27) of clip(exposure(C)) against an 8-bit target:
// accumulates the integer squared error into sse (uint64, caller-zeroed).
template <typename T>
__global__ void psnr8_kernel(int64_t npx, const T *__restrict__ C, const T *__restrict__ E,
                             const uint8_t *__restrict__ gt8, unsigned long long *__restrict__ sse)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long e = 0;
    if (p < npx) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            T v = y_at<T>(nullptr, C, E, p, c);
            v = v < (T)0 ? (T)0 : (v > (T)1 ? (T)1 : v);
            const T s = v * (T)255.0;
            const int q = (int)rint((double)s);   // np.round: half to even
            const int d = q - (int)gt8[3 * p + c];
            e += (unsigned long long)(d * d);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    // one atomic per block, not per warp (~29k warps on one address)
    __shared__ unsigned long long s_e[8];
    if ((threadIdx.x & 31) == 0) s_e[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_e[w];
        if (t) atomicAdd(sse, t);
    }
}
}  // namespace sb

extern "C" int32_t sb_apply_exposure(int32_t dtype, int64_t npx, const void *color,
                                     const void *exposure, void *out, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    if (npx == 0) return SB_OK;
    const unsigned g = grid_for(npx, 256);
    if (dtype == SB_F32)
        apply_exposure_kernel<float><<<g, 256, 0, as_stream(stream)>>>(npx, (const float *)color, (const float *)exposure, (float *)out);
    else
        apply_exposure_kernel<double><<<g, 256, 0, as_stream(stream)>>>(npx, (const double *)color, (const double *)exposure, (double *)out);
    return check_launch("apply_exposure_kernel");
}

extern "C" int32_t sb_psnr8_sse(int32_t dtype, int64_t npx, const void *color, const void *exposure,
                                const uint8_t *gt8, unsigned long long *sse, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    if (npx == 0) return SB_OK;
    const unsigned g = grid_for(npx, 256);
    if (dtype == SB_F32)
        psnr8_kernel<float><<<g, 256, 0, as_stream(stream)>>>(npx, (const float *)color, (const float *)exposure, gt8, sse);
    else
        psnr8_kernel<double><<<g, 256, 0, as_stream(stream)>>>(npx, (const double *)color, (const double *)exposure, gt8, sse);
    return check_launch("psnr8_kernel");
}

// quantize_8bit (metrics.py:12-13) of a float image, in double like numpy:
// clip to [0, 1], * 255, round half to even
namespace sb {
template <typename T>
__global__ void quantize8_kernel(int64_t n, const T *__restrict__ x, uint8_t *__restrict__ q)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = fmin(fmax((double)x[i], 0.0), 1.0);
    q[i] = (uint8_t)rint(v * 255.0);
}
}  // namespace sb

extern "C" int32_t sb_quantize8(int32_t dtype, int64_t n, const void *src, uint8_t *dst,
                                void *stream)
{
    SB_DTYPE_CHECK(dtype);
    if (n == 0) return SB_OK;
    const unsigned g = grid_for(n, 256);
    if (dtype == SB_F32)
        quantize8_kernel<float><<<g, 256, 0, as_stream(stream)>>>(n, (const float *)src, dst);
    else
        quantize8_kernel<double><<<g, 256, 0, as_stream(stream)>>>(n, (const double *)src, dst);
    return check_launch("quantize8_kernel");
}

extern "C" int32_t sb_memset_async(void *ptr, int32_t value, size_t bytes, void *stream)
{
    if (bytes == 0) return SB_OK;
    SB_CUDA(cudaMemsetAsync(ptr, value, bytes, as_stream(stream)));
    return SB_OK;
}
