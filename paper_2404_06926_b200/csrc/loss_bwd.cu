// loss_bwd.cu -- the gradient passes of K7 (ssim_backward loss.py:107-134,
// _conv_valid_adjoint 54-78, the L1 subgradient and the exposure chain,
// loss.py:143-177): B1 the transposed blur of the SSIM cotangent maps, B2
// the reflect-padding fold, L1 subgradient, d_rendered = dY M and the dE
// sums.  Their outputs are gradients (tolerance-checked), so this file is
// compiled with FMA contraction; the loss value comes from pass A in loss.cu.
#include "loss_common.cuh"

namespace sb {

// Pass B1: padded-grid adjoint of the separable blur, combined per channel.
// Both passes slide a register window (as pass A): a thread owns a run of
// outputs along the pass direction and loads each input once; each output
// still adds its 11 taps in the same order.  The reflected source row and
// column of every output are computed once per CTA.
constexpr int kB1Run = 2;   // outputs per thread in both passes

template <typename T>
__global__ void __launch_bounds__(256) ssim_adjoint_kernel(int h, int w, const T *__restrict__ y,
                                                           const T *__restrict__ C,
                                                           const T *__restrict__ E,
                                                           const T *__restrict__ gt, LossK<T> K,
                                                           const T *__restrict__ maps,
                                                           T *__restrict__ vp)
{
    constexpr int HH = kLH + 2 * kPad, WW = kLW + 2 * kPad;  // rows pr0-10.., cols pc0-10..
    static_assert(kLW % kB1Run == 0 && kLH % kB1Run == 0, "runs must tile the block");
    constexpr int kCItems = HH * (kLW / kB1Run);   // column-pass work items
    constexpr int kRItems = (kLH / kB1Run) * kLW;  // row-pass work items
    constexpr int kTaps = kB1Run + kWin - 1;
    __shared__ T D[3][HH][WW];
    __shared__ T Ht[3][HH][kLW];
    __shared__ int s_sr[kLH], s_sc[kLW];
    const int hp = h + 2 * kPad, wp = w + 2 * kPad;
    const int pr0 = blockIdx.y * kLH, pc0 = blockIdx.x * kLW;
    const int64_t hw = (int64_t)h * w;
    if (threadIdx.x < kLH) s_sr[threadIdx.x] = reflect_idx(pr0 + (int)threadIdx.x - kPad, h);
    else if (threadIdx.x >= 32 && threadIdx.x < 32 + kLW)
        s_sc[threadIdx.x - 32] = reflect_idx(pc0 + (int)threadIdx.x - 32 - kPad, w);
    for (int ch = 0; ch < 3; ++ch) {
        // dout rows [pr0-10, pr0+16) x cols [pc0-10, pc0+32), zero outside the
        // image: every load of the thread's share issued before any store
        // (kDIters x 3 in flight; the halo load is the pass's latency)
        constexpr int kDIters = (HH * WW + 255) / 256;
        T dv[kDIters][3];
#pragma unroll
        for (int it = 0; it < kDIters; ++it) {
            const int t = threadIdx.x + it * 256;
            const int rr = t / WW, cc = t - rr * WW;
            const int r = pr0 + rr - 2 * kPad, c = pc0 + cc - 2 * kPad;
            const bool in = t < HH * WW && r >= 0 && r < h && c >= 0 && c < w;
            const int64_t pix = (int64_t)r * w + c;
#pragma unroll
            for (int q = 0; q < 3; ++q) dv[it][q] = in ? __ldg(maps + (3 * ch + q) * hw + pix) : (T)0;
        }
#pragma unroll
        for (int it = 0; it < kDIters; ++it) {
            const int t = threadIdx.x + it * 256;
            if (t >= HH * WW) continue;
            const int rr = t / WW, cc = t - rr * WW;
#pragma unroll
            for (int q = 0; q < 3; ++q) D[q][rr][cc] = dv[it][q];
        }
        __syncthreads();
        // columns first (loss.py:72-74): dtmp[r][pc] = sum_b k[b] dout[r][pc-b]
        for (int t = threadIdx.x; t < kCItems; t += blockDim.x) {
            const int rr = t / (kLW / kB1Run), cb = (t - rr * (kLW / kB1Run)) * kB1Run;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                // dout[rr][cb + o + 10 - b] for o < run, b < 11: columns cb .. cb + run + 9
                T v[kTaps];
#pragma unroll
                for (int i = 0; i < kTaps; ++i) v[i] = D[q][rr][cb + i];
#pragma unroll
                for (int o = 0; o < kB1Run; ++o) {
                    T acc = 0;
#pragma unroll
                    for (int b = 0; b < kWin; ++b) acc += K.k[b] * v[o + 2 * kPad - b];
                    Ht[q][rr][cb + o] = acc;
                }
            }
        }
        __syncthreads();
        // then rows (loss.py:76-77): dxp[pr][pc] = sum_a k[a] dtmp[pr-a][pc]
        for (int t = threadIdx.x; t < kRItems; t += blockDim.x) {
            const int g = t / kLW, cc = t - g * kLW, rb = g * kB1Run;
            T ad[kB1Run][3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                T v[kTaps];
#pragma unroll
                for (int i = 0; i < kTaps; ++i) v[i] = Ht[q][rb + i][cc];
#pragma unroll
                for (int o = 0; o < kB1Run; ++o) {
                    T acc = 0;
#pragma unroll
                    for (int a = 0; a < kWin; ++a) acc += K.k[a] * v[o + 2 * kPad - a];
                    ad[o][q] = acc;
                }
            }
            const int pc = pc0 + cc;
#pragma unroll
            for (int o = 0; o < kB1Run; ++o) {
                const int rr = rb + o, pr = pr0 + rr;
                if (pr >= hp || pc >= wp) continue;
                const int64_t pix = (int64_t)s_sr[rr] * w + s_sc[cc];
                const T xp = y_at(y, C, E, pix, ch), ypv = gt[3 * pix + ch];
                vp[((int64_t)ch * hp + pr) * wp + pc] =
                    ad[o][0] + (T)2 * xp * ad[o][1] + ypv * ad[o][2];
            }
        }
        __syncthreads();
    }
}

// fold positions of unpadded index i along an axis of length n, ascending
__device__ __forceinline__ int fold_set(int i, int n, int out[3])
{
    int k = 0;
    if (i >= 1 && i <= kPad) out[k++] = kPad - i;
    out[k++] = i + kPad;
    if (i >= n - 1 - kPad && i <= n - 2) out[k++] = kPad + 2 * (n - 1) - i;
    return k;
}

// Pass B2: fold + L1 + exposure chain + dE reduction
template <typename T>
__global__ void __launch_bounds__(256) loss_grad_kernel(int h, int w, const T *__restrict__ y,
                                                        const T *__restrict__ C,
                                                        const T *__restrict__ E,
                                                        const T *__restrict__ gt, LossK<T> K,
                                                        const T *__restrict__ vp,
                                                        T *__restrict__ d_rendered,
                                                        double *__restrict__ accum)
{
    __shared__ double red[8];
    const int hp = h + 2 * kPad, wp = w + 2 * kPad;
    const int64_t pix = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t hw = (int64_t)h * w;
    double part[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) part[q] = 0;
    if (pix < hw) {
        const int i = (int)(pix / w), j = (int)(pix - (int64_t)i * w);
        int pr[3], pc[3];
        const int nr = fold_set(i, h, pr), ncl = fold_set(j, w, pc);
        T dY[3], fl[3];
        if (nr == 1 && ncl == 1) {
            // interior pixels (all but a 5-pixel frame): one padded cell per
            // channel -- straight-line loads, all in flight at once
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) fl[ch] = vp[((int64_t)ch * hp + pr[0]) * wp + pc[0]];
        } else {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                T fold = 0;
                for (int a = 0; a < nr; ++a)
                    for (int b = 0; b < ncl; ++b) fold += vp[((int64_t)ch * hp + pr[a]) * wp + pc[b]];
                fl[ch] = fold;
            }
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const T fold = fl[ch];
            const T diff = y_at(y, C, E, pix, ch) - gt[3 * pix + ch];
            const T sg = diff > (T)0 ? (T)1 : (diff < (T)0 ? (T)-1 : (T)0);
            dY[ch] = K.one_m_lam * sg / K.n3 + fold;
        }
        const T *c = C + 3 * pix;
#pragma unroll
        for (int j2 = 0; j2 < 3; ++j2)
            d_rendered[3 * pix + j2] = rfma(dY[2], E[8 + j2], rfma(dY[1], E[4 + j2], dY[0] * E[j2]));
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
#pragma unroll
            for (int k = 0; k < 3; ++k) part[4 * ch + k] = (double)dY[ch] * (double)c[k];
            part[4 * ch + 3] = (double)dY[ch];
        }
    }
    // 12 block sums at once: warp shuffles, one barrier, 12 lanes finish
    __shared__ double wred[8][12];
#pragma unroll
    for (int q = 0; q < 12; ++q) {
        double v = part[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        part[q] = v;
    }
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int q = 0; q < 12; ++q) wred[wid][q] = part[q];
    }
    __syncthreads();
    if (threadIdx.x < 12) {
        double t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += wred[i][threadIdx.x];
        accum[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = t;   // quantity-major block partial (fixed-order tail)
    }
    (void)red;
}

template <typename T>
cudaError_t launch_loss_bwd(dim3 gB, unsigned gC, cudaStream_t st, int h, int w, const T *y,
                            const T *C, const T *E, const T *gt, const LossK<T> &K, T *maps,
                            T *vp, T *d_rendered, double *accum)
{
    ssim_adjoint_kernel<T><<<gB, 256, 0, st>>>(h, w, y, C, E, gt, K, maps, vp);
    loss_grad_kernel<T><<<gC, 256, 0, st>>>(h, w, y, C, E, gt, K, vp, d_rendered, accum);
    return cudaGetLastError();
}

template cudaError_t launch_loss_bwd<float>(dim3, unsigned, cudaStream_t, int, int, const float *,
                                            const float *, const float *, const float *,
                                            const LossK<float> &, float *, float *, float *,
                                            double *);
template cudaError_t launch_loss_bwd<double>(dim3, unsigned, cudaStream_t, int, int,
                                             const double *, const double *, const double *,
                                             const double *, const LossK<double> &, double *,
                                             double *, double *, double *);

}  // namespace sb
