// loss_bwd.cu -- the gradient passes of K7 (ssim_backward loss.py:107-134,
// _conv_valid_adjoint 54-78, the L1 subgradient and the exposure chain,
// loss.py:143-177): B1 the transposed blur of the SSIM cotangent maps, B2
// the reflect-padding fold, L1 subgradient, d_rendered = dY M and the dE
// sums.  Their outputs are gradients (tolerance-checked), so this file is
// compiled with FMA contraction; the loss value comes from pass A in loss.cu.
#include "loss_common.cuh"

namespace sb {

// Pass B1: padded-grid adjoint of the separable blur, combined per channel.
template <typename T>
__global__ void __launch_bounds__(256) ssim_adjoint_kernel(int h, int w, const T *__restrict__ y,
                                                           const T *__restrict__ C,
                                                           const T *__restrict__ E,
                                                           const T *__restrict__ gt, LossK<T> K,
                                                           const T *__restrict__ maps,
                                                           T *__restrict__ vp)
{
    constexpr int HH = kLH + 2 * kPad, WW = kLW + 2 * kPad;  // rows pr0-10.., cols pc0-10..
    __shared__ T D[3][HH][WW];
    __shared__ T Ht[3][HH][kLW];
    const int hp = h + 2 * kPad, wp = w + 2 * kPad;
    const int pr0 = blockIdx.y * kLH, pc0 = blockIdx.x * kLW;
    const int64_t hw = (int64_t)h * w;
    for (int ch = 0; ch < 3; ++ch) {
        // dout rows [pr0-10, pr0+16) x cols [pc0-10, pc0+32), zero outside the image
        for (int t = threadIdx.x; t < HH * WW; t += blockDim.x) {
            const int rr = t / WW, cc = t - rr * WW;
            const int r = pr0 + rr - 2 * kPad, c = pc0 + cc - 2 * kPad;
            const bool in = r >= 0 && r < h && c >= 0 && c < w;
            const int64_t pix = (int64_t)r * w + c;
#pragma unroll
            for (int q = 0; q < 3; ++q) D[q][rr][cc] = in ? maps[(3 * ch + q) * hw + pix] : (T)0;
        }
        __syncthreads();
        // columns first (loss.py:72-74): dtmp[r][pc] = sum_b k[b] dout[r][pc-b]
        for (int t = threadIdx.x; t < HH * kLW; t += blockDim.x) {
            const int rr = t / kLW, cc = t - rr * kLW;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                T acc = 0;
#pragma unroll
                for (int b = 0; b < kWin; ++b) acc += K.k[b] * D[q][rr][cc + 2 * kPad - b];
                Ht[q][rr][cc] = acc;
            }
        }
        __syncthreads();
        // then rows (loss.py:76-77): dxp[pr][pc] = sum_a k[a] dtmp[pr-a][pc]
        for (int t = threadIdx.x; t < kLH * kLW; t += blockDim.x) {
            const int rr = t / kLW, cc = t - rr * kLW;
            const int pr = pr0 + rr, pc = pc0 + cc;
            if (pr >= hp || pc >= wp) continue;
            T ad[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                T acc = 0;
#pragma unroll
                for (int a = 0; a < kWin; ++a) acc += K.k[a] * Ht[q][rr + 2 * kPad - a][cc];
                ad[q] = acc;
            }
            const int sr = reflect_idx(pr - kPad, h), sc = reflect_idx(pc - kPad, w);
            const int64_t pix = (int64_t)sr * w + sc;
            const T xp = y_at(y, C, E, pix, ch), ypv = gt[3 * pix + ch];
            vp[((int64_t)ch * hp + pr) * wp + pc] = ad[0] + (T)2 * xp * ad[1] + ypv * ad[2];
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
        T dY[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            T fold = 0;
            for (int a = 0; a < nr; ++a)
                for (int b = 0; b < ncl; ++b) fold += vp[((int64_t)ch * hp + pr[a]) * wp + pc[b]];
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
