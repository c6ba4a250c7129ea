// loss_common.cuh -- tile geometry, constants and helpers shared by the loss
// value pass (loss.cu, exact arithmetic) and its gradient passes
// (loss_bwd.cu, compiled with FMA contraction).
#pragma once

#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

constexpr int kLW = 32, kLH = 16, kPad = 5, kWin = 11;

template <typename T>
struct LossK {
    T k[kWin];
    T c1, c2, coeff, lam, one_m_lam, n3;
};

__device__ __forceinline__ int reflect_idx(int p, int n)
{
    while (p < 0 || p >= n) {
        if (p < 0) p = -p;
        if (p >= n) p = 2 * (n - 1) - p;
    }
    return p;
}

template <typename T>
__device__ __forceinline__ T y_at(const T *__restrict__ y, const T *__restrict__ C,
                                  const T *__restrict__ E, int64_t pix, int ch)
{
    if (y) return y[3 * pix + ch];
    const T *c = C + 3 * pix;
    return rfma(c[2], E[4 * ch + 2], rfma(c[1], E[4 * ch + 1], c[0] * E[4 * ch])) + E[4 * ch + 3];
}

template <typename T>
__device__ __forceinline__ double block_sum(double v, double *red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    return t;  // valid on thread 0
}


// passes B1 + B2 (loss_bwd.cu)
template <typename T>
cudaError_t launch_loss_bwd(dim3 gB, unsigned gC, cudaStream_t st, int h, int w, const T *y,
                            const T *C, const T *E, const T *gt, const LossK<T> &K, T *maps,
                            T *vp, T *d_rendered, double *accum);

}  // namespace sb
