// blend_common.cuh -- pieces shared by the forward (blend.cu) and backward
// (blend_bwd.cu) blends: the staged splat record and the forward's exp.
#pragma once

#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

// exp(x) for the blend's range (x = -q/2 with 0 <= q <= q_cut + 1/64 <
// 2 ln 255 + 1/64, so -5.6 < x <= ~0), in double, then ONE rounding to float
// -- correctly rounded except with probability ~2^-27 per evaluation, like
// the (float)exp((double)x) of the oracle.  Table-driven: x = (32 m + j) ln2/32
// + r with |r| <= ln2/64, exp(x) = 2^m 2^(j/32) e^r; the 2^(j/32) are
// correctly rounded doubles (shared-memory copy, see kExp2Tab), e^r - 1 a
// degree-6 polynomial (truncation 3.5e-18) evaluated with depth 4.
__constant__ double kExp2Tab[32] = {
    0x1.0000000000000p+0,
    0x1.059b0d3158574p+0,
    0x1.0b5586cf9890fp+0,
    0x1.11301d0125b51p+0,
    0x1.172b83c7d517bp+0,
    0x1.1d4873168b9aap+0,
    0x1.2387a6e756238p+0,
    0x1.29e9df51fdee1p+0,
    0x1.306fe0a31b715p+0,
    0x1.371a7373aa9cbp+0,
    0x1.3dea64c123422p+0,
    0x1.44e086061892dp+0,
    0x1.4bfdad5362a27p+0,
    0x1.5342b569d4f82p+0,
    0x1.5ab07dd485429p+0,
    0x1.6247eb03a5585p+0,
    0x1.6a09e667f3bcdp+0,
    0x1.71f75e8ec5f74p+0,
    0x1.7a11473eb0187p+0,
    0x1.82589994cce13p+0,
    0x1.8ace5422aa0dbp+0,
    0x1.93737b0cdc5e5p+0,
    0x1.9c49182a3f090p+0,
    0x1.a5503b23e255dp+0,
    0x1.ae89f995ad3adp+0,
    0x1.b7f76f2fb5e47p+0,
    0x1.c199bdd85529cp+0,
    0x1.cb720dcef9069p+0,
    0x1.d5818dcfba487p+0,
    0x1.dfc97337b9b5fp+0,
    0x1.ea4afa2a490dap+0,
    0x1.f50765b6e4540p+0
};

__device__ __forceinline__ float blend_exp(float xf, const double *__restrict__ tab)
{
    const double x = (double)xf;
    const double nd = rint(x * 0x1.71547652b82fep+5);              // x 32 / ln 2
    const int n = (int)nd;
    const int j = n & 31, m = n >> 5;                                // n = 32 m + j
    // ln2/32 = HI + LO, HI with 33 significant bits: nd HI is exact, so is x - nd HI
    const double r = __fma_rn(-nd, 0x1.473de6af278edp-39, __fma_rn(-nd, 0x1.62e42fef00000p-6, x));
    const double r2 = r * r;
    const double q = __fma_rn(r2, __fma_rn(r2, 1.0 / 720.0, __fma_rn(r, 1.0 / 120.0, 1.0 / 24.0)),
                              __fma_rn(r, 1.0 / 6.0, 0.5));
    const double p = __fma_rn(r2, q, r);                             // e^r - 1
    const double t = tab[j];
    const double y = __fma_rn(t, p, t);
    return (float)(y * __longlong_as_double((long long)(m + 1023) << 52));
}

__device__ __forceinline__ double blend_exp(double x, const double *) { return exp(x); }

// 16 reals, 16-byte aligned: a thread copies a staged record into registers
// with four 128-bit shared loads per Gaussian
template <typename T>
struct __align__(16) SmemSplat {
    T mx, my, a, b, c, opa, qc, c0, c1, c2, dep;
    T bx0, bx1, by0, by1;  // pixel box [ceil(m - r), floor(m + r)] (forward.py:296-299)
    T pad;
};

// The mapping step's Mahalanobis form and Gaussian weight, shared bit for
// bit by its forward (sb_blend_fwd fast_exp) and the backward's replay
// (blend_bwd.cu): explicit no-contraction intrinsics, so both translation
// units (compiled with and without -fmad) evaluate exactly the same
// operations and take the same cutoff, clamp and termination decisions.  q
// is the reference's own operation sequence (forward.py:283-286,
// left-to-right, no FMA): bit-identical to it; only the exp differs.
__device__ __forceinline__ float step_q(const SmemSplat<float> &s, float dx, float dy)
{
    const float qy = __fmul_rn(__fmul_rn(s.c, dy), dy);
    const float bdy = __fmul_rn(__fmul_rn(2.0f, s.b), dy);
    return __fadd_rn(__fadd_rn(__fmul_rn(__fmul_rn(s.a, dx), dx), __fmul_rn(bdy, dx)), qy);
}

__device__ __forceinline__ float step_gauss(float q) { return __expf(__fmul_rn(-0.5f, q)); }

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

// Heavy-first tile schedule.  The blends launch one CTA per tile and the
// hardware dispatches CTAs in blockIdx order; tiles differ in cost by two
// orders of magnitude (sky vs foreground) and row-major order puts the
// heaviest (lower, foreground) rows last, into the final partial wave.  This
// single-CTA kernel orders the tiles by a cost estimate, descending, with a
// 64-bucket counting sort (log2 with one fractional bit); the order within
// a bucket is arbitrary (each tile's result does not depend on it).
//   cost[t]: a per-tile replay length recorded by the forward (the
//   previous iteration's for the forward itself, this iteration's for the
//   backward), or, without one, offsets[t+1] - offsets[t].
constexpr int kSchedThreads = 1024;

__device__ __forceinline__ int sched_bucket(int c)
{
    if (c <= 0) return 0;
    const int lg = 31 - __clz(c);                    // floor(log2 c)
    const int half = lg > 0 ? (c >> (lg - 1)) & 1 : 0;
    return min(63, 2 * lg + half + 1);
}

//   heavy (nullable): set to 1 when the costs add up to more than
//   heavy_total, else 0 (the backward's launch shape, blend_bwd.cu).
static __global__ void __launch_bounds__(kSchedThreads) tile_order_kernel(
    const int32_t *__restrict__ offsets, const int32_t *__restrict__ cost, int n_tiles,
    int32_t *__restrict__ order, int32_t *__restrict__ heavy = nullptr,
    long long heavy_total = 0)
{
    __shared__ int hist[64];
    __shared__ unsigned long long s_sum;
    if (threadIdx.x < 64) hist[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    unsigned long long mine = 0;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const int c = cost ? cost[t] : offsets[t + 1] - offsets[t];
        atomicAdd(&hist[sched_bucket(c)], 1);
        mine += (unsigned long long)max(c, 0);
    }
    if (heavy) {   // warp sums first: one shared atomic per warp (integer: order-free)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_sum, mine);
    }
    __syncthreads();
    if (heavy && threadIdx.x == 0) *heavy = s_sum > (unsigned long long)heavy_total ? 1 : 0;
    if (threadIdx.x == 0) {
        int run = 0;
        for (int b = 63; b >= 0; --b) {   // descending cost
            const int h = hist[b];
            hist[b] = run;
            run += h;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const int c = cost ? cost[t] : offsets[t + 1] - offsets[t];
        order[atomicAdd(&hist[sched_bucket(c)], 1)] = t;
    }
}

}  // namespace sb
