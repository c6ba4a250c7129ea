// blend_common.cuh -- pieces shared by the forward (blend.cu) and backward
// (blend_bwd.cu) blends: the staged splat record and the forward's exp.
#pragma once

#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

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

}  // namespace sb
