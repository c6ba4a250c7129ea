// common.cuh -- shared device math for the sm_100a hot-path kernels.
//
// Numerics contract: the reference evaluates the
// per-pixel kernels in numba without FMA contraction and the camera transform
// as an OpenBLAS FMA chain.  The library is compiled with -fmad=false so no
// multiply-add is fused implicitly; the chains the reference fuses are written
// with fma() below.  exp/log in float are evaluated in double and rounded once
// (correctly rounded in practice), matching numba's expf on >99.9% of inputs.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/splatb200.h"

namespace sb {

constexpr double kAlphaClamp = 0.99;          // projection.py:22
constexpr double kAlphaCutoff = 1.0 / 255.0;  // projection.py:23
constexpr double kGuard = 1.3;                // projection.py:27
constexpr int kTile = 16;                     // forward.py:35
constexpr int kTilePx = kTile * kTile;
// the deterministic backward's per-(tile, row) partial adjoint record: 9 reals
// padded to 12 (three 16-byte vectors for float)
constexpr int kPartialReals = 12;

// The deterministic backward's view of an sb_bin workspace (binning.cu): per
// map row its depth rank; per rank its kept tiles (candidate-rectangle word +
// bit mask, or an explicit list), its kept count, its first rank-major pair
// index and a "replayed" flag; per rank-major pair index a replayed flag.
// The j-th kept tile of rank r (tiles ascending) has rank-major index
// rank_e0[r] + j: a row's pairs are contiguous there.
constexpr uint32_t kGeoBig = 1u << 31;   // geo flag: explicit tile list
struct BinMaps {
    const uint32_t *rank_of, *geo, *counts, *rank_e0;
    const uint64_t *masks;
    const uint16_t *big;
    uint8_t *pvalid, *rank_hit;
};

// index j of tile (tx, ty) among rank r's kept tiles, ascending (rank r keeps
// the tile); the candidate-rectangle word is tbase | (nx - 1) << 16
__device__ __forceinline__ uint32_t kept_index(const BinMaps &M, uint32_t r, int tx, int ty,
                                               int tiles_x)
{
    const uint32_t gw = __ldg(M.geo + r);
    const uint64_t mask = __ldg(M.masks + r);
    if (gw != kGeoBig) {
        const int tbase = (int)(gw & 0xFFFFu), nx = (int)((gw >> 16) & 0x7Fu) + 1;
        const int ty0 = tbase / tiles_x, tx0 = tbase - ty0 * tiles_x;
        const int bit = (ty - ty0) * nx + (tx - tx0);
        return (uint32_t)__popcll(mask & ((1ull << bit) - 1ull));
    }
    // explicit list (ascending tiles) at big[mask .. mask + counts[r])
    const uint16_t t = (uint16_t)(ty * tiles_x + tx);
    uint32_t a = 0, b = __ldg(M.counts + r);
    while (b - a > 1) {
        const uint32_t mid = (a + b) >> 1;
        if (__ldg(M.big + mask + mid) <= t) a = mid;
        else b = mid;
    }
    return a;
}

BinMaps bin_maps(int64_t m, int64_t pair_capacity, int32_t width, int32_t height,
                 const void *bin_workspace);
int32_t launch_gather_adjoints(int32_t dtype, int64_t m, int64_t pair_capacity, int32_t width,
                               int32_t height, int64_t sort_capacity, const void *bin_workspace,
                               const void *partial, void *d_mean, void *d_conic, void *d_op,
                               void *d_col, void *queue, uint32_t *queue_n,
                               uint8_t *reached_rows, cudaStream_t st);
constexpr int64_t kGatherQueueDiv = 64;   // a long rank has > 64 kept pairs

// Append the flagged values of a block (up to 1024 threads) to a list with
// ONE atomic per block (warp ballots -> shared prefix -> one atomicAdd): a
// per-warp atomic on the single counter serialises ~30k warps at one L2
// address.  Every thread of the block calls it (it has barriers); the
// entries of a block land in thread order.
__device__ __forceinline__ void block_append(bool reached, uint32_t r, uint32_t *__restrict__ list,
                                             uint32_t *__restrict__ count)
{
    __shared__ uint32_t s_off[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned m = __ballot_sync(0xffffffffu, reached);
    if (lane == 0) s_off[warp] = (uint32_t)__popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            const uint32_t c = s_off[w];
            s_off[w] = tot;
            tot += c;
        }
        const uint32_t base = tot ? atomicAdd(count, tot) : 0u;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s_off[w] += base;
    }
    __syncthreads();
    if (reached && list) list[s_off[warp] + __popc(m & ((1u << lane) - 1u))] = r;   // list NULL: count only
}

// Two block_appends in one pass (one pair of barriers): flag a -> list_a /
// count_a, flag b -> list_b / count_b (a NULL list: counted only).
__device__ __forceinline__ void block_append2(bool fa, uint32_t va, uint32_t *__restrict__ list_a,
                                              uint32_t *__restrict__ count_a, bool fb,
                                              uint32_t vb, uint32_t *__restrict__ list_b,
                                              uint32_t *__restrict__ count_b)
{
    __shared__ uint32_t s_a[32], s_b[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned ma = __ballot_sync(0xffffffffu, fa), mb = __ballot_sync(0xffffffffu, fb);
    if (lane == 0) {
        s_a[warp] = (uint32_t)__popc(ma);
        s_b[warp] = (uint32_t)__popc(mb);
    }
    __syncthreads();
    if (threadIdx.x < 2) {   // thread 0: list a, thread 1: list b
        uint32_t *so = threadIdx.x ? s_b : s_a;
        uint32_t tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            const uint32_t c = so[w];
            so[w] = tot;
            tot += c;
        }
        const uint32_t base = tot ? atomicAdd(threadIdx.x ? count_b : count_a, tot) : 0u;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) so[w] += base;
    }
    __syncthreads();
    const unsigned below = (1u << lane) - 1u;
    if (fa && list_a) list_a[s_a[warp] + __popc(ma & below)] = va;
    if (fb && list_b) list_b[s_b[warp] + __popc(mb & below)] = vb;
}


// projection.py:12-19
constexpr double SH_C0 = 0.28209479177387814;
constexpr double SH_C1 = 0.4886025119029199;
constexpr double SH_C2_0 = 1.0925484305920792, SH_C2_1 = -1.0925484305920792,
                 SH_C2_2 = 0.3153915652525205, SH_C2_3 = -1.0925484305920792,
                 SH_C2_4 = 0.5462742152960396;
constexpr double SH_C3_0 = -0.5900435899266435, SH_C3_1 = 2.890611442640554,
                 SH_C3_2 = -0.4570457994644658, SH_C3_3 = 0.3731763325901154,
                 SH_C3_4 = -0.4570457994644658, SH_C3_5 = 1.445305721320277,
                 SH_C3_6 = -0.5900435899266435;

// ---------------------------------------------------------------------------
// real-type helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float rexp(float x) { return (float)exp((double)x); }
__device__ __forceinline__ double rexp(double x) { return exp(x); }
__device__ __forceinline__ float rlog(float x) { return (float)log((double)x); }
__device__ __forceinline__ double rlog(double x) { return log(x); }
__device__ __forceinline__ float rsqrt_(float x) { return sqrtf(x); }
__device__ __forceinline__ double rsqrt_(double x) { return sqrt(x); }
__device__ __forceinline__ float rceil(float x) { return ceilf(x); }
__device__ __forceinline__ double rceil(double x) { return ceil(x); }
__device__ __forceinline__ float rfloor(float x) { return floorf(x); }
__device__ __forceinline__ double rfloor(double x) { return floor(x); }
__device__ __forceinline__ float rfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double rfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float rpow(float a, float b) { return (float)pow((double)a, (double)b); }
__device__ __forceinline__ double rpow(double a, double b) { return pow(a, b); }
__device__ __forceinline__ bool risfinite(float x) { return isfinite(x); }
__device__ __forceinline__ bool risfinite(double x) { return isfinite(x); }

// 16-byte vector of reals for record traffic
template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double2; };

// Load/store the 12-real splat record (3 x 16B for float, 6 x 16B for double)
template <typename T>
__device__ __forceinline__ void load_record(const T *__restrict__ rec, int64_t row, T out[12])
{
    using V = typename Vec4<T>::type;
    const V *p = reinterpret_cast<const V *>(rec + row * SB_RECORD_REALS);
    constexpr int nv = 12 * sizeof(T) / sizeof(V);
#pragma unroll
    for (int i = 0; i < nv; ++i) {
        V v = __ldg(p + i);
        reinterpret_cast<V *>(out)[i] = v;
    }
}

template <typename T>
__device__ __forceinline__ void store_record(T *__restrict__ rec, int64_t row, const T in[12])
{
    using V = typename Vec4<T>::type;
    V *p = reinterpret_cast<V *>(rec + row * SB_RECORD_REALS);
    constexpr int nv = 12 * sizeof(T) / sizeof(V);
#pragma unroll
    for (int i = 0; i < nv; ++i) p[i] = reinterpret_cast<const V *>(in)[i];
}

// Depth sort key: IEEE bits of a positive depth order like the value
// (depth > near > 0); invalid rows sort last.
template <typename T>
__device__ __forceinline__ void store_depth_key(void *keys, int64_t i, T depth, bool ok);
template <>
__device__ __forceinline__ void store_depth_key<float>(void *keys, int64_t i, float d, bool ok)
{
    reinterpret_cast<uint32_t *>(keys)[i] = ok ? __float_as_uint(d) : 0xFFFFFFFFu;
}
template <>
__device__ __forceinline__ void store_depth_key<double>(void *keys, int64_t i, double d, bool ok)
{
    reinterpret_cast<unsigned long long *>(keys)[i] =
        ok ? (unsigned long long)__double_as_longlong(d) : 0xFFFFFFFFFFFFFFFFull;
}

// Record field indices
enum { R_MX = 0, R_MY, R_A, R_B, R_C, R_OP, R_QC, R_RAD, R_C0, R_C1, R_C2, R_DEP };

// ---------------------------------------------------------------------------
// Camera in the working dtype, cast exactly where the reference casts.
// ---------------------------------------------------------------------------
template <typename T>
struct CamT {
    T W[9];       // rotation_wc
    T t[3];       // translation_wc
    T fx, fy, cx, cy;
    T nfx, nfy;   // -fx, -fy (Python float negated, then cast)
    T lim_x, lim_y;  // guard band (projection.py:204-205, double then cast)
    T cc[3];      // camera centre -W^T t (double then cast, projection.py:368)
    T ulo, uhi, vlo, vhi;  // frustum bounds (scene.py:294-298)
    T near_, dil;
    int32_t width, height;
};

template <typename T>
inline CamT<T> make_cam(const sb_camera_t &c, double near_, double dilation, double margin)
{
    CamT<T> k;
    for (int i = 0; i < 9; ++i) k.W[i] = (T)c.W[i];
    for (int i = 0; i < 3; ++i) k.t[i] = (T)c.t[i];
    k.fx = (T)c.fx; k.fy = (T)c.fy; k.cx = (T)c.cx; k.cy = (T)c.cy;
    k.nfx = (T)(-c.fx); k.nfy = (T)(-c.fy);
    k.lim_x = (T)(kGuard * (0.5 * c.width) / c.fx);
    k.lim_y = (T)(kGuard * (0.5 * c.height) / c.fy);
    for (int j = 0; j < 3; ++j)
        k.cc[j] = (T)(-(c.W[0 * 3 + j] * c.t[0] + c.W[1 * 3 + j] * c.t[1] + c.W[2 * 3 + j] * c.t[2]));
    const double mx = margin * c.width, my = margin * c.height;
    k.ulo = (T)(-mx); k.uhi = (T)(c.width - 1 + mx);
    k.vlo = (T)(-my); k.vhi = (T)(c.height - 1 + my);
    k.near_ = (T)near_;
    k.dil = (T)dilation;
    k.width = c.width;
    k.height = c.height;
    return k;
}

// x_cam = W x + t as the OpenBLAS FMA chain
template <typename T>
__device__ __forceinline__ void cam_transform(const CamT<T> &cam, T x, T y, T z, T tc[3])
{
#pragma unroll
    for (int j = 0; j < 3; ++j)
        tc[j] = rfma(z, cam.W[3 * j + 2], rfma(y, cam.W[3 * j + 1], x * cam.W[3 * j])) + cam.t[j];
}

// small row-major matmul C[m x p] = A[m x k] B[k x p], FMA chain over k
template <typename T, int M, int K, int P>
__device__ __forceinline__ void mm(const T *A, const T *B, T *Cm)
{
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j) {
            T acc = A[i * K] * B[j];
#pragma unroll
            for (int l = 1; l < K; ++l) acc = rfma(A[i * K + l], B[l * P + j], acc);
            Cm[i * P + j] = acc;
        }
}

template <typename T, int M, int N>
__device__ __forceinline__ void transpose(const T *A, T *Tm)
{
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) Tm[j * M + i] = A[i * N + j];
}

// quat_to_rot, projection.py:116-136 (renormalises)
template <typename T>
__device__ __forceinline__ void quat_to_rot(const T q[4], T Rm[9])
{
    const T n = rsqrt_(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    const T w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    const T one = (T)1, two = (T)2;
    Rm[0] = one - two * (y * y + z * z);
    Rm[1] = two * (x * y - w * z);
    Rm[2] = two * (x * z + w * y);
    Rm[3] = two * (x * y + w * z);
    Rm[4] = one - two * (x * x + z * z);
    Rm[5] = two * (y * z - w * x);
    Rm[6] = two * (x * z - w * y);
    Rm[7] = two * (y * z + w * x);
    Rm[8] = one - two * (x * x + y * y);
}

// projection_jacobian, projection.py:173-183
template <typename T>
__device__ __forceinline__ void jacobian(const CamT<T> &cam, const T t[3], T J[6])
{
    const T z = t[2];
    J[0] = cam.fx / z; J[1] = (T)0; J[2] = cam.nfx * t[0] / (z * z);
    J[3] = (T)0; J[4] = cam.fy / z; J[5] = cam.nfy * t[1] / (z * z);
}

// sh_basis, projection.py:39-62
template <typename T>
__device__ __forceinline__ void sh_basis(T x, T y, T z, T b[16])
{
    const T xx = x * x, yy = y * y, zz = z * z;
    const T xy = x * y, yz = y * z, xz = x * z;
    b[0] = (T)SH_C0;
    b[1] = (T)(-SH_C1) * y;
    b[2] = (T)SH_C1 * z;
    b[3] = (T)(-SH_C1) * x;
    b[4] = (T)SH_C2_0 * xy;
    b[5] = (T)SH_C2_1 * yz;
    b[6] = (T)SH_C2_2 * ((T)2.0 * zz - xx - yy);
    b[7] = (T)SH_C2_3 * xz;
    b[8] = (T)SH_C2_4 * (xx - yy);
    b[9] = (T)SH_C3_0 * y * ((T)3.0 * xx - yy);
    b[10] = (T)SH_C3_1 * xy * z;
    b[11] = (T)SH_C3_2 * y * ((T)4.0 * zz - xx - yy);
    b[12] = (T)SH_C3_3 * z * ((T)2.0 * zz - (T)3.0 * xx - (T)3.0 * yy);
    b[13] = (T)SH_C3_4 * x * ((T)4.0 * zz - xx - yy);
    b[14] = (T)SH_C3_5 * z * (xx - yy);
    b[15] = (T)SH_C3_6 * x * (xx - (T)3.0 * yy);
}

// d_dir[j] = sum_k d_basis[k] * d basis_k / d dir_j  (sh_basis_grad,
// projection.py:65-104, contracted on the fly; k order preserved)
template <typename T>
__device__ __forceinline__ void sh_dir_grad(T x, T y, T z, const T db[16], T dd[3])
{
    const T xx = x * x, yy = y * y, zz = z * z;
    T g[16][3];
#pragma unroll
    for (int k = 0; k < 16; ++k) g[k][0] = g[k][1] = g[k][2] = (T)0;
    g[1][1] = (T)(-SH_C1);
    g[2][2] = (T)SH_C1;
    g[3][0] = (T)(-SH_C1);
    g[4][0] = (T)SH_C2_0 * y;
    g[4][1] = (T)SH_C2_0 * x;
    g[5][1] = (T)SH_C2_1 * z;
    g[5][2] = (T)SH_C2_1 * y;
    g[6][0] = (T)SH_C2_2 * ((T)(-2.0) * x);
    g[6][1] = (T)SH_C2_2 * ((T)(-2.0) * y);
    g[6][2] = (T)SH_C2_2 * ((T)4.0 * z);
    g[7][0] = (T)SH_C2_3 * z;
    g[7][2] = (T)SH_C2_3 * x;
    g[8][0] = (T)SH_C2_4 * ((T)2.0 * x);
    g[8][1] = (T)SH_C2_4 * ((T)(-2.0) * y);
    g[9][0] = (T)(SH_C3_0 * 6.0) * x * y;
    g[9][1] = (T)SH_C3_0 * ((T)3.0 * xx - (T)3.0 * yy);
    g[10][0] = (T)SH_C3_1 * y * z;
    g[10][1] = (T)SH_C3_1 * x * z;
    g[10][2] = (T)SH_C3_1 * x * y;
    g[11][0] = (T)SH_C3_2 * ((T)(-2.0) * x * y);
    g[11][1] = (T)SH_C3_2 * ((T)4.0 * zz - xx - (T)3.0 * yy);
    g[11][2] = (T)SH_C3_2 * ((T)8.0 * y * z);
    g[12][0] = (T)SH_C3_3 * ((T)(-6.0) * x * z);
    g[12][1] = (T)SH_C3_3 * ((T)(-6.0) * y * z);
    g[12][2] = (T)SH_C3_3 * ((T)6.0 * zz - (T)3.0 * xx - (T)3.0 * yy);
    g[13][0] = (T)SH_C3_4 * ((T)4.0 * zz - (T)3.0 * xx - yy);
    g[13][1] = (T)SH_C3_4 * ((T)(-2.0) * x * y);
    g[13][2] = (T)SH_C3_4 * ((T)8.0 * x * z);
    g[14][0] = (T)SH_C3_5 * ((T)2.0 * x * z);
    g[14][1] = (T)SH_C3_5 * ((T)(-2.0) * y * z);
    g[14][2] = (T)SH_C3_5 * (xx - yy);
    g[15][0] = (T)SH_C3_6 * ((T)3.0 * xx - (T)3.0 * yy);
    g[15][1] = (T)SH_C3_6 * ((T)(-6.0) * x * y);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        T acc = (T)0;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += db[k] * g[k][j];
        dd[j] = acc;
    }
}

// ---------------------------------------------------------------------------
// Forward projection of one map row (projection.py:307-392).  Returns false
// when the reference would drop the row (near plane, opacity cutoff, det).
// ---------------------------------------------------------------------------
template <typename T>
struct Proj {
    T tc[3];       // t_cam
    T tcl[3];      // t_clamped
    bool clx, cly;
    T o;           // sigmoid opacity
    T m0, m1;      // mean2d
    T c2[4];       // dilated cov2d
    T det;
    T inv[4];      // conic
    T vd[3];       // view dir
    T basis[16];
    T craw[3], col[3];
    T qcut, radius;
};

// SH degree 3 -> colour from the view direction (projection.py:364-376); the
// colour half of project_row, callable after the geometry half decided the
// row is kept (so a dropped row never loads its 192-byte SH block).
template <typename T>
__device__ __forceinline__ void project_color(const CamT<T> &cam, const T p[3],
                                              const T *__restrict__ sh, Proj<T> &P)
{
    T v[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) v[j] = p[j] - cam.cc[j];
    const T vn = rsqrt_(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
#pragma unroll
    for (int j = 0; j < 3; ++j) P.vd[j] = v[j] / vn;
    sh_basis(P.vd[0], P.vd[1], P.vd[2], P.basis);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        T acc = (T)0;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += P.basis[k] * sh[3 * k + c];
        acc = acc + (T)0.5;
        P.craw[c] = acc;
        P.col[c] = acc > (T)0 ? acc : (T)0;
    }
}

template <typename T>
__device__ __forceinline__ bool project_row(const CamT<T> &cam, const T p[3], const T ls[3],
                                            const T q[4], T ol, const T *__restrict__ sh,
                                            bool need_color, Proj<T> &P)
{
    cam_transform(cam, p[0], p[1], p[2], P.tc);
    const T z = P.tc[2];
    if (!(z > cam.near_)) return false;
    // sigmoid, projection.py:293-300
    if (ol >= (T)0) P.o = (T)1 / ((T)1 + rexp(-ol));
    else { const T e = rexp(ol); P.o = e / ((T)1 + e); }
    if (!(P.o >= (T)kAlphaCutoff)) return false;
    P.m0 = cam.fx * P.tc[0] / z + cam.cx;
    P.m1 = cam.fy * P.tc[1] / z + cam.cy;
    T Rm[9];
    quat_to_rot(q, Rm);
    T s[3] = {rexp(ls[0]), rexp(ls[1]), rexp(ls[2])};
    T M3[9], M3t[9], cov3[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) M3[3 * a + b] = Rm[3 * a + b] * s[b];
    transpose<T, 3, 3>(M3, M3t);
    mm<T, 3, 3, 3>(M3, M3t, cov3);
    // clamp_for_jacobian, projection.py:197-211
    const T tx = P.tc[0] / z, ty = P.tc[1] / z;
    const T cxl = tx < -cam.lim_x ? -cam.lim_x : (tx > cam.lim_x ? cam.lim_x : tx);
    const T cyl = ty < -cam.lim_y ? -cam.lim_y : (ty > cam.lim_y ? cam.lim_y : ty);
    P.tcl[0] = cxl * z; P.tcl[1] = cyl * z; P.tcl[2] = z;
    P.clx = tx != cxl;
    P.cly = ty != cyl;
    T J[6], T2[6], TC[6], T2t[6];
    jacobian(cam, P.tcl, J);
    mm<T, 2, 3, 3>(J, cam.W, T2);
    mm<T, 2, 3, 3>(T2, cov3, TC);
    transpose<T, 2, 3>(T2, T2t);
    mm<T, 2, 3, 2>(TC, T2t, P.c2);
    P.c2[0] += cam.dil;
    P.c2[3] += cam.dil;
    P.det = P.c2[0] * P.c2[3] - P.c2[1] * P.c2[2];
    if (!(risfinite(P.det) && P.det > (T)0)) return false;
    P.inv[0] = P.c2[3] / P.det;
    P.inv[3] = P.c2[0] / P.det;
    P.inv[1] = -P.c2[1] / P.det;
    P.inv[2] = P.inv[1];
    // cutoff support, projection.py:378-384
    const T mid = (T)0.5 * (P.c2[0] + P.c2[3]);
    const T d2 = mid * mid - P.det;
    const T lam = mid + rsqrt_(d2 > (T)0 ? d2 : (T)0);
    P.qcut = (T)2.0 * rlog(P.o * (T)255.0);
    const T qpos = P.qcut > (T)0 ? P.qcut : (T)0;
    P.radius = rsqrt_(qpos * lam) * (T)(1 + 1e-5) + (T)1e-3;
    if (need_color) project_color(cam, p, sh, P);
    return true;
}

// Inputs of the chain rule that the reference takes from the SplatScreen
template <typename T>
struct ChainIn {
    T inv[4], tc[3], tcl[3], vd[3], basis[16], craw[3], o;
    bool clx, cly;
};

// Outputs: the 59 gradient reals of one row
template <typename T>
struct ChainOut {
    T dpos[3], dls[3], dq[4], dlogit, draw[3];   // d_sh = basis (x) draw
};

// _chain_to_parameters, backward.py:415-500, for one row
template <typename T>
__device__ __forceinline__ void chain_row(const CamT<T> &cam, const ChainIn<T> &in,
                                          const T pos[3], const T ls[3], const T q[4],
                                          const T *__restrict__ sh, const T dm[2],
                                          const T dcon3[3], T dop, const T dcol[3],
                                          ChainOut<T> &out)
{
    // dSigma' = -M dM M (backward.py:429-431), einsum order i,j,k,l
    const T dcon[4] = {dcon3[0], dcon3[1], dcon3[1], dcon3[2]};
    T dS2[4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int l = 0; l < 2; ++l) {
            T acc = (T)0;
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int k = 0; k < 2; ++k) acc += in.inv[2 * i + j] * dcon[2 * j + k] * in.inv[2 * k + l];
            dS2[2 * i + l] = -acc;
        }
    T Jm[6], J[6], T2[6], T2t[6], Wt[9];
    jacobian(cam, in.tc, Jm);
    jacobian(cam, in.tcl, J);
    mm<T, 2, 3, 3>(J, cam.W, T2);
    transpose<T, 2, 3>(T2, T2t);
    transpose<T, 3, 3>(cam.W, Wt);
    // q_unit = q/|q|; R = quat_to_rot(q_unit) (backward.py:441-443)
    T qu[4];
    {
        const T nn = rsqrt_(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
#pragma unroll
        for (int j = 0; j < 4; ++j) qu[j] = q[j] / nn;
    }
    T Rm[9];
    quat_to_rot(qu, Rm);
    T s[3] = {rexp(ls[0]), rexp(ls[1]), rexp(ls[2])};
    T M3[9], M3t[9], cov3[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) M3[3 * a + b] = Rm[3 * a + b] * s[b];
    transpose<T, 3, 3>(M3, M3t);
    mm<T, 3, 3, 3>(M3, M3t, cov3);
    // dT2, dJ, dSigma (backward.py:448-450)
    T dS2x2[4], a23[6], dT2[6], dJ[6], b32[6], dSig[9];
#pragma unroll
    for (int j = 0; j < 4; ++j) dS2x2[j] = (T)2.0 * dS2[j];
    mm<T, 2, 2, 3>(dS2x2, T2, a23);
    mm<T, 2, 3, 3>(a23, cov3, dT2);
    mm<T, 2, 3, 3>(dT2, Wt, dJ);
    mm<T, 3, 2, 2>(T2t, dS2, b32);
    mm<T, 3, 2, 3>(b32, T2, dSig);
    // camera-space point (backward.py:456-472)
    T dtc[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dtc[i] = Jm[i] * dm[0] + Jm[3 + i] * dm[1];
    const T xc = in.tcl[0], yc = in.tcl[1], z = in.tcl[2];
    const T z2 = z * z, z3 = z2 * z;
    const T d_xc = dJ[2] * (cam.nfx / z2);
    const T d_yc = dJ[5] * (cam.nfy / z2);
    dtc[0] += !in.clx ? d_xc : (T)0;
    dtc[1] += !in.cly ? d_yc : (T)0;
    dtc[2] += (dJ[0] * (cam.nfx / z2) + dJ[4] * (cam.nfy / z2)
               + dJ[2] * ((T)2 * cam.fx * xc / z3)
               + dJ[5] * ((T)2 * cam.fy * yc / z3)
               + (!in.clx ? (T)0 : d_xc * (xc / z))
               + (!in.cly ? (T)0 : d_yc * (yc / z)));
    mm<T, 1, 3, 3>(dtc, cam.W, out.dpos);
    // Sigma = M3 M3^T (backward.py:475-479)
    T dSig2x[9], dM3[9], dR[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) dSig2x[j] = (T)2.0 * dSig[j];
    mm<T, 3, 3, 3>(dSig2x, M3, dM3);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) dR[3 * a + b] = dM3[3 * a + b] * s[b];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const T ds = Rm[j] * dM3[j] + Rm[3 + j] * dM3[3 + j] + Rm[6 + j] * dM3[6 + j];
        out.dls[j] = ds * s[j];
    }
    // quat_rot_backward, projection.py:139-162
    {
        const T w = qu[0], x = qu[1], y = qu[2], zq = qu[3];
        const T *d = dR;
        const T two = (T)2;
        T dq[4];
        dq[0] = two * (-zq * d[1] + y * d[2] + zq * d[3] - x * d[5] - y * d[6] + x * d[7]);
        dq[1] = two * (y * d[1] + zq * d[2] + y * d[3] - two * x * d[4] - w * d[5]
                       + zq * d[6] + w * d[7] - two * x * d[8]);
        dq[2] = two * ((T)(-2) * y * d[0] + x * d[1] + w * d[2] + x * d[3] + zq * d[5]
                       - w * d[6] + zq * d[7] - two * y * d[8]);
        dq[3] = two * ((T)(-2) * zq * d[0] - w * d[1] + x * d[2] + w * d[3] - two * zq * d[4]
                       + y * d[5] + x * d[6] + y * d[7]);
        const T radial = dq[0] * w + dq[1] * x + dq[2] * y + dq[3] * zq;
#pragma unroll
        for (int j = 0; j < 4; ++j) out.dq[j] = dq[j] - radial * qu[j];
    }
    // SH colour and view-direction pull (backward.py:482-490)
#pragma unroll
    for (int c = 0; c < 3; ++c) out.draw[c] = dcol[c] * (in.craw[c] > (T)0 ? (T)1 : (T)0);
    T dbasis[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
        dbasis[k] = sh[3 * k] * out.draw[0] + sh[3 * k + 1] * out.draw[1] + sh[3 * k + 2] * out.draw[2];
    T ddir[3];
    sh_dir_grad(in.vd[0], in.vd[1], in.vd[2], dbasis, ddir);
    T v[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) v[j] = pos[j] - cam.cc[j];
    const T vn = rsqrt_(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    const T radial = ddir[0] * in.vd[0] + ddir[1] * in.vd[1] + ddir[2] * in.vd[2];
#pragma unroll
    for (int j = 0; j < 3; ++j) out.dpos[j] += (ddir[j] - radial * in.vd[j]) / vn;
    out.dlogit = dop * in.o * ((T)1 - in.o);
}

}  // namespace sb
