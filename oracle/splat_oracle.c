/*
 * splat_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, scalar restatement of the reference's CPU algorithm for the
 * Gaussian-LIC map-optimisation hot path (package `splatmap`, pure Python +
 * numba, under /root/reference/pkg/src/splatmap).  It is the CHECKER for the
 * sm_100a CUDA product in paper_2404_06926_b200/csrc/: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  Nothing in the product path links or calls this file.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference and records its
 * outputs) and against the reference's own closed-form KATs.
 *
 * The file is compiled twice: once with REAL=float (production dtype,
 * RunConfig precision 32, cli.py:52) and once with -DORACLE_F64 (the
 * reference's float64 verification mode).  Build flags are
 * -ffp-contract=off: the numba kernels never contract to FMA (SURVEY
 * Appendix A.2/A.11), while the OpenBLAS camera transform is an explicit FMA
 * chain, written below with RFMA.
 *
 * exp/log in float mode are evaluated in double and rounded once, i.e.
 * correctly rounded in practice; numba's float exp (glibc expf) agrees on
 * >99.9% of inputs and numpy's SIMD expf on ~61% -- the
 * parity comparators account for the resulting one-ulp decision flips.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef ORACLE_F64
typedef double real;
#define SFX(name) name##_f64
#define RFMA(a, b, c) fma((a), (b), (c))
#define RSQRT(x) sqrt(x)
#define REXP(x) exp(x)
#define RLOG(x) log(x)
#define RCEIL(x) ceil(x)
#define RFLOOR(x) floor(x)
#define RPOW(a, b) pow((a), (b))
#define RISFINITE(x) isfinite(x)
#define RMAXV 1.7976931348623157e308
#else
typedef float real;
#define SFX(name) name##_f32
#define RFMA(a, b, c) fmaf((a), (b), (c))
#define RSQRT(x) sqrtf(x)
#define REXP(x) ((float)exp((double)(x)))
#define RLOG(x) ((float)log((double)(x)))
#define RCEIL(x) ceilf(x)
#define RFLOOR(x) floorf(x)
#define RPOW(a, b) ((float)pow((double)(a), (double)(b)))
#define RISFINITE(x) isfinite(x)
#define RMAXV 3.4028234663852886e38f
#endif

#define R(x) ((real)(x))

/* projection.py:12-19 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.3153915652525205,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};
static const double ALPHA_CLAMP = 0.99;          /* projection.py:22 */
static const double ALPHA_CUTOFF = 1.0 / 255.0;  /* projection.py:23 */
static const double FRUSTUM_GUARD = 1.3;         /* projection.py:27 */

/* Camera = pose (world->camera, scene.py:67-80) + intrinsics (scene.py:51-64).
 * Kept in double exactly like the reference's host objects; each use casts to
 * the working dtype at the same point the reference does. */
typedef struct {
    double W[9];   /* rotation_wc, row-major */
    double t[3];   /* translation_wc */
    double fx, fy, cx, cy;
    int32_t width, height;
} ocam_t;

static inline real rmin(real a, real b) { return a < b ? a : b; }
static inline real rmax(real a, real b) { return a > b ? a : b; }

/* ------------------------------------------------------------------------ */
/* a1: frustum_mask, scene.py:283-298                                        */
/* pts @ W.T + t is an OpenBLAS FMA chain for N >= 2.  */
/* ------------------------------------------------------------------------ */
void SFX(oracle_frustum_mask)(int64_t n, const real *pos, const ocam_t *cam,
                              double near_, double margin, uint8_t *out)
{
    real W[9], t[3];
    for (int i = 0; i < 9; ++i) W[i] = R(cam->W[i]);
    for (int i = 0; i < 3; ++i) t[i] = R(cam->t[i]);
    const real fx = R(cam->fx), fy = R(cam->fy), cx = R(cam->cx), cy = R(cam->cy);
    const double mx = margin * cam->width, my = margin * cam->height;
    const real ulo = R(-mx), uhi = R(cam->width - 1 + mx);
    const real vlo = R(-my), vhi = R(cam->height - 1 + my);
    const real rnear = R(near_);
    for (int64_t i = 0; i < n; ++i) {
        const real x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
        real pc[3];
        for (int j = 0; j < 3; ++j)
            pc[j] = RFMA(z, W[3 * j + 2], RFMA(y, W[3 * j + 1], x * W[3 * j])) + t[j];
        const real zc = pc[2];
        int ok = zc > rnear;
        const real u = fx * pc[0] / zc + cx;   /* scene.py:292 */
        const real v = fy * pc[1] / zc + cy;
        ok = ok && (u >= ulo) && (u <= uhi) && (v >= vlo) && (v <= vhi);
        out[i] = (uint8_t)ok;
    }
}

/* ------------------------------------------------------------------------ */
/* SH basis and its direction gradient, projection.py:39-104                 */
/* Python-float coefficients are "weak" (NEP 50): a product of two Python    */
/* floats is formed in double before it meets the array dtype.               */
/* ------------------------------------------------------------------------ */
static void sh_basis(real x, real y, real z, real b[16])
{
    const real xx = x * x, yy = y * y, zz = z * z;
    const real xy = x * y, yz = y * z, xz = x * z;
    b[0] = R(SH_C0);
    b[1] = R(-SH_C1) * y;
    b[2] = R(SH_C1) * z;
    b[3] = R(-SH_C1) * x;
    b[4] = R(SH_C2[0]) * xy;
    b[5] = R(SH_C2[1]) * yz;
    b[6] = R(SH_C2[2]) * (R(2.0) * zz - xx - yy);
    b[7] = R(SH_C2[3]) * xz;
    b[8] = R(SH_C2[4]) * (xx - yy);
    b[9] = R(SH_C3[0]) * y * (R(3.0) * xx - yy);
    b[10] = R(SH_C3[1]) * xy * z;
    b[11] = R(SH_C3[2]) * y * (R(4.0) * zz - xx - yy);
    b[12] = R(SH_C3[3]) * z * (R(2.0) * zz - R(3.0) * xx - R(3.0) * yy);
    b[13] = R(SH_C3[4]) * x * (R(4.0) * zz - xx - yy);
    b[14] = R(SH_C3[5]) * z * (xx - yy);
    b[15] = R(SH_C3[6]) * x * (xx - R(3.0) * yy);
}

static void sh_basis_grad(real x, real y, real z, real g[16][3])
{
    const real xx = x * x, yy = y * y, zz = z * z;
    memset(g, 0, sizeof(real) * 48);
    g[1][1] = R(-SH_C1);
    g[2][2] = R(SH_C1);
    g[3][0] = R(-SH_C1);
    g[4][0] = R(SH_C2[0]) * y;
    g[4][1] = R(SH_C2[0]) * x;
    g[5][1] = R(SH_C2[1]) * z;
    g[5][2] = R(SH_C2[1]) * y;
    g[6][0] = R(SH_C2[2]) * (R(-2.0) * x);
    g[6][1] = R(SH_C2[2]) * (R(-2.0) * y);
    g[6][2] = R(SH_C2[2]) * (R(4.0) * z);
    g[7][0] = R(SH_C2[3]) * z;
    g[7][2] = R(SH_C2[3]) * x;
    g[8][0] = R(SH_C2[4]) * (R(2.0) * x);
    g[8][1] = R(SH_C2[4]) * (R(-2.0) * y);
    g[9][0] = R(SH_C3[0] * 6.0) * x * y;
    g[9][1] = R(SH_C3[0]) * (R(3.0) * xx - R(3.0) * yy);
    g[10][0] = R(SH_C3[1]) * y * z;
    g[10][1] = R(SH_C3[1]) * x * z;
    g[10][2] = R(SH_C3[1]) * x * y;
    g[11][0] = R(SH_C3[2]) * (R(-2.0) * x * y);
    g[11][1] = R(SH_C3[2]) * (R(4.0) * zz - xx - R(3.0) * yy);
    g[11][2] = R(SH_C3[2]) * (R(8.0) * y * z);
    g[12][0] = R(SH_C3[3]) * (R(-6.0) * x * z);
    g[12][1] = R(SH_C3[3]) * (R(-6.0) * y * z);
    g[12][2] = R(SH_C3[3]) * (R(6.0) * zz - R(3.0) * xx - R(3.0) * yy);
    g[13][0] = R(SH_C3[4]) * (R(4.0) * zz - R(3.0) * xx - yy);
    g[13][1] = R(SH_C3[4]) * (R(-2.0) * x * y);
    g[13][2] = R(SH_C3[4]) * (R(8.0) * x * z);
    g[14][0] = R(SH_C3[5]) * (R(2.0) * x * z);
    g[14][1] = R(SH_C3[5]) * (R(-2.0) * y * z);
    g[14][2] = R(SH_C3[5]) * (xx - yy);
    g[15][0] = R(SH_C3[6]) * (R(3.0) * xx - R(3.0) * yy);
    g[15][1] = R(SH_C3[6]) * (R(-6.0) * x * y);
}

/* quat_to_rot, projection.py:116-136 (renormalises first) */
static void quat_to_rot(const real *qin, real Rm[9], real qn[4])
{
    const real n = RSQRT(qin[0] * qin[0] + qin[1] * qin[1] + qin[2] * qin[2] + qin[3] * qin[3]);
    const real w = qin[0] / n, x = qin[1] / n, y = qin[2] / n, z = qin[3] / n;
    if (qn) { qn[0] = w; qn[1] = x; qn[2] = y; qn[3] = z; }
    Rm[0] = R(1) - R(2) * (y * y + z * z);
    Rm[1] = R(2) * (x * y - w * z);
    Rm[2] = R(2) * (x * z + w * y);
    Rm[3] = R(2) * (x * y + w * z);
    Rm[4] = R(1) - R(2) * (x * x + z * z);
    Rm[5] = R(2) * (y * z - w * x);
    Rm[6] = R(2) * (x * z - w * y);
    Rm[7] = R(2) * (y * z + w * x);
    Rm[8] = R(1) - R(2) * (x * x + y * y);
}

/* small row-major matmul C[m x p] = A[m x k] B[k x p] as an FMA chain over k
 * (the OpenBLAS small-kernel pattern) */
static void mm(const real *A, const real *B, real *C, int m, int k, int p)
{
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < p; ++j) {
            real acc = A[i * k] * B[j];
            for (int l = 1; l < k; ++l) acc = RFMA(A[i * k + l], B[l * p + j], acc);
            C[i * p + j] = acc;
        }
}

static void transpose(const real *A, real *T, int m, int n)
{
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) T[j * m + i] = A[i * n + j];
}

/* projection_jacobian, projection.py:173-183 (fx, fy are Python floats) */
static void jacobian(const real t[3], double fx, double fy, real J[6])
{
    const real z = t[2];
    J[0] = R(fx) / z; J[1] = 0; J[2] = R(-fx) * t[0] / (z * z);
    J[3] = 0; J[4] = R(fy) / z; J[5] = R(-fy) * t[1] / (z * z);
}

/* ------------------------------------------------------------------------ */
/* a2: project_gaussians, projection.py:307-392                              */
/* Outputs are N-indexed (row i <-> map row i); valid[i] says whether the    */
/* reference would keep the row.  Compaction preserves source order, so the  */
/* caller's nonzero(valid) reproduces SplatScreen.source_index.              */
/* ------------------------------------------------------------------------ */
void SFX(oracle_project)(int64_t n, const real *positions, const real *log_scales,
                         const real *rotations, const real *opacity_logits,
                         const real *sh_coeffs, const uint8_t *select, const ocam_t *cam,
                         double near_, double dilation,
                         uint8_t *valid, real *mean2d, real *cov2d, real *inv_cov2d,
                         real *depth, real *color, real *opacity, real *t_cam,
                         real *t_clamped, uint8_t *clamped_x, uint8_t *clamped_y,
                         real *view_dir, real *basis, real *color_raw,
                         real *radius_cut, real *q_cut)
{
    real W[9], Wt[9], tv[3];
    for (int i = 0; i < 9; ++i) W[i] = R(cam->W[i]);
    transpose(W, Wt, 3, 3);
    for (int i = 0; i < 3; ++i) tv[i] = R(cam->t[i]);
    /* camera centre -R^T t in double, then cast (projection.py:368) */
    real cc[3];
    for (int j = 0; j < 3; ++j)
        cc[j] = R(-(cam->W[0 * 3 + j] * cam->t[0] + cam->W[1 * 3 + j] * cam->t[1]
                    + cam->W[2 * 3 + j] * cam->t[2]));
    const real fx = R(cam->fx), fy = R(cam->fy), cx = R(cam->cx), cy = R(cam->cy);
    const double lim_x_d = FRUSTUM_GUARD * (0.5 * cam->width) / cam->fx;   /* projection.py:204-205 */
    const double lim_y_d = FRUSTUM_GUARD * (0.5 * cam->height) / cam->fy;
    const real lim_x = R(lim_x_d), lim_y = R(lim_y_d);
    const real rnear = R(near_), rdil = R(dilation);

    for (int64_t i = 0; i < n; ++i) {
        valid[i] = 0;
        if (select && !select[i]) continue;
        const real *p = positions + 3 * i;
        real tc[3];
        for (int j = 0; j < 3; ++j)
            tc[j] = RFMA(p[2], W[3 * j + 2], RFMA(p[1], W[3 * j + 1], p[0] * W[3 * j])) + tv[j];
        const real z = tc[2];
        if (!(z > rnear)) continue;                                   /* projection.py:329 */
        /* sigmoid, projection.py:293-300 */
        const real xl = opacity_logits[i];
        real o;
        if (xl >= 0) o = R(1) / (R(1) + REXP(-xl));
        else { const real e = REXP(xl); o = e / (R(1) + e); }
        if (!(o >= R(ALPHA_CUTOFF))) continue;                       /* projection.py:331-332 */

        const real m0 = fx * tc[0] / z + cx;                           /* projection.py:339 */
        const real m1 = fy * tc[1] / z + cy;

        real Rm[9];
        quat_to_rot(rotations + 4 * i, Rm, NULL);
        real s[3];
        for (int j = 0; j < 3; ++j) s[j] = REXP(log_scales[3 * i + j]);
        real M3[9], M3t[9], cov3[9];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) M3[3 * a + b] = Rm[3 * a + b] * s[b];
        transpose(M3, M3t, 3, 3);
        mm(M3, M3t, cov3, 3, 3, 3);

        /* clamp_for_jacobian, projection.py:197-211 */
        const real tx = tc[0] / z, ty = tc[1] / z;
        const real cxl = tx < -lim_x ? -lim_x : (tx > lim_x ? lim_x : tx);
        const real cyl = ty < -lim_y ? -lim_y : (ty > lim_y ? lim_y : ty);
        real tcl[3] = {cxl * z, cyl * z, z};
        real J[6], T[6], TC[6], Tt[6], c2[4];
        jacobian(tcl, cam->fx, cam->fy, J);
        mm(J, W, T, 2, 3, 3);
        mm(T, cov3, TC, 2, 3, 3);
        transpose(T, Tt, 2, 3);
        mm(TC, Tt, c2, 2, 3, 2);
        c2[0] += rdil;
        c2[3] += rdil;
        const real det = c2[0] * c2[3] - c2[1] * c2[2];
        if (!(RISFINITE(det) && det > 0)) continue;                  /* projection.py:353-360 */

        valid[i] = 1;
        mean2d[2 * i] = m0; mean2d[2 * i + 1] = m1;
        for (int j = 0; j < 4; ++j) cov2d[4 * i + j] = c2[j];
        inv_cov2d[4 * i + 0] = c2[3] / det;                            /* projection.py:362-366 */
        inv_cov2d[4 * i + 3] = c2[0] / det;
        inv_cov2d[4 * i + 1] = -c2[1] / det;
        inv_cov2d[4 * i + 2] = inv_cov2d[4 * i + 1];
        depth[i] = z;
        opacity[i] = o;
        for (int j = 0; j < 3; ++j) { t_cam[3 * i + j] = tc[j]; t_clamped[3 * i + j] = tcl[j]; }
        clamped_x[i] = tx != cxl;
        clamped_y[i] = ty != cyl;

        /* view direction + SH colour, projection.py:368-374 */
        real v[3];
        for (int j = 0; j < 3; ++j) v[j] = p[j] - cc[j];
        const real vn = RSQRT(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        real d[3] = {v[0] / vn, v[1] / vn, v[2] / vn};
        real b[16];
        sh_basis(d[0], d[1], d[2], b);
        for (int j = 0; j < 3; ++j) view_dir[3 * i + j] = d[j];
        for (int k = 0; k < 16; ++k) basis[16 * i + k] = b[k];
        const real *sh = sh_coeffs + 48 * i;
        for (int c = 0; c < 3; ++c) {
            real acc = 0;
            for (int k = 0; k < 16; ++k) acc += b[k] * sh[3 * k + c];
            acc = acc + R(0.5);
            color_raw[3 * i + c] = acc;
            color[3 * i + c] = acc > 0 ? acc : R(0);
        }

        /* cutoff support, projection.py:378-384 */
        const real mid = R(0.5) * (c2[0] + c2[3]);
        const real lam = mid + RSQRT(rmax(mid * mid - det, R(0)));
        const real qc = R(2.0) * RLOG(o * R(255.0));
        q_cut[i] = qc;
        radius_cut[i] = RSQRT(rmax(qc, R(0)) * lam) * R(1 + 1e-5) + R(1e-3);
    }
}

/* ------------------------------------------------------------------------ */
/* a3: bin_and_sort, forward.py:184-255, with _cull_pairs forward.py:112-159 */
/* Rows are whatever the screen holds (M rows, all valid).                   */
/* Returns P; writes outputs only when P <= capacity.                        */
/* ------------------------------------------------------------------------ */
static int cull_keep(real mx, real my, real a, real b, real c, real qcut,
                     real x0, real x1, real y0, real y1)
{
    if (x0 <= mx && mx <= x1 && y0 <= my && my <= y1) return 1;
    real qmin = (real)INFINITY;
    const real xe_[2] = {x0, x1}, ye_[2] = {y0, y1};
    for (int e = 0; e < 2; ++e) {
        const real xe = xe_[e];
        real yv = my - (b / c) * (xe - mx);
        if (yv < y0) yv = y0; else if (yv > y1) yv = y1;
        const real dx = xe - mx, dy = yv - my;
        const real q = a * dx * dx + R(2) * b * dx * dy + c * dy * dy;
        if (q < qmin) qmin = q;
    }
    for (int e = 0; e < 2; ++e) {
        const real ye = ye_[e];
        real xv = mx - (b / a) * (ye - my);
        if (xv < x0) xv = x0; else if (xv > x1) xv = x1;
        const real dx = xv - mx, dy = ye - my;
        const real q = a * dx * dx + R(2) * b * dx * dy + c * dy * dy;
        if (q < qmin) qmin = q;
    }
    return qmin <= qcut;
}

typedef struct { real d; int64_t i; } dkey_t;
static int cmp_dkey(const void *pa, const void *pb)
{
    const dkey_t *a = (const dkey_t *)pa, *b = (const dkey_t *)pb;
    if (a->d < b->d) return -1;
    if (a->d > b->d) return 1;
    return (a->i > b->i) - (a->i < b->i);
}

int64_t SFX(oracle_bin)(int64_t m, const real *mean2d, const real *inv_cov2d,
                        const real *depth, const real *radius, const real *q_cut,
                        int32_t width, int32_t height, int32_t ts, int32_t cull,
                        int64_t capacity, int64_t *pair_gaussian, int64_t *pair_tile,
                        int64_t *offsets)
{
    const int64_t tiles_x = (width + ts - 1) / ts, tiles_y = (height + ts - 1) / ts;
    const int64_t n_tiles = tiles_x * tiles_y;
    /* stable depth rank (forward.py:248-249) */
    dkey_t *dk = (dkey_t *)malloc(sizeof(dkey_t) * (m > 0 ? m : 1));
    for (int64_t i = 0; i < m; ++i) { dk[i].d = depth[i]; dk[i].i = i; }
    qsort(dk, (size_t)m, sizeof(dkey_t), cmp_dkey);
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
    for (int64_t r = 0; r < m; ++r) order[r] = dk[r].i;
    free(dk);

    int64_t *tcount = (int64_t *)calloc((size_t)n_tiles + 1, sizeof(int64_t));
    const real Wm1 = R(width - 1), Hm1 = R(height - 1);
    /* two passes in depth-rank order: count, then emit; a counting sort by
     * tile over rank-ordered pairs is exactly the (tile, rank) order */
    for (int pass = 0; pass < 2; ++pass) {
        int64_t *cursor = NULL;
        if (pass == 1) {
            int64_t total = 0;
            for (int64_t t = 0; t < n_tiles; ++t) total += tcount[t];
            if (total > capacity) { free(order); free(tcount); return total; }
            cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_tiles + 1));
            offsets[0] = 0;
            for (int64_t t = 0; t < n_tiles; ++t) offsets[t + 1] = offsets[t] + tcount[t];
            for (int64_t t = 0; t < n_tiles; ++t) cursor[t] = offsets[t];
        }
        for (int64_t r = 0; r < m; ++r) {
            const int64_t g = order[r];
            const real u = mean2d[2 * g], v = mean2d[2 * g + 1], rr = radius[g];
            /* forward.py:211-215 */
            if (!((u + rr >= 0) && (u - rr <= Wm1) && (v + rr >= 0) && (v - rr <= Hm1))) continue;
            real f;
            f = RFLOOR((u - rr) / R(ts)); int64_t tx0 = f < 0 ? 0 : (f > tiles_x - 1 ? tiles_x - 1 : (int64_t)f);
            f = RFLOOR((u + rr) / R(ts)); int64_t tx1 = f < 0 ? 0 : (f > tiles_x - 1 ? tiles_x - 1 : (int64_t)f);
            f = RFLOOR((v - rr) / R(ts)); int64_t ty0 = f < 0 ? 0 : (f > tiles_y - 1 ? tiles_y - 1 : (int64_t)f);
            f = RFLOOR((v + rr) / R(ts)); int64_t ty1 = f < 0 ? 0 : (f > tiles_y - 1 ? tiles_y - 1 : (int64_t)f);
            const real a = inv_cov2d[4 * g], b = inv_cov2d[4 * g + 1], c = inv_cov2d[4 * g + 3];
            for (int64_t ty = ty0; ty <= ty1; ++ty)
                for (int64_t tx = tx0; tx <= tx1; ++tx) {
                    if (cull) {
                        const real x0 = R(tx * ts), y0 = R(ty * ts);
                        const int64_t xe = tx * ts + ts - 1 < width - 1 ? tx * ts + ts - 1 : width - 1;
                        const int64_t ye = ty * ts + ts - 1 < height - 1 ? ty * ts + ts - 1 : height - 1;
                        if (!cull_keep(u, v, a, b, c, q_cut[g], x0, R(xe), y0, R(ye))) continue;
                    }
                    const int64_t tid = ty * tiles_x + tx;
                    if (pass == 0) tcount[tid]++;
                    else {
                        const int64_t k = cursor[tid]++;
                        pair_gaussian[k] = g;
                        pair_tile[k] = tid;
                    }
                }
        }
        if (pass == 1) free(cursor);
    }
    int64_t total = offsets[n_tiles];
    free(order);
    free(tcount);
    return total;
}

/* ------------------------------------------------------------------------ */
/* a4: _composite_tiles, forward.py:261-342 (numba prange over tiles; tiles  */
/* write disjoint pixels so the OpenMP loop is deterministic)                */
/* ------------------------------------------------------------------------ */
void SFX(oracle_composite)(const int64_t *pair_gaussian, const int64_t *offsets, int32_t tiles_x,
                           int32_t tiles_y, int32_t ts, int32_t width, int32_t height,
                           const real *mean2d, const real *inv_cov, const real *color,
                           const real *opacity, const real *depth, const real *q_cut,
                           const real *radius, int32_t early_termination, double thresh_d,
                           real *out_c, real *out_d, real *out_t, int32_t *out_nc)
{
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    const real thresh = R(thresh_d), cutoff = R(ALPHA_CUTOFF), clamp = R(ALPHA_CLAMP);
    const real one = R(1), half = one / R(2), two = one + one, q_margin = one / R(64);
    for (int64_t p = 0; p < (int64_t)width * height; ++p) {
        out_c[3 * p] = out_c[3 * p + 1] = out_c[3 * p + 2] = 0;
        out_d[p] = 0; out_t[p] = 1; out_nc[p] = 0;
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t t = 0; t < n_tiles; ++t) {
        const int64_t lo = offsets[t], hi = offsets[t + 1];
        if (hi == lo) continue;
        const int32_t ty = (int32_t)(t / tiles_x), tx = (int32_t)(t - (int64_t)ty * tiles_x);
        const int32_t x_lo = tx * ts, y_lo = ty * ts;
        const int32_t x_hi = x_lo + ts < width ? x_lo + ts : width;
        const int32_t y_hi = y_lo + ts < height ? y_lo + ts : height;
        for (int64_t k = lo; k < hi; ++k) {
            const int64_t g = pair_gaussian[k];
            const real mx = mean2d[2 * g], my = mean2d[2 * g + 1], r = radius[g];
            /* int(np.ceil(..)) clipped to the tile; clip in real first so a
             * huge radius cannot overflow the integer conversion */
            real f0 = RCEIL(mx - r), f1 = RFLOOR(mx + r), f2 = RCEIL(my - r), f3 = RFLOOR(my + r);
            const int32_t px0 = f0 > x_lo ? (f0 > x_hi ? x_hi : (int32_t)f0) : x_lo;
            const int32_t px1 = f1 < x_hi - 1 ? (f1 < x_lo - 1 ? x_lo - 1 : (int32_t)f1) : x_hi - 1;
            const int32_t py0 = f2 > y_lo ? (f2 > y_hi ? y_hi : (int32_t)f2) : y_lo;
            const int32_t py1 = f3 < y_hi - 1 ? (f3 < y_lo - 1 ? y_lo - 1 : (int32_t)f3) : y_hi - 1;
            if (px0 > px1 || py0 > py1) continue;
            const real a = inv_cov[4 * g], b = inv_cov[4 * g + 1], c = inv_cov[4 * g + 3];
            const real qc = q_cut[g] + q_margin, opa = opacity[g];
            const real c0 = color[3 * g], c1 = color[3 * g + 1], c2 = color[3 * g + 2], dep = depth[g];
            for (int32_t py = py0; py <= py1; ++py) {
                const real dy = R(py) - my;
                const real qy = c * dy * dy;
                const real bdy = two * b * dy;
                for (int32_t px = px0; px <= px1; ++px) {
                    const int64_t pix = (int64_t)py * width + px;
                    const real trans = out_t[pix];
                    if (early_termination && trans < thresh) continue;
                    const real dx = R(px) - mx;
                    const real q = a * dx * dx + bdy * dx + qy;
                    if (q > qc) continue;
                    real alpha = opa * REXP(-(half * q));
                    if (alpha > clamp) alpha = clamp;
                    if (alpha < cutoff) continue;
                    const real w = alpha * trans;
                    out_c[3 * pix] += w * c0;
                    out_c[3 * pix + 1] += w * c1;
                    out_c[3 * pix + 2] += w * c2;
                    out_d[pix] += w * dep;
                    out_nc[pix] += 1;
                    out_t[pix] = trans * (one - alpha);
                }
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* a6: _backward_tiles, backward.py:91-213 -- serial, private per-pair       */
/* accumulators merged once in (tile, rank) order.                           */
/* out_conic is (M, 3) = (aa, ab, cc).                                       */
/* ------------------------------------------------------------------------ */
void SFX(oracle_backward_tiles)(const int64_t *pair_gaussian, const int64_t *offsets,
                                int32_t tiles_x, int32_t tiles_y, int32_t ts, int32_t width,
                                int32_t height, const real *mean2d, const real *inv_cov,
                                const real *color, const real *opacity, const real *radius,
                                const real *q_cut, const real *dc_img, const real *c_final,
                                int32_t early_termination, double thresh_d, real *out_mean,
                                real *out_conic, real *out_opacity, real *out_color)
{
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    const real thresh = R(thresh_d), cutoff = R(ALPHA_CUTOFF), clamp = R(ALPHA_CLAMP);
    const real one = R(1), half = one / R(2), two = one + one, q_margin = one / R(64);
    const int npx = ts * ts;
    real *T = (real *)malloc(sizeof(real) * npx);
    real *P0 = (real *)malloc(sizeof(real) * npx);
    real *P1 = (real *)malloc(sizeof(real) * npx);
    real *P2 = (real *)malloc(sizeof(real) * npx);
    for (int64_t t = 0; t < n_tiles; ++t) {
        const int64_t lo = offsets[t], hi = offsets[t + 1];
        if (hi == lo) continue;
        const int32_t ty = (int32_t)(t / tiles_x), tx = (int32_t)(t - (int64_t)ty * tiles_x);
        const int32_t x_lo = tx * ts, y_lo = ty * ts;
        const int32_t x_hi = x_lo + ts < width ? x_lo + ts : width;
        const int32_t y_hi = y_lo + ts < height ? y_lo + ts : height;
        const int32_t w_t = x_hi - x_lo;
        for (int i = 0; i < npx; ++i) { T[i] = one; P0[i] = P1[i] = P2[i] = 0; }
        for (int64_t k = lo; k < hi; ++k) {
            const int64_t g = pair_gaussian[k];
            const real mx = mean2d[2 * g], my = mean2d[2 * g + 1], r = radius[g];
            real f0 = RCEIL(mx - r), f1 = RFLOOR(mx + r), f2 = RCEIL(my - r), f3 = RFLOOR(my + r);
            const int32_t px0 = f0 > x_lo ? (f0 > x_hi ? x_hi : (int32_t)f0) : x_lo;
            const int32_t px1 = f1 < x_hi - 1 ? (f1 < x_lo - 1 ? x_lo - 1 : (int32_t)f1) : x_hi - 1;
            const int32_t py0 = f2 > y_lo ? (f2 > y_hi ? y_hi : (int32_t)f2) : y_lo;
            const int32_t py1 = f3 < y_hi - 1 ? (f3 < y_lo - 1 ? y_lo - 1 : (int32_t)f3) : y_hi - 1;
            if (px0 > px1 || py0 > py1) continue;
            const real a = inv_cov[4 * g], b = inv_cov[4 * g + 1], c = inv_cov[4 * g + 3];
            const real qc = q_cut[g] + q_margin, opa = opacity[g];
            const real col0 = color[3 * g], col1 = color[3 * g + 1], col2 = color[3 * g + 2];
            real acc_mx = 0, acc_my = 0, acc_aa = 0, acc_ab = 0, acc_cc = 0, acc_o = 0;
            real acc_c0 = 0, acc_c1 = 0, acc_c2 = 0;
            for (int32_t py = py0; py <= py1; ++py) {
                const real dy = R(py) - my;
                const real qy = c * dy * dy;
                const real bdy = two * b * dy;
                const int32_t row = (py - y_lo) * w_t - x_lo;
                for (int32_t px = px0; px <= px1; ++px) {
                    const int32_t slot = row + px;
                    const real trans = T[slot];
                    if (early_termination && trans < thresh) continue;
                    const real dx = R(px) - mx;
                    const real q = a * dx * dx + bdy * dx + qy;
                    if (q > qc) continue;
                    const real gauss = REXP(-(half * q));
                    const real alpha_raw = opa * gauss;
                    real alpha = alpha_raw;
                    if (alpha > clamp) alpha = clamp;
                    if (alpha < cutoff) continue;
                    const real w = alpha * trans;
                    const real p0 = P0[slot] + w * col0;
                    const real p1 = P1[slot] + w * col1;
                    const real p2 = P2[slot] + w * col2;
                    const int64_t pix = (int64_t)py * width + px;
                    const real dc0 = dc_img[3 * pix], dc1 = dc_img[3 * pix + 1], dc2 = dc_img[3 * pix + 2];
                    acc_c0 += w * dc0;
                    acc_c1 += w * dc1;
                    acc_c2 += w * dc2;
                    if (alpha_raw < clamp) {
                        const real inv_rest = one / (one - alpha);
                        const real dalpha = (dc0 * (col0 * trans - (c_final[3 * pix] - p0) * inv_rest)
                                             + dc1 * (col1 * trans - (c_final[3 * pix + 1] - p1) * inv_rest)
                                             + dc2 * (col2 * trans - (c_final[3 * pix + 2] - p2) * inv_rest));
                        acc_o += dalpha * gauss;
                        const real dq = -(half * gauss * (dalpha * opa));
                        acc_mx += -(two * dq * (a * dx + b * dy));
                        acc_my += -(two * dq * (b * dx + c * dy));
                        acc_aa += dq * dx * dx;
                        acc_ab += dq * dx * dy;
                        acc_cc += dq * dy * dy;
                    }
                    P0[slot] = p0; P1[slot] = p1; P2[slot] = p2;
                    T[slot] = trans * (one - alpha);
                }
            }
            out_mean[2 * g] += acc_mx;
            out_mean[2 * g + 1] += acc_my;
            out_conic[3 * g] += acc_aa;
            out_conic[3 * g + 1] += acc_ab;
            out_conic[3 * g + 2] += acc_cc;
            out_opacity[g] += acc_o;
            out_color[3 * g] += acc_c0;
            out_color[3 * g + 1] += acc_c1;
            out_color[3 * g + 2] += acc_c2;
        }
    }
    free(T); free(P0); free(P1); free(P2);
}

/* ------------------------------------------------------------------------ */
/* a7: _chain_to_parameters, backward.py:415-500 (+ quat_rot_backward       */
/* projection.py:139-162, sh_basis_grad projection.py:65-104).               */
/* Rows are screen rows; src maps them to map rows; outputs accumulate      */
/* (np.add.at semantics) into N-row buffers the caller zeroed.               */
/* ------------------------------------------------------------------------ */
void SFX(oracle_chain)(int64_t m, const int64_t *src, const real *positions,
                       const real *log_scales, const real *rotations, const real *sh_coeffs,
                       const real *inv_cov2d, const real *t_cam, const real *t_clamped,
                       const uint8_t *clamped_x, const uint8_t *clamped_y,
                       const real *view_dir, const real *basis, const real *color_raw,
                       const real *opacity, const real *d_mean2d, const real *d_conic3,
                       const real *d_opacity, const real *d_color, const ocam_t *cam,
                       real *g_pos, real *g_log_scale, real *g_rot, real *g_opacity_logit,
                       real *g_sh)
{
    real W[9], Wt[9];
    for (int i = 0; i < 9; ++i) W[i] = R(cam->W[i]);
    transpose(W, Wt, 3, 3);
    const real fx = R(cam->fx), fy = R(cam->fy);
    real cc[3];
    for (int j = 0; j < 3; ++j)
        cc[j] = R(-(cam->W[0 * 3 + j] * cam->t[0] + cam->W[1 * 3 + j] * cam->t[1]
                    + cam->W[2 * 3 + j] * cam->t[2]));
    for (int64_t r = 0; r < m; ++r) {
        const int64_t n = src[r];
        /* dSigma' = -M dM M (backward.py:429-431) */
        const real *Mi = inv_cov2d + 4 * r;
        const real dcon[4] = {d_conic3[3 * r], d_conic3[3 * r + 1], d_conic3[3 * r + 1], d_conic3[3 * r + 2]};
        real dS2[4];
        for (int i = 0; i < 2; ++i)
            for (int l = 0; l < 2; ++l) {
                real acc = 0;
                for (int j = 0; j < 2; ++j)
                    for (int k = 0; k < 2; ++k) acc += Mi[2 * i + j] * dcon[2 * j + k] * Mi[2 * k + l];
                dS2[2 * i + l] = -acc;
            }
        const real *t = t_cam + 3 * r, *tc = t_clamped + 3 * r;
        real Jm[6], J[6], T2[6], T2t[6];
        jacobian(t, cam->fx, cam->fy, Jm);
        jacobian(tc, cam->fx, cam->fy, J);
        mm(J, W, T2, 2, 3, 3);
        transpose(T2, T2t, 2, 3);
        real Rm[9];
        /* backward.py:441-442 normalises q, then quat_to_rot normalises again */
        real qu[4];
        {
            const real *q = rotations + 4 * n;
            const real nn = RSQRT(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
            for (int j = 0; j < 4; ++j) qu[j] = q[j] / nn;
            quat_to_rot(qu, Rm, NULL);
        }
        real s[3];
        for (int j = 0; j < 3; ++j) s[j] = REXP(log_scales[3 * n + j]);
        real M3[9], M3t[9], cov3[9];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) M3[3 * a + b] = Rm[3 * a + b] * s[b];
        transpose(M3, M3t, 3, 3);
        mm(M3, M3t, cov3, 3, 3, 3);

        /* dT2 = 2 dS2 T2 cov3d; dJ = dT2 W^T; dSigma = T2^T dS2 T2 (448-450) */
        real dS2x2[4], a23[6], dT2[6], dJ[6], b32[6], dSig[9];
        for (int j = 0; j < 4; ++j) dS2x2[j] = R(2.0) * dS2[j];
        mm(dS2x2, T2, a23, 2, 2, 3);
        mm(a23, cov3, dT2, 2, 3, 3);
        mm(dT2, Wt, dJ, 2, 3, 3);
        mm(T2t, dS2, b32, 3, 2, 2);
        mm(b32, T2, dSig, 3, 2, 3);

        /* camera-space point adjoint (456-472) */
        const real *dm = d_mean2d + 2 * r;
        real dtc[3];
        for (int i = 0; i < 3; ++i) dtc[i] = Jm[i] * dm[0] + Jm[3 + i] * dm[1];
        const real xc = tc[0], yc = tc[1], z = tc[2];
        const real z2 = z * z, z3 = z2 * z;
        const real d_xc = dJ[2] * (-fx / z2);
        const real d_yc = dJ[5] * (-fy / z2);
        const int free_x = !clamped_x[r], free_y = !clamped_y[r];
        dtc[0] += free_x ? d_xc : R(0);
        dtc[1] += free_y ? d_yc : R(0);
        dtc[2] += (dJ[0] * (-fx / z2) + dJ[4] * (-fy / z2)
                   + dJ[2] * (R(2) * fx * xc / z3)
                   + dJ[5] * (R(2) * fy * yc / z3)
                   + (free_x ? R(0) : d_xc * (xc / z))
                   + (free_y ? R(0) : d_yc * (yc / z)));
        real dpos[3];
        mm(dtc, W, dpos, 1, 3, 3);

        /* Sigma = M3 M3^T (475-479) */
        real dSig2x[9], dM3[9];
        for (int j = 0; j < 9; ++j) dSig2x[j] = R(2.0) * dSig[j];
        mm(dSig2x, M3, dM3, 3, 3, 3);
        real dR[9], ds[3], dls[3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) dR[3 * a + b] = dM3[3 * a + b] * s[b];
        for (int j = 0; j < 3; ++j) {
            ds[j] = Rm[j] * dM3[j] + Rm[3 + j] * dM3[3 + j] + Rm[6 + j] * dM3[6 + j];
            dls[j] = ds[j] * s[j];
        }
        /* quat_rot_backward, projection.py:139-162 */
        const real w = qu[0], x = qu[1], y = qu[2], zq = qu[3];
        const real *d = dR;
        real dq[4];
        dq[0] = R(2) * (-zq * d[1] + y * d[2] + zq * d[3] - x * d[5] - y * d[6] + x * d[7]);
        dq[1] = R(2) * (y * d[1] + zq * d[2] + y * d[3] - R(2) * x * d[4] - w * d[5]
                        + zq * d[6] + w * d[7] - R(2) * x * d[8]);
        dq[2] = R(2) * (R(-2) * y * d[0] + x * d[1] + w * d[2] + x * d[3] + zq * d[5]
                        - w * d[6] + zq * d[7] - R(2) * y * d[8]);
        dq[3] = R(2) * (R(-2) * zq * d[0] - w * d[1] + x * d[2] + w * d[3] - R(2) * zq * d[4]
                        + y * d[5] + x * d[6] + y * d[7]);
        const real radial_q = dq[0] * w + dq[1] * x + dq[2] * y + dq[3] * zq;
        for (int j = 0; j < 4; ++j) dq[j] = dq[j] - radial_q * qu[j];

        /* SH colour and view-direction pull (482-490) */
        const real *b16 = basis + 16 * r, *vd = view_dir + 3 * r;
        real draw[3];
        for (int c = 0; c < 3; ++c) draw[c] = d_color[3 * r + c] * (color_raw[3 * r + c] > 0 ? R(1) : R(0));
        const real *shc = sh_coeffs + 48 * n;
        real dbasis[16];
        for (int k = 0; k < 16; ++k)
            dbasis[k] = shc[3 * k] * draw[0] + shc[3 * k + 1] * draw[1] + shc[3 * k + 2] * draw[2];
        real bg[16][3];
        sh_basis_grad(vd[0], vd[1], vd[2], bg);
        real ddir[3];
        for (int j = 0; j < 3; ++j) {
            real acc = 0;
            for (int k = 0; k < 16; ++k) acc += dbasis[k] * bg[k][j];
            ddir[j] = acc;
        }
        real v[3];
        for (int j = 0; j < 3; ++j) v[j] = positions[3 * n + j] - cc[j];
        const real vn = RSQRT(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        const real radial = ddir[0] * vd[0] + ddir[1] * vd[1] + ddir[2] * vd[2];
        for (int j = 0; j < 3; ++j) dpos[j] += (ddir[j] - radial * vd[j]) / vn;

        const real o = opacity[r];
        const real dlogit = d_opacity[r] * o * (R(1) - o);

        for (int j = 0; j < 3; ++j) { g_pos[3 * n + j] += dpos[j]; g_log_scale[3 * n + j] += dls[j]; }
        for (int j = 0; j < 4; ++j) g_rot[4 * n + j] += dq[j];
        g_opacity_logit[n] += dlogit;
        for (int k = 0; k < 16; ++k)
            for (int c = 0; c < 3; ++c) g_sh[48 * n + 3 * k + c] += b16[k] * draw[c];
    }
}

/* ------------------------------------------------------------------------ */
/* a5: photometric_loss + apply_exposure + ssim_forward/ssim_backward,      */
/* loss.py:31-177.  Images are (H, W, 3) row-major, E is the f64 3x4.       */
/* parts[0..2] = loss, l1, dssim; parts[3] = ssim.                           */
/* ------------------------------------------------------------------------ */
#define SS_WIN 11
#define SS_PAD 5

static void gauss_kernel(real k[SS_WIN])   /* loss.py:39-42 */
{
    double kd[SS_WIN], s = 0;
    for (int i = 0; i < SS_WIN; ++i) {
        const double x = (double)(i - SS_PAD);
        kd[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
        s += kd[i];
    }
    for (int i = 0; i < SS_WIN; ++i) k[i] = R(kd[i] / s);
}

static inline int reflect_idx(int p, int n)   /* numpy mode="reflect" */
{
    while (p < 0 || p >= n) {
        if (p < 0) p = -p;
        if (p >= n) p = 2 * (n - 1) - p;
    }
    return p;
}

/* _conv_valid on a reflect-padded plane: rows first, then columns (loss.py:54-65) */
static void conv_valid(const real *xp, int hp, int wp, const real k[SS_WIN], real *out, real *tmp)
{
    const int h = hp - 2 * SS_PAD, w = wp - 2 * SS_PAD;
    for (int i = 0; i < h * wp; ++i) tmp[i] = 0;
    for (int a = 0; a < SS_WIN; ++a)
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < wp; ++c) tmp[r * wp + c] += k[a] * xp[(r + a) * wp + c];
    for (int i = 0; i < h * w; ++i) out[i] = 0;
    for (int b = 0; b < SS_WIN; ++b)
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c) out[r * w + c] += k[b] * tmp[r * wp + c + b];
}

/* _conv_valid_adjoint (loss.py:68-78) */
static void conv_adj(const real *dout, int h, int w, const real k[SS_WIN], real *dxp, real *dtmp)
{
    const int wp = w + 2 * SS_PAD, hp = h + 2 * SS_PAD;
    for (int i = 0; i < h * wp; ++i) dtmp[i] = 0;
    for (int b = 0; b < SS_WIN; ++b)
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c) dtmp[r * wp + c + b] += k[b] * dout[r * w + c];
    for (int i = 0; i < hp * wp; ++i) dxp[i] = 0;
    for (int a = 0; a < SS_WIN; ++a)
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < wp; ++c) dxp[(r + a) * wp + c] += k[a] * dtmp[r * wp + c];
}

void SFX(oracle_loss)(int32_t h, int32_t w, const real *rendered, const real *gt,
                      const double *E, double lam_d, double *parts, real *d_rendered,
                      double *d_E)
{
    const int hp = h + 2 * SS_PAD, wp = w + 2 * SS_PAD;
    const int64_t npx = (int64_t)h * w;
    const real lam = R(lam_d);
    const real nn = R((double)h * w * 3);
    real M[9], bvec[3];
    for (int c = 0; c < 3; ++c) {
        for (int j = 0; j < 3; ++j) M[3 * c + j] = R(E[4 * c + j]);
        bvec[c] = R(E[4 * c + 3]);
    }
    real k[SS_WIN];
    gauss_kernel(k);
    const real c1 = R(0.01 * 0.01), c2 = R(0.03 * 0.03);

    real *Y = (real *)malloc(sizeof(real) * npx * 3);
    real *dY = (real *)malloc(sizeof(real) * npx * 3);
    /* Y = C @ M.T + b (loss.py:157-158; BLAS FMA chain) */
    double l1 = 0;
    for (int64_t p = 0; p < npx; ++p) {
        const real *C = rendered + 3 * p;
        for (int c = 0; c < 3; ++c) {
            const real y = RFMA(C[2], M[3 * c + 2], RFMA(C[1], M[3 * c + 1], C[0] * M[3 * c])) + bvec[c];
            Y[3 * p + c] = y;
            const real diff = y - gt[3 * p + c];
            l1 += fabs((double)diff);
            const real sg = diff > 0 ? R(1) : (diff < 0 ? R(-1) : R(0));
            dY[3 * p + c] = (R(1) - lam) * sg / nn;            /* loss.py:164 */
        }
    }
    const real l1r = R(l1 / (double)(npx * 3));

    real *xp = (real *)malloc(sizeof(real) * hp * wp);
    real *yp = (real *)malloc(sizeof(real) * hp * wp);
    real *prod = (real *)malloc(sizeof(real) * hp * wp);
    real *tmp = (real *)malloc(sizeof(real) * h * wp);
    real *mu_x = (real *)malloc(sizeof(real) * npx), *mu_y = (real *)malloc(sizeof(real) * npx);
    real *sxx = (real *)malloc(sizeof(real) * npx), *syy = (real *)malloc(sizeof(real) * npx);
    real *sxy = (real *)malloc(sizeof(real) * npx);
    real *dmu = (real *)malloc(sizeof(real) * npx), *dsxx = (real *)malloc(sizeof(real) * npx);
    real *dsxy = (real *)malloc(sizeof(real) * npx);
    real *A = (real *)malloc(sizeof(real) * hp * wp), *B = (real *)malloc(sizeof(real) * hp * wp);
    real *Cc = (real *)malloc(sizeof(real) * hp * wp);
    double ssim_total = 0;
    const real coeff = R(-(double)lam / 2.0) / R((double)3 * h * w);   /* loss.py:114, 170 */
    for (int ch = 0; ch < 3; ++ch) {
        for (int r = 0; r < hp; ++r)
            for (int c = 0; c < wp; ++c) {
                const int sr = reflect_idx(r - SS_PAD, h), sc = reflect_idx(c - SS_PAD, w);
                xp[r * wp + c] = Y[3 * ((int64_t)sr * w + sc) + ch];
                yp[r * wp + c] = gt[3 * ((int64_t)sr * w + sc) + ch];
            }
        conv_valid(xp, hp, wp, k, mu_x, tmp);
        conv_valid(yp, hp, wp, k, mu_y, tmp);
        for (int i = 0; i < hp * wp; ++i) prod[i] = xp[i] * xp[i];
        conv_valid(prod, hp, wp, k, sxx, tmp);
        for (int i = 0; i < hp * wp; ++i) prod[i] = yp[i] * yp[i];
        conv_valid(prod, hp, wp, k, syy, tmp);
        for (int i = 0; i < hp * wp; ++i) prod[i] = xp[i] * yp[i];
        conv_valid(prod, hp, wp, k, sxy, tmp);
        double ssum = 0;
        for (int64_t i = 0; i < npx; ++i) {
            const real mx = mu_x[i], my = mu_y[i];
            const real vxx = sxx[i] - mx * mx, vyy = syy[i] - my * my, vxy = sxy[i] - mx * my;
            const real a1 = R(2) * mx * my + c1, a2 = R(2) * vxy + c2;
            const real b1 = mx * mx + my * my + c1, b2 = vxx + vyy + c2;
            const real s = (a1 * a2) / (b1 * b2);
            ssum += s;
            /* ssim_backward per-pixel part (loss.py:116-126) */
            const real denom = b1 * b2;
            const real da1 = coeff * a2 / denom, da2 = coeff * a1 / denom;
            const real db1 = -coeff * s / b1, db2 = -coeff * s / b2;
            real dmx = R(2) * my * da1 + R(2) * mx * db1;
            const real dvxy = R(2) * da2, dvxx = db2;
            dmx += R(-2) * mx * dvxx - my * dvxy;
            dmu[i] = dmx; dsxx[i] = dvxx; dsxy[i] = dvxy;
        }
        ssim_total += ssum / (double)npx;
        conv_adj(dmu, h, w, k, A, tmp);
        conv_adj(dsxx, h, w, k, B, tmp);
        conv_adj(dsxy, h, w, k, Cc, tmp);
        /* dxp = A + 2 xp B + yp C (loss.py:128-130) */
        for (int i = 0; i < hp * wp; ++i) A[i] = A[i] + R(2) * xp[i] * B[i] + yp[i] * Cc[i];
        /* accumulate fold into a temporary, then add to dY (loss.py:131-134, 172) */
        real *fold = prod;
        for (int64_t i = 0; i < npx; ++i) fold[i] = 0;
        for (int r = 0; r < hp; ++r)
            for (int c = 0; c < wp; ++c) {
                const int sr = reflect_idx(r - SS_PAD, h), sc = reflect_idx(c - SS_PAD, w);
                fold[(int64_t)sr * w + sc] += A[r * wp + c];
            }
        for (int64_t i = 0; i < npx; ++i) dY[3 * i + ch] = dY[3 * i + ch] + fold[i];
    }
    const real ssim_val = R(ssim_total / 3.0);
    const real dssim = (R(1) - ssim_val) / R(2);
    const real loss = (R(1) - lam) * l1r + lam * dssim;
    parts[0] = loss; parts[1] = l1r; parts[2] = dssim; parts[3] = ssim_val;

    /* d_rendered = dY @ M; dM = sum dY (x) C; db = sum dY (loss.py:174-176) */
    double dE[12] = {0};
    for (int64_t p = 0; p < npx; ++p) {
        const real *g = dY + 3 * p, *C = rendered + 3 * p;
        for (int j = 0; j < 3; ++j)
            d_rendered[3 * p + j] = RFMA(g[2], M[6 + j], RFMA(g[1], M[3 + j], g[0] * M[j]));
        for (int c = 0; c < 3; ++c) {
            for (int j = 0; j < 3; ++j) dE[4 * c + j] += (double)g[c] * (double)C[j];
            dE[4 * c + 3] += g[c];
        }
    }
    for (int i = 0; i < 12; ++i) d_E[i] = (double)R(dE[i]);
    free(Y); free(dY); free(xp); free(yp); free(prod); free(tmp); free(mu_x); free(mu_y);
    free(sxx); free(syy); free(sxy); free(dmu); free(dsxx); free(dsxy); free(A); free(B); free(Cc);
}

/* ------------------------------------------------------------------------ */
/* a8: adam_step sparse/dense, adam.py:76-122.  Groups are passed as flat   */
/* arrays with their per-row width; lr_rows gives one lr per (row-local)    */
/* coefficient block (SH row 0 vs rows 1..15, adam.py:67-73).               */
/* active: NULL = dense; else uint8 mask over rows.                          */
/* ------------------------------------------------------------------------ */
void SFX(oracle_adam)(int64_t n, int32_t n_groups, real *const *params, const real *const *grads,
                      real *const *m1, real *const *m2, const int32_t *widths,
                      const double *lr_first, const double *lr_rest, const int32_t *first_len,
                      int64_t *steps, const uint8_t *active)
{
    const real b1 = R(0.9), b2 = R(0.999), eps = R(1e-15);
    for (int64_t i = 0; i < n; ++i) {
        if (active && !active[i]) continue;
        steps[i] += 1;
        const real tt = R((double)steps[i]);
        const real bc1 = R(1) - RPOW(b1, tt);
        const real bc2 = R(1) - RPOW(b2, tt);
        for (int gi = 0; gi < n_groups; ++gi) {
            const int32_t wdt = widths[gi];
            const real lr0 = R(lr_first[gi]), lr1 = R(lr_rest[gi]);
            for (int32_t j = 0; j < wdt; ++j) {
                const int64_t e = i * wdt + j;
                const real g = grads[gi][e];
                const real m = b1 * m1[gi][e] + (R(1) - b1) * g;
                const real v = b2 * m2[gi][e] + (R(1) - b2) * g * g;
                m1[gi][e] = m;
                m2[gi][e] = v;
                const real mh = m / bc1, vh = v / bc2;
                const real lr = j < first_len[gi] ? lr0 : lr1;
                params[gi][e] -= lr * mh / (RSQRT(vh) + eps);
            }
        }
    }
}

/* Host threads for the OpenMP-parallel blend (the CPU baseline times the
 * oracle with every host core; a torchrun launch defaults OMP to 1 thread). */
void SFX(oracle_set_threads)(int32_t n)
{
    if (n > 0) omp_set_num_threads(n);
}
