// preprocess.cu -- K1 frustum mask, K2 projection, K9 chain rule.
//
// a1 frustum_mask   scene.py:283-298
// a2 project_gaussians projection.py:307-392
// a7 _chain_to_parameters backward.py:415-500
//
// One thread per map row.  The 236 B of parameters per Gaussian are read with
// 16-byte vector loads where the row is 16-byte aligned (the SH block is
// 192 B); rows are independent, so the kernels are HBM-bound streams.
#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

template <typename T>
__device__ __forceinline__ void load_sh(const T *__restrict__ sh_coeffs, int64_t i, T sh[48])
{
    using V = typename Vec4<T>::type;
    const V *p = reinterpret_cast<const V *>(sh_coeffs + i * 48);
    constexpr int nv = 48 * sizeof(T) / sizeof(V);
#pragma unroll
    for (int k = 0; k < nv; ++k) reinterpret_cast<V *>(sh)[k] = __ldg(p + k);
}

template <typename T>
__global__ void __launch_bounds__(256) frustum_kernel(int64_t n, const T *__restrict__ pos,
                                                      CamT<T> cam, uint8_t *__restrict__ out)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    T tc[3];
    cam_transform(cam, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], tc);
    const T z = tc[2];
    bool ok = z > cam.near_;
    const T u = cam.fx * tc[0] / z + cam.cx;
    const T v = cam.fy * tc[1] / z + cam.cy;
    ok = ok && (u >= cam.ulo) && (u <= cam.uhi) && (v >= cam.vlo) && (v <= cam.vhi);
    out[i] = ok;
}

template <typename T>
__global__ void __launch_bounds__(128, sizeof(T) == 4 ? 7 : 1) preprocess_fwd_kernel(
    int64_t n, const T *__restrict__ pos, const T *__restrict__ ls, const T *__restrict__ rot,
    const T *__restrict__ ol, const T *__restrict__ shc, const uint8_t *__restrict__ select,
    CamT<T> cam, T *__restrict__ records, uint8_t *__restrict__ valid,
    void *__restrict__ depth_key, uint32_t *__restrict__ depth_val,
    uint8_t *__restrict__ frustum, sb_screen_extras_t ex, const float *__restrict__ coarse)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const T p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    // the rest of the geometry (32 B) loaded with the position, before the
    // near-plane test needs it: one dependent round trip less per row
    const T l[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
    const T q[4] = {rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]};
    const T olog = ol[i];
    if (frustum) {
        // a1 fused: the same FMA-chain transform the projection uses
        T tc[3];
        cam_transform(cam, p[0], p[1], p[2], tc);
        const T z = tc[2];
        bool ok = z > cam.near_;
        const T u = cam.fx * tc[0] / z + cam.cx;
        const T v = cam.fy * tc[1] / z + cam.cy;
        frustum[i] = ok && (u >= cam.ulo) && (u <= cam.uhi) && (v >= cam.vlo) && (v <= cam.vhi);
    }
    bool keep = select == nullptr || select[i];
    if (keep) {
        // rows behind the near plane fail project_row's first test
        // (projection.py:329): decide that from the position alone, before
        // loading the row's 192-byte SH block (half of a map that surrounds
        // the camera)
        T tc[3];
        cam_transform(cam, p[0], p[1], p[2], tc);
        keep = tc[2] > cam.near_;
    }
    Proj<T> P;
    if (keep) {
        // geometry first: the colour (and its 192-byte SH load) only for rows
        // that survive the coarse depth-limit drop below
        keep = project_row(cam, p, l, q, olog, (const T *)nullptr, false, P);
    }
    if (keep && coarse) {
        // behind every tile depth limit under its cutoff box (the 4x4-tile
        // maxima of the previous iteration's limits): the row can have no
        // pair in this iteration's depth-limited lists (sb_bin), so it is
        // dropped here -- no record, an invalid-row sort key
        const T r = P.radius, ts = (T)kTile;
        const T Wm1 = (T)(cam.width - 1), Hm1 = (T)(cam.height - 1);
        if ((P.m0 + r >= (T)0) && (P.m0 - r <= Wm1) && (P.m1 + r >= (T)0) && (P.m1 - r <= Hm1)) {
            const int tiles_x = (cam.width + kTile - 1) / kTile, tiles_y = (cam.height + kTile - 1) / kTile;
            auto clampi = [](T f, int hi) -> int { return f < (T)0 ? 0 : (f > (T)hi ? hi : (int)f); };
            const int tx0 = clampi(rfloor((P.m0 - r) / ts), tiles_x - 1);
            const int tx1 = clampi(rfloor((P.m0 + r) / ts), tiles_x - 1);
            const int ty0 = clampi(rfloor((P.m1 - r) / ts), tiles_y - 1);
            const int ty1 = clampi(rfloor((P.m1 + r) / ts), tiles_y - 1);
            const int cgx = (tiles_x + 3) >> 2;
            float lim = 0.f;
            for (int cy = ty0 >> 2; cy <= ty1 >> 2; ++cy)
                for (int cx = tx0 >> 2; cx <= tx1 >> 2; ++cx)
                    lim = fmaxf(lim, __ldg(coarse + cy * cgx + cx));
            keep = !(P.tc[2] > (T)lim);
        }
    }
    valid[i] = keep;
    depth_val[i] = (uint32_t)i;
    if (!keep) {
        store_depth_key<T>(depth_key, i, (T)0, false);
        return;
    }
    {
        T sh[48];
        load_sh(shc, i, sh);
        project_color(cam, p, sh, P);
    }
    T rec[12];
    rec[R_MX] = P.m0; rec[R_MY] = P.m1;
    rec[R_A] = P.inv[0]; rec[R_B] = P.inv[1]; rec[R_C] = P.inv[3];
    rec[R_OP] = P.o; rec[R_QC] = P.qcut; rec[R_RAD] = P.radius;
    rec[R_C0] = P.col[0]; rec[R_C1] = P.col[1]; rec[R_C2] = P.col[2];
    rec[R_DEP] = P.tc[2];
    store_record(records, i, rec);
    // a row whose cutoff box misses the image has no pair (binning's
    // tile_rect test, the same float expression): it keeps its record but
    // sorts with the invalid rows, so a bounded sort can leave it out
    const T Wm1 = (T)(cam.width - 1), Hm1 = (T)(cam.height - 1), rr = P.radius;
    const bool onscreen = (P.m0 + rr >= (T)0) && (P.m0 - rr <= Wm1) && (P.m1 + rr >= (T)0) &&
                          (P.m1 - rr <= Hm1);
    store_depth_key<T>(depth_key, i, P.tc[2], onscreen);
    if (ex.cov2d) for (int j = 0; j < 4; ++j) ((T *)ex.cov2d)[4 * i + j] = P.c2[j];
    if (ex.inv_cov2d) for (int j = 0; j < 4; ++j) ((T *)ex.inv_cov2d)[4 * i + j] = P.inv[j];
    if (ex.t_cam) for (int j = 0; j < 3; ++j) ((T *)ex.t_cam)[3 * i + j] = P.tc[j];
    if (ex.t_clamped) for (int j = 0; j < 3; ++j) ((T *)ex.t_clamped)[3 * i + j] = P.tcl[j];
    if (ex.clamped_x) ex.clamped_x[i] = P.clx;
    if (ex.clamped_y) ex.clamped_y[i] = P.cly;
    if (ex.view_dir) for (int j = 0; j < 3; ++j) ((T *)ex.view_dir)[3 * i + j] = P.vd[j];
    if (ex.basis) for (int j = 0; j < 16; ++j) ((T *)ex.basis)[16 * i + j] = P.basis[j];
    if (ex.color_raw) for (int j = 0; j < 3; ++j) ((T *)ex.color_raw)[3 * i + j] = P.craw[j];
    if (ex.mean2d) { ((T *)ex.mean2d)[2 * i] = P.m0; ((T *)ex.mean2d)[2 * i + 1] = P.m1; }
    if (ex.depth) ((T *)ex.depth)[i] = P.tc[2];
    if (ex.color) for (int j = 0; j < 3; ++j) ((T *)ex.color)[3 * i + j] = P.col[j];
    if (ex.opacity) ((T *)ex.opacity)[i] = P.o;
    if (ex.radius_cut) ((T *)ex.radius_cut)[i] = P.radius;
    if (ex.q_cut) ((T *)ex.q_cut)[i] = P.qcut;
}

template <typename T>
__global__ void pack_kernel(int64_t m, const T *__restrict__ mean2d, const T *__restrict__ inv,
                            const T *__restrict__ op, const T *__restrict__ qc,
                            const T *__restrict__ rad, const T *__restrict__ col,
                            const T *__restrict__ dep, T *__restrict__ records,
                            uint8_t *__restrict__ valid, void *__restrict__ depth_key,
                            uint32_t *__restrict__ depth_val)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    T rec[12];
    rec[R_MX] = mean2d[2 * i]; rec[R_MY] = mean2d[2 * i + 1];
    rec[R_A] = inv[4 * i]; rec[R_B] = inv[4 * i + 1]; rec[R_C] = inv[4 * i + 3];
    rec[R_OP] = op[i]; rec[R_QC] = qc[i]; rec[R_RAD] = rad[i];
    rec[R_C0] = col[3 * i]; rec[R_C1] = col[3 * i + 1]; rec[R_C2] = col[3 * i + 2];
    rec[R_DEP] = dep[i];
    store_record(records, i, rec);
    valid[i] = 1;
    store_depth_key<T>(depth_key, i, dep[i], true);
    depth_val[i] = (uint32_t)i;
}

// a7 from explicit SplatScreen fields (compact rows), accumulating into the
// map rows with atomics (np.add.at, backward.py:495-499)
template <typename T>
__global__ void __launch_bounds__(128) chain_screen_kernel(
    int64_t m, const int64_t *__restrict__ src, const T *__restrict__ pos,
    const T *__restrict__ ls, const T *__restrict__ rot, const T *__restrict__ shc,
    const T *__restrict__ s_inv, const T *__restrict__ s_tc, const T *__restrict__ s_tcl,
    const T *__restrict__ s_vd, const T *__restrict__ s_basis, const T *__restrict__ s_craw,
    const T *__restrict__ s_op, const uint8_t *__restrict__ s_clx,
    const uint8_t *__restrict__ s_cly, const T *__restrict__ dmean, const T *__restrict__ dconic,
    const T *__restrict__ dopac, const T *__restrict__ dcolor, CamT<T> cam, T *__restrict__ g_pos,
    T *__restrict__ g_ls, T *__restrict__ g_rot, T *__restrict__ g_ol, T *__restrict__ g_sh)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int64_t n = src[r];
    ChainIn<T> in;
    for (int j = 0; j < 4; ++j) in.inv[j] = s_inv[4 * r + j];
    for (int j = 0; j < 3; ++j) {
        in.tc[j] = s_tc[3 * r + j];
        in.tcl[j] = s_tcl[3 * r + j];
        in.vd[j] = s_vd[3 * r + j];
        in.craw[j] = s_craw[3 * r + j];
    }
    for (int k = 0; k < 16; ++k) in.basis[k] = s_basis[16 * r + k];
    in.o = s_op[r];
    in.clx = s_clx[r];
    in.cly = s_cly[r];
    const T p[3] = {pos[3 * n], pos[3 * n + 1], pos[3 * n + 2]};
    const T l[3] = {ls[3 * n], ls[3 * n + 1], ls[3 * n + 2]};
    const T q[4] = {rot[4 * n], rot[4 * n + 1], rot[4 * n + 2], rot[4 * n + 3]};
    T sh[48];
    load_sh(shc, n, sh);
    const T dm[2] = {dmean[2 * r], dmean[2 * r + 1]};
    const T dc3[3] = {dconic[3 * r], dconic[3 * r + 1], dconic[3 * r + 2]};
    const T dcol[3] = {dcolor[3 * r], dcolor[3 * r + 1], dcolor[3 * r + 2]};
    ChainOut<T> o;
    chain_row(cam, in, p, l, q, sh, dm, dc3, dopac[r], dcol, o);
    for (int j = 0; j < 3; ++j) atomicAdd(g_pos + 3 * n + j, o.dpos[j]);
    for (int j = 0; j < 3; ++j) atomicAdd(g_ls + 3 * n + j, o.dls[j]);
    for (int j = 0; j < 4; ++j) atomicAdd(g_rot + 4 * n + j, o.dq[j]);
    atomicAdd(g_ol + n, o.dlogit);
    for (int k = 0; k < 16; ++k)
        for (int c = 0; c < 3; ++c) atomicAdd(g_sh + 48 * n + 3 * k + c, in.basis[k] * o.draw[c]);
}

// a7 for map-indexed rows: recompute the screen quantities from parameters.
template <typename T>
__global__ void __launch_bounds__(128) chain_rows_kernel(
    int64_t n, const uint8_t *__restrict__ valid, const T *__restrict__ pos,
    const T *__restrict__ ls, const T *__restrict__ rot, const T *__restrict__ ol,
    const T *__restrict__ shc, CamT<T> cam, const T *__restrict__ dmean,
    const T *__restrict__ dconic, const T *__restrict__ dopac, const T *__restrict__ dcolor,
    T *__restrict__ g_pos, T *__restrict__ g_ls, T *__restrict__ g_rot, T *__restrict__ g_ol,
    T *__restrict__ g_sh, int accumulate)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    using V = typename Vec4<T>::type;
    if (accumulate) {
        // keyframe-batch mode: add this view's gradient to the
        // running sum; rows no pixel reached contribute exactly zero
        if (!valid[i]) return;
        const T dm[2] = {dmean[2 * i], dmean[2 * i + 1]};
        const T dc3[3] = {dconic[3 * i], dconic[3 * i + 1], dconic[3 * i + 2]};
        const T dcol[3] = {dcolor[3 * i], dcolor[3 * i + 1], dcolor[3 * i + 2]};
        const T dop = dopac[i];
        if (dm[0] == (T)0 && dm[1] == (T)0 && dc3[0] == (T)0 && dc3[1] == (T)0 &&
            dc3[2] == (T)0 && dop == (T)0 && dcol[0] == (T)0 && dcol[1] == (T)0 &&
            dcol[2] == (T)0)
            return;
        const T p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        const T l[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
        const T q[4] = {rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]};
        T sh[48];
        load_sh(shc, i, sh);
        Proj<T> P;
        project_row(cam, p, l, q, ol[i], sh, true, P);
        ChainIn<T> in;
        for (int j = 0; j < 4; ++j) in.inv[j] = P.inv[j];
        for (int j = 0; j < 3; ++j) {
            in.tc[j] = P.tc[j]; in.tcl[j] = P.tcl[j]; in.vd[j] = P.vd[j]; in.craw[j] = P.craw[j];
        }
        for (int k = 0; k < 16; ++k) in.basis[k] = P.basis[k];
        in.o = P.o; in.clx = P.clx; in.cly = P.cly;
        ChainOut<T> o;
        chain_row(cam, in, p, l, q, sh, dm, dc3, dop, dcol, o);
        for (int j = 0; j < 3; ++j) { g_pos[3 * i + j] += o.dpos[j]; g_ls[3 * i + j] += o.dls[j]; }
        for (int j = 0; j < 4; ++j) g_rot[4 * i + j] += o.dq[j];
        g_ol[i] += o.dlogit;
        for (int k = 0; k < 16; ++k)
            for (int c = 0; c < 3; ++c) g_sh[48 * i + 3 * k + c] += in.basis[k] * o.draw[c];
        return;
    }
    if (!valid[i]) {
        for (int j = 0; j < 3; ++j) { g_pos[3 * i + j] = (T)0; g_ls[3 * i + j] = (T)0; }
        for (int j = 0; j < 4; ++j) g_rot[4 * i + j] = (T)0;
        g_ol[i] = (T)0;
        V z;
        memset(&z, 0, sizeof(V));
        V *gs = reinterpret_cast<V *>(g_sh + 48 * i);
        for (int k = 0; k < 48 * (int)sizeof(T) / (int)sizeof(V); ++k) gs[k] = z;
        return;
    }
    const T p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    const T l[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
    const T q[4] = {rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]};
    T sh[48];
    load_sh(shc, i, sh);
    Proj<T> P;
    project_row(cam, p, l, q, ol[i], sh, true, P);
    ChainIn<T> in;
    for (int j = 0; j < 4; ++j) in.inv[j] = P.inv[j];
    for (int j = 0; j < 3; ++j) {
        in.tc[j] = P.tc[j]; in.tcl[j] = P.tcl[j]; in.vd[j] = P.vd[j]; in.craw[j] = P.craw[j];
    }
    for (int k = 0; k < 16; ++k) in.basis[k] = P.basis[k];
    in.o = P.o; in.clx = P.clx; in.cly = P.cly;
    const T dm[2] = {dmean[2 * i], dmean[2 * i + 1]};
    const T dc3[3] = {dconic[3 * i], dconic[3 * i + 1], dconic[3 * i + 2]};
    const T dcol[3] = {dcolor[3 * i], dcolor[3 * i + 1], dcolor[3 * i + 2]};
    ChainOut<T> o;
    chain_row(cam, in, p, l, q, sh, dm, dc3, dopac[i], dcol, o);
    for (int j = 0; j < 3; ++j) { g_pos[3 * i + j] = o.dpos[j]; g_ls[3 * i + j] = o.dls[j]; }
    for (int j = 0; j < 4; ++j) g_rot[4 * i + j] = o.dq[j];
    g_ol[i] = o.dlogit;
    T gs[48];
    for (int k = 0; k < 16; ++k)
        for (int c = 0; c < 3; ++c) gs[3 * k + c] = in.basis[k] * o.draw[c];
    V *dst = reinterpret_cast<V *>(g_sh + 48 * i);
    for (int k = 0; k < 48 * (int)sizeof(T) / (int)sizeof(V); ++k) dst[k] = reinterpret_cast<V *>(gs)[k];
}

}  // namespace sb

using namespace sb;

extern "C" int32_t sb_frustum_mask(int32_t dtype, int64_t n, const void *positions,
                                   const sb_camera_t *cam, double near_, double margin,
                                   uint8_t *out, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(cam != nullptr, "cam is NULL");
    if (n == 0) return SB_OK;
    const unsigned g = grid_for(n, 256);
    if (dtype == SB_F32)
        frustum_kernel<float><<<g, 256, 0, as_stream(stream)>>>(
            n, (const float *)positions, make_cam<float>(*cam, near_, 0.0, margin), out);
    else
        frustum_kernel<double><<<g, 256, 0, as_stream(stream)>>>(
            n, (const double *)positions, make_cam<double>(*cam, near_, 0.0, margin), out);
    return check_launch("frustum_kernel");
}

extern "C" int32_t sb_preprocess_fwd(int32_t dtype, int64_t n, const void *positions,
                                     const void *log_scales, const void *rotations,
                                     const void *opacity_logits, const void *sh_coeffs,
                                     const uint8_t *select, const sb_camera_t *cam, double near_,
                                     double dilation, double margin, void *records,
                                     uint8_t *valid, void *depth_key, uint32_t *depth_val,
                                     uint8_t *frustum, const sb_screen_extras_t *extras,
                                     const float *coarse_depth_limit, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(cam != nullptr, "cam is NULL");
    SB_REQUIRE(n < 0xFFFFFFFFll, "too many rows");
    if (n == 0) return SB_OK;
    sb_screen_extras_t ex;
    memset(&ex, 0, sizeof(ex));
    if (extras) ex = *extras;
    const unsigned g = grid_for(n, 128);
    if (dtype == SB_F32)
        preprocess_fwd_kernel<float><<<g, 128, 0, as_stream(stream)>>>(
            n, (const float *)positions, (const float *)log_scales, (const float *)rotations,
            (const float *)opacity_logits, (const float *)sh_coeffs, select,
            make_cam<float>(*cam, near_, dilation, margin), (float *)records, valid, depth_key,
            depth_val, frustum, ex, coarse_depth_limit);
    else
        preprocess_fwd_kernel<double><<<g, 128, 0, as_stream(stream)>>>(
            n, (const double *)positions, (const double *)log_scales, (const double *)rotations,
            (const double *)opacity_logits, (const double *)sh_coeffs, select,
            make_cam<double>(*cam, near_, dilation, margin), (double *)records, valid, depth_key,
            depth_val, frustum, ex, coarse_depth_limit);
    return check_launch("preprocess_fwd_kernel");
}

extern "C" int32_t sb_pack_records(int32_t dtype, int64_t m, const void *mean2d,
                                   const void *inv_cov2d, const void *opacity, const void *q_cut,
                                   const void *radius_cut, const void *color, const void *depth,
                                   void *records, uint8_t *valid, void *depth_key,
                                   uint32_t *depth_val, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    if (m == 0) return SB_OK;
    const unsigned g = grid_for(m, 256);
#define PACK_ARGS(T)                                                                        \
    m, (const T *)mean2d, (const T *)inv_cov2d, (const T *)opacity, (const T *)q_cut,         \
        (const T *)radius_cut, (const T *)color, (const T *)depth, (T *)records, valid,       \
        depth_key, depth_val
    if (dtype == SB_F32) pack_kernel<float><<<g, 256, 0, as_stream(stream)>>>(PACK_ARGS(float));
    else pack_kernel<double><<<g, 256, 0, as_stream(stream)>>>(PACK_ARGS(double));
#undef PACK_ARGS
    return check_launch("pack_kernel");
}

extern "C" int32_t sb_preprocess_bwd(int32_t dtype, int64_t m, const int64_t *src,
                                     const void *positions, const void *log_scales,
                                     const void *rotations, const void *sh_coeffs,
                                     const sb_chain_screen_t *screen, const void *d_mean2d,
                                     const void *d_conic, const void *d_opacity,
                                     const void *d_color, const sb_camera_t *cam,
                                     void *g_position, void *g_log_scale, void *g_rotation,
                                     void *g_opacity_logit, void *g_sh, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(cam != nullptr && screen != nullptr, "cam/screen is NULL");
    if (m == 0) return SB_OK;
    const unsigned g = grid_for(m, 128);
#define CHAIN_ARGS(T)                                                                        \
    m, src, (const T *)positions, (const T *)log_scales, (const T *)rotations,                 \
        (const T *)sh_coeffs, (const T *)screen->inv_cov2d, (const T *)screen->t_cam,          \
        (const T *)screen->t_clamped, (const T *)screen->view_dir, (const T *)screen->basis,   \
        (const T *)screen->color_raw, (const T *)screen->opacity, screen->clamped_x,           \
        screen->clamped_y, (const T *)d_mean2d, (const T *)d_conic, (const T *)d_opacity,      \
        (const T *)d_color, make_cam<T>(*cam, 0.01, 0.3, 0.1), (T *)g_position,               \
        (T *)g_log_scale, (T *)g_rotation, (T *)g_opacity_logit, (T *)g_sh
    if (dtype == SB_F32) chain_screen_kernel<float><<<g, 128, 0, as_stream(stream)>>>(CHAIN_ARGS(float));
    else chain_screen_kernel<double><<<g, 128, 0, as_stream(stream)>>>(CHAIN_ARGS(double));
#undef CHAIN_ARGS
    return check_launch("chain_screen_kernel");
}

extern "C" int32_t sb_preprocess_bwd_rows(int32_t dtype, int64_t n, const uint8_t *valid,
                                          const void *positions, const void *log_scales,
                                          const void *rotations, const void *opacity_logits,
                                          const void *sh_coeffs, const sb_camera_t *cam,
                                          double dilation, const void *d_mean2d,
                                          const void *d_conic, const void *d_opacity,
                                          const void *d_color, void *g_position,
                                          void *g_log_scale, void *g_rotation,
                                          void *g_opacity_logit, void *g_sh, int32_t accumulate,
                                          void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(cam != nullptr, "cam is NULL");
    if (n == 0) return SB_OK;
    const unsigned g = grid_for(n, 128);
#define ROWS_ARGS(T)                                                                         \
    n, valid, (const T *)positions, (const T *)log_scales, (const T *)rotations,               \
        (const T *)opacity_logits, (const T *)sh_coeffs, make_cam<T>(*cam, -HUGE_VAL, dilation, 0.1), \
        (const T *)d_mean2d, (const T *)d_conic, (const T *)d_opacity, (const T *)d_color,     \
        (T *)g_position, (T *)g_log_scale, (T *)g_rotation, (T *)g_opacity_logit, (T *)g_sh,   \
        (int)accumulate
    if (dtype == SB_F32) chain_rows_kernel<float><<<g, 128, 0, as_stream(stream)>>>(ROWS_ARGS(float));
    else chain_rows_kernel<double><<<g, 128, 0, as_stream(stream)>>>(ROWS_ARGS(double));
#undef ROWS_ARGS
    return check_launch("chain_rows_kernel");
}
