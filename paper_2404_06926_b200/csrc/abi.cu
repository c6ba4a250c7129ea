// abi.cu -- library identity, error reporting, and the map-growth selector.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// Map growth selector, Mapper.expand mapper.py:262-274: points are projected
// in float64 (BLAS FMA chain for the transform), nearest pixel floor(u + 0.5),
// then gated by the expansion mask O < tau (mapper.py:245-250) of the
// keyframe's render.
template <typename T>
__global__ void expand_select_kernel(int64_t k, const double *__restrict__ pts, sb_camera_t cam,
                                     double near_, const T *__restrict__ opacity, T tau,
                                     uint8_t *__restrict__ sel)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= k) return;
    const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    double pc[3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
        pc[j] = __fma_rn(z, cam.W[3 * j + 2], __fma_rn(y, cam.W[3 * j + 1], x * cam.W[3 * j])) + cam.t[j];
    bool ok = pc[2] > near_;
    const double u = cam.fx * pc[0] / pc[2] + cam.cx;
    const double v = cam.fy * pc[1] / pc[2] + cam.cy;
    const double fc = floor(u + 0.5), fr = floor(v + 0.5);
    ok = ok && fc >= 0.0 && fc < (double)cam.width && fr >= 0.0 && fr < (double)cam.height;
    if (ok) {
        const int64_t pix = (int64_t)fr * cam.width + (int64_t)fc;
        ok = opacity[pix] < tau;
    }
    sel[i] = ok;
}

// Depth-limit freshness gate (engine-side, no reference counterpart).  A
// keyframe's tile depth limits were recorded by its last forward blend; they
// stay usable while the map has been updated at most once since (the update
// of that same iteration), which is exactly the case of a keyframe stepped
// repeatedly or of a view in a repeated keyframe batch.  Otherwise other
// updates have changed the map and the iteration bins full lists (limits
// reset to +inf, re-recorded by its forward).  clock counts map updates
// (bumped by the caller once per update), stamp is the key's clock value at
// its last use.  Decided on the device, so graph replays stay correct.
__global__ void limits_gate_kernel(float *__restrict__ limits, int64_t count,
                                   int64_t *__restrict__ clock, int64_t *__restrict__ stamp,
                                   int bump)
{
    __shared__ bool stale;
    __shared__ int64_t now;
    if (threadIdx.x == 0) {
        const int64_t c = *clock + bump;
        now = c;
        stale = stamp == nullptr || c - *stamp > 1;
    }
    __syncthreads();
    if (limits && stale)
        for (int64_t i = threadIdx.x; i < count; i += blockDim.x) limits[i] = HUGE_VALF;
    __syncthreads();
    if (threadIdx.x == 0) {
        *clock = now;
        if (stamp) *stamp = now;
    }
}

}  // namespace sb

using namespace sb;

extern "C" int32_t sb_depth_limits_gate(float *limits, int64_t count, int64_t *clock,
                                        int64_t *stamp, int32_t bump, void *stream)
{
    SB_REQUIRE(clock != nullptr, "NULL clock");
    limits_gate_kernel<<<1, 1024, 0, as_stream(stream)>>>(limits, count, clock, stamp, (int)bump);
    return check_launch("limits_gate_kernel");
}

extern "C" int32_t sb_version(void) { return 11100; /* 1.11.0: gathered reached rows feed the chain rule (no adjoint zeroing) */ }

extern "C" const char *sb_last_error(void) { return g_err; }

extern "C" int32_t sb_expand_select(int64_t k, const double *points, const sb_camera_t *cam,
                                    double near_, int32_t dtype, const void *opacity_image,
                                    double mask_threshold, uint8_t *out_select, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(cam != nullptr, "cam is NULL");
    if (k == 0) return SB_OK;
    const unsigned g = grid_for(k, 256);
    if (dtype == SB_F32)
        expand_select_kernel<float><<<g, 256, 0, as_stream(stream)>>>(
            k, points, *cam, near_, (const float *)opacity_image, (float)mask_threshold, out_select);
    else
        expand_select_kernel<double><<<g, 256, 0, as_stream(stream)>>>(
            k, points, *cam, near_, (const double *)opacity_image, mask_threshold, out_select);
    return check_launch("expand_select_kernel");
}
