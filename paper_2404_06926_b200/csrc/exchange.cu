// Packed gradient exchange of the keyframe batch step (batch.PackedBatchStep,
// SURVEY.md §8(e)): the rows some view reached are gathered from the flat
// map-layout gradient (group-major: positions 3, log_scales 3, rotations 4,
// opacity 1, sh 48 reals per row, each group n_pad rows) into a row-major
// [k, 59] buffer that one all-reduce carries, and scattered back after it.
// One launch each, one warp per packed row.
// Slots may repeat a dump row (the fixed-capacity packing pads with row n,
// whose gradient is zero everywhere and which Adam never reads).
#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

constexpr int kRowReals = 59;

// One warp per packed row (grid-stride over rows): the row id and its held
// flag are loaded once and broadcast, lane l moves reals l and l + 32 -- the
// packed side is one contiguous 236 B run, the SH slice another (the narrow
// groups' slices stay sector-granular in the group-major layout).
// kPack with rows_held (nullable): a row not marked there packs as zeros (a
// first-touch gradient buffer holds valid values on the rows this rank
// reached only, sb_chain_accumulate)
template <typename T, bool kPack>
__global__ void __launch_bounds__(256) k_pack_rows(int64_t n_pad, T *__restrict__ flat,
                                                   const int64_t *__restrict__ pos, int64_t k,
                                                   T *__restrict__ packed,
                                                   const uint8_t *__restrict__ rows_held)
{
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // each lane's two columns: their flat group start and width, once
    int64_t off[2];
    int w[2], c0[2];
    bool has[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int col = lane + 32 * h;
        has[h] = col < kRowReals;
        const int cc = has[h] ? col : 0;
        int start, wd;
        if (cc < 3) { start = 0; wd = 3; }
        else if (cc < 6) { start = 3; wd = 3; }
        else if (cc < 10) { start = 6; wd = 4; }
        else if (cc < 11) { start = 10; wd = 1; }
        else { start = 11; wd = 48; }
        off[h] = (int64_t)start * n_pad;
        w[h] = wd;
        c0[h] = cc - start;
    }
    for (int64_t slot = (((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); slot < k;
         slot += nw) {
        const int64_t row = __ldg(pos + slot);
        const bool held = !kPack || !rows_held || __ldg(rows_held + row);
        T *prow = packed + slot * kRowReals;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!has[h]) continue;
            const int64_t f = off[h] + row * w[h] + c0[h];
            if (kPack) prow[lane + 32 * h] = held ? flat[f] : (T)0;
            else flat[f] = prow[lane + 32 * h];
        }
    }
}

template <typename T, bool kPack>
int32_t pack_rows(int64_t n_pad, void *flat, const int64_t *pos, int64_t k, void *packed,
                  const uint8_t *rows_held, void *stream)
{
    if (k == 0) return SB_OK;
    const int64_t blocks = std::min<int64_t>((k + 7) / 8, 148 * 8);   // 8 rows per CTA
    k_pack_rows<T, kPack><<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        n_pad, static_cast<T *>(flat), pos, k, static_cast<T *>(packed), rows_held);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

}  // namespace sb

extern "C" int32_t sb_pack_rows(int32_t dtype, int64_t n_pad, const void *flat,
                                const int64_t *pos, int64_t k, void *packed,
                                const uint8_t *rows_held, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(n_pad >= 0 && k >= 0, "sb_pack_rows: negative size");
    void *f = const_cast<void *>(flat);
    return dtype == SB_F32
               ? sb::pack_rows<float, true>(n_pad, f, pos, k, packed, rows_held, stream)
               : sb::pack_rows<double, true>(n_pad, f, pos, k, packed, rows_held, stream);
}

extern "C" int32_t sb_unpack_rows(int32_t dtype, int64_t n_pad, void *flat, const int64_t *pos,
                                  int64_t k, const void *packed, void *stream)
{
    SB_DTYPE_CHECK(dtype);
    SB_REQUIRE(n_pad >= 0 && k >= 0, "sb_unpack_rows: negative size");
    void *p = const_cast<void *>(packed);
    return dtype == SB_F32 ? sb::pack_rows<float, false>(n_pad, flat, pos, k, p, nullptr, stream)
                           : sb::pack_rows<double, false>(n_pad, flat, pos, k, p, nullptr, stream);
}
