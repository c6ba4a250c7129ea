// Packed gradient exchange of the keyframe batch step (batch.PackedBatchStep,
// SURVEY.md §8(e)): the rows some view reached are gathered from the flat
// map-layout gradient (group-major: positions 3, log_scales 3, rotations 4,
// opacity 1, sh 48 reals per row, each group n_pad rows) into a row-major
// [k, 59] buffer that one all-reduce carries, and scattered back after it.
// One launch each, one thread per packed real: the packed side is coalesced,
// the flat side reads/writes each reached row's contiguous group slice.
// Slots may repeat a dump row (the fixed-capacity packing pads with row n,
// whose gradient is zero everywhere and which Adam never reads).
#include "abi_util.cuh"
#include "common.cuh"

namespace sb {

constexpr int kRowReals = 59;

__device__ __forceinline__ int64_t flat_index(int col, int64_t row, int64_t n_pad)
{
    // group starts (in reals) and widths: 0/3, 3/3, 6/4, 10/1, 11/48
    int start, w;
    if (col < 3) { start = 0; w = 3; }
    else if (col < 6) { start = 3; w = 3; }
    else if (col < 10) { start = 6; w = 4; }
    else if (col < 11) { start = 10; w = 1; }
    else { start = 11; w = 48; }
    return (int64_t)start * n_pad + row * w + (col - start);
}

// kPack with rows_held (nullable): a row not marked there packs as zeros (a
// first-touch gradient buffer holds valid values on the rows this rank
// reached only, sb_chain_accumulate)
template <typename T, bool kPack>
__global__ void __launch_bounds__(256) k_pack_rows(int64_t n_pad, T *__restrict__ flat,
                                                   const int64_t *__restrict__ pos, int64_t k,
                                                   T *__restrict__ packed,
                                                   const uint8_t *__restrict__ rows_held)
{
    const int64_t total = k * kRowReals;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = i / kRowReals;
        const int col = (int)(i - slot * kRowReals);
        const int64_t row = __ldg(pos + slot);
        const int64_t f = flat_index(col, row, n_pad);
        if (kPack) packed[i] = (!rows_held || __ldg(rows_held + row)) ? flat[f] : (T)0;
        else flat[f] = packed[i];
    }
}

template <typename T, bool kPack>
int32_t pack_rows(int64_t n_pad, void *flat, const int64_t *pos, int64_t k, void *packed,
                  const uint8_t *rows_held, void *stream)
{
    if (k == 0) return SB_OK;
    const int64_t total = k * kRowReals;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
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
