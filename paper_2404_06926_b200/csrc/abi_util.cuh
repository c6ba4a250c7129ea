// abi_util.cuh -- error reporting and dtype dispatch for the C ABI.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/splatb200.h"

namespace sb {

void set_error(const char *fmt, ...);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int32_t check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return SB_ERR_CUDA;
    }
    return SB_OK;
}

inline unsigned grid_for(int64_t n, int block)
{
    int64_t g = (n + block - 1) / block;
    return (unsigned)(g > 0 ? g : 1);
}

}  // namespace sb

#define SB_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t _e = (call);                                                   \
        if (_e != cudaSuccess) {                                                   \
            sb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                \
                          cudaGetErrorString(_e));                                 \
            return SB_ERR_CUDA;                                                    \
        }                                                                          \
    } while (0)

#define SB_REQUIRE(cond, ...)                                                      \
    do {                                                                           \
        if (!(cond)) {                                                             \
            sb::set_error(__VA_ARGS__);                                            \
            return SB_ERR_INVALID;                                                 \
        }                                                                          \
    } while (0)

#define SB_DTYPE_CHECK(dtype) \
    SB_REQUIRE((dtype) == SB_F32 || (dtype) == SB_F64, "unsupported dtype %d", (int)(dtype))
