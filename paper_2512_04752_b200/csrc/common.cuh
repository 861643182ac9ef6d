// Shared plumbing for the rlhfspec_core C ABI: status codes, thread-local error text,
// CUDA error mapping. No arithmetic of the method lives here.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "rlhfspec_core.h"

namespace rs {

void set_error(const char* fmt, ...);
void bind_device(const void* device_ptr);   // make the owner of device_ptr the current device

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace rs

#define RS_REQUIRE(cond, code, ...)             \
    do {                                        \
        if (!(cond)) {                          \
            ::rs::set_error(__VA_ARGS__);       \
            return (code);                      \
        }                                       \
    } while (0)

#define RS_CUDA_CHECK(expr)                                                              \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess) {                                                         \
            ::rs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
            return RS_ERR_CUDA;                                                          \
        }                                                                                \
    } while (0)

#define RS_LAUNCH_CHECK() RS_CUDA_CHECK(cudaGetLastError())
