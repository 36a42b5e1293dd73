// common.cuh -- shared helpers for the sm_100a kernels and the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/cspq_b200.h"

namespace cspq {

// per-thread last-error message (cspq_last_error)
void set_error(const char *fmt, ...);
// host-side count of this library's kernel launches (cspq_launch_count): every launch site is
// followed by exactly one CSPQ_LAUNCH_CHECK
void count_launch();

#define CSPQ_CUDA_TRY(expr)                                                              \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess) {                                                         \
            ::cspq::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),    \
                              __FILE__, __LINE__);                                       \
            return CSPQ_E_CUDA;                                                          \
        }                                                                                \
    } while (0)

#define CSPQ_LAUNCH_CHECK()              \
    do {                                 \
        ::cspq::count_launch();          \
        CSPQ_CUDA_TRY(cudaGetLastError()); \
    } while (0)

#define CSPQ_REQUIRE(cond, code, ...)                                                    \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            ::cspq::set_error(__VA_ARGS__);                                              \
            return (code);                                                               \
        }                                                                                \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

__device__ __forceinline__ float pos_inf_f() { return __int_as_float(0x7f800000); }
__device__ __forceinline__ double pos_inf_d() { return __longlong_as_double(0x7ff0000000000000LL); }

// 3-input minimum: one FMNMX3 on sm_100a.  NaN operands are ignored unless all are NaN.
__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// cp.async helpers (LDGSTS); zero-fill when src_bytes == 0
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes = 16) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, int src_bytes = 8) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, int src_bytes = 4) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace cspq
