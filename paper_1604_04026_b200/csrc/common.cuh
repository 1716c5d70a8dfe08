// Internal helpers shared by the libklnmf translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/klnmf.h"

namespace klnmf {

// Records a CUDA error message for klnmf_last_error(); returns the code.
int set_error(cudaError_t err, const char *where);
int set_error_msg(int code, const char *msg);

#define KLNMF_CHECK(expr)                                         \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return ::klnmf::set_error(_e, #expr); \
    } while (0)

#define KLNMF_CHECK_LAUNCH(where)                                 \
    do {                                                          \
        cudaError_t _e = cudaGetLastError();                      \
        if (_e != cudaSuccess) return ::klnmf::set_error(_e, where); \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size,
// so launch paths replayed under CUDA-graph capture issue no attribute calls.
cudaError_t ensure_smem(const void *fn, size_t bytes);

constexpr unsigned FULL_MASK = 0xffffffffu;

__device__ __forceinline__ float4 ldg_f4(const float *p) {
    return __ldg(reinterpret_cast<const float4 *>(p));
}

__device__ __forceinline__ float f4_get(const float4 &v, int c) {
    return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// Deterministic sum of one double across a block (fixed tree); result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum_det(double v, double *sh /* NT/32 */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double tot = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NT / 32; ++i) tot += sh[i];
    }
    __syncthreads();
    return tot;
}

}  // namespace klnmf
