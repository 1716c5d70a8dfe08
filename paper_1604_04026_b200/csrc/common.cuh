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

// Scratch of the plan-building helpers comes from the device's default
// stream-ordered pool (cudaMallocAsync).  Its default release threshold of 0
// hands freed memory back to the driver at every synchronisation, so the next
// plan re-maps GBs (seen as 0.05-0.5 s stalls of a C4 transpose); keep it in
// the pool instead (once per device; the scratch stays reserved in-process).
inline cudaError_t keep_async_pool() {
    static bool kept[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess || dev < 0 || dev >= 64 || kept[dev]) return e;
    cudaMemPool_t pool;
    e = cudaDeviceGetDefaultMemPool(&pool, dev);
    if (e != cudaSuccess) return e;
    uint64_t keep = UINT64_MAX;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if (e == cudaSuccess) kept[dev] = true;
    return e;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size,
// so launch paths replayed under CUDA-graph capture issue no attribute calls.
cudaError_t ensure_smem(const void *fn, size_t bytes);

constexpr unsigned FULL_MASK = 0xffffffffu;

// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): one 128-bit block of the
// counter c under key (k0, k1); the published round function, key bumped
// between rounds.  Shared by the kernels and the host (klnmf_chunk_order).
__host__ __device__ inline void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
    for (int rnd = 0; rnd < 10; ++rnd) {
        if (rnd > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c[0] = hi1 ^ c[1] ^ k0;
        c[1] = lo1;
        c[2] = hi0 ^ c[3] ^ k1;
        c[3] = lo0;
    }
}

constexpr int MAX_CHUNKS = 64;  // 4-coordinate chunks of the largest padded rank (256)

// Counter-mode visit order of a subproblem's n 4-coordinate chunks:
// Fisher-Yates from the top, step k = n-1-i using word k of the Philox stream
// (counter (k/4, item, iter, side), key (seed lo, seed hi)), index
// (word * (i+1)) >> 32.  Identical on host and device.
__host__ __device__ inline void chunk_order(uint64_t seed, uint32_t iter, uint32_t item, uint32_t side, int n,
                                            uint8_t *order) {
    for (int i = 0; i < n; ++i) order[i] = (uint8_t)i;
    uint32_t w[4] = {0, 0, 0, 0};
    for (int i = n - 1, k = 0; i >= 1; --i, ++k) {
        if ((k & 3) == 0) {
            w[0] = (uint32_t)(k >> 2);
            w[1] = item;
            w[2] = iter;
            w[3] = side;
            philox4x32_10(w, (uint32_t)seed, (uint32_t)(seed >> 32));
        }
        const int wk = k & 3;  // register selects, no local-memory array
        const uint32_t word = wk == 0 ? w[0] : (wk == 1 ? w[1] : (wk == 2 ? w[2] : w[3]));
        const uint32_t j = (uint32_t)(((uint64_t)word * (uint32_t)(i + 1)) >> 32);
        const uint8_t tmp = order[i];
        order[i] = order[j];
        order[j] = tmp;
    }
}

// Counter-mode visit order of the 4 coordinates inside the chunk visited at
// position `pos` of subproblem `item`: Fisher-Yates over (0,1,2,3) from the
// top, driven by word pos%4 of the Philox block with counter
// (0x100 + pos/4, item, iter, side) -- disjoint from chunk_order's counters
// (< 16); each step takes the high word of word*(i+1) and continues with the
// low word.  Packed 2 bits per slot: slot c visits coordinate
// (perm >> 2c) & 3 of the chunk.  Identical on host and device.
constexpr uint32_t PERM4_IDENTITY = 0xE4u;  // 0 | 1<<2 | 2<<4 | 3<<6
__host__ __device__ inline uint32_t chunk_perm4(uint64_t seed, uint32_t iter, uint32_t item, uint32_t side, int pos) {
    uint32_t w[4] = {0x100u + (uint32_t)(pos >> 2), item, iter, side};
    philox4x32_10(w, (uint32_t)seed, (uint32_t)(seed >> 32));
    const int wk = pos & 3;
    uint32_t word = wk == 0 ? w[0] : (wk == 1 ? w[1] : (wk == 2 ? w[2] : w[3]));
    uint32_t perm = PERM4_IDENTITY;
    for (int i = 3; i >= 1; --i) {
        const uint64_t m = (uint64_t)word * (uint32_t)(i + 1);
        const uint32_t j = (uint32_t)(m >> 32);
        word = (uint32_t)m;
        const uint32_t a = (perm >> (2 * i)) & 3u, b = (perm >> (2 * j)) & 3u;
        perm &= ~((3u << (2 * i)) | (3u << (2 * j)));
        perm |= (b << (2 * i)) | (a << (2 * j));
    }
    return perm;
}

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
