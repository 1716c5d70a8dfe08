// Throughput of small cp.async.bulk (TMA, UBLKCP) gathers from 400-byte rows: BYTES per copy,
// every lane of a warp issuing its own copy (tools/README.md).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_tp bulk_tp.cu && ./bulk_tp
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned s32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int BYTES, int NPL>
__global__ void __launch_bounds__(128) gather(const float *table, const int *rows, int n_idx, int iters,
                                              unsigned long long *sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long mbar[4];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned mb = s32(&mbar[w]);
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    __syncthreads();
    const unsigned base = s32(smem) + BYTES * tid;
    const int gw = (blockIdx.x * blockDim.x + tid) / 32;
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(32 * NPL * BYTES));
        __syncwarp();
#pragma unroll
        for (int e = 0; e < NPL; ++e) {
            const int ent = (gw * 131 + it * 17 + e) * 32 + lane;
            const int row = rows[ent % n_idx];
            const float *src = table + (size_t)row * 100 + ((it * 8) % 64 & ~(BYTES / 4 - 1));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             base + BYTES * 128u * e),
                         "l"(src), "r"(BYTES), "r"(mb)
                         : "memory");
        }
        unsigned ok = 0;
        while (!ok)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok)
                         : "r"(mb), "r"(it & 1)
                         : "memory");
        acc += reinterpret_cast<const unsigned *>(smem)[tid * 4 + (it & 3)];
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <int BYTES, int NPL>
void run(const float *table, const int *rows, int n_idx, unsigned long long *sink, int warps_per_sm) {
    const int iters = 500, sms = 148;
    const int blocks = sms * warps_per_sm / 4;
    const size_t smem = (size_t)BYTES * 128 * NPL;
    cudaFuncSetAttribute(gather<BYTES, NPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<BYTES, NPL><<<blocks, 128, smem>>>(table, rows, n_idx, 20, sink);
    cudaEventRecord(a);
    gather<BYTES, NPL><<<blocks, 128, smem>>>(table, rows, n_idx, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cycles = ms * 1e-3 * clk * 1e3;
    const double copies = (double)blocks * 128 * iters * NPL;
    printf("bulk %3d B npl %d warps/SM %2d: %.3f ms  %.2f cycles per copy per SM  %.2f B/cycle/SM  %.2f TB/s  (%s)\n", BYTES, NPL,
           warps_per_sm, ms, cycles / (copies / sms), copies * BYTES / sms / cycles, copies * BYTES / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int n_rows = 102660, n_idx = 1 << 22;
    float *table;
    int *rows;
    unsigned long long *sink;
    cudaMalloc(&table, (size_t)n_rows * 400);
    cudaMemset(table, 0, (size_t)n_rows * 400);
    std::vector<int> h(n_idx);
    srand(1);
    for (auto &x : h) x = rand() % n_rows;
    cudaMalloc(&rows, n_idx * sizeof(int));
    cudaMemcpy(rows, h.data(), n_idx * sizeof(int), cudaMemcpyHostToDevice);
    cudaMalloc(&sink, 8);
    for (int w : {8, 16}) {
        run<16, 4>(table, rows, n_idx, sink, w);
        run<32, 4>(table, rows, n_idx, sink, w);
        run<64, 4>(table, rows, n_idx, sink, w);
        run<128, 2>(table, rows, n_idx, sink, w);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
