// Throughput of 16-byte cp.async gathers from an L2-resident table of 400-byte rows, by how
// many lanes of one instruction share a 128-byte line (tools/README.md).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_tp gather_tp.cu && ./gather_tp
// SHARE = 1: every lane its own row (32 lines per instruction, 16 B used of each 32-B sector:
// the solver kernels' gather); 2: lane pairs fetch the two halves of one sector; 4 / 8: 64 / 128
// contiguous bytes of one row.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(unsigned s, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}

template <int SHARE, int NPL>
__global__ void __launch_bounds__(128) gather(const float *table, const int *rows, int n_rows_idx, int iters,
                                              unsigned long long *sink) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned base = (unsigned)__cvta_generic_to_shared(smem) + 16u * tid;
    const int gw = (blockIdx.x * blockDim.x + tid) / 32;
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int e = 0; e < NPL; ++e) {
            // entry handled by this lane group in this request
            const int ent = (gw * 131 + it * 17 + e) * (32 / SHARE) + lane / SHARE;
            const int row = rows[ent % n_rows_idx];
            const float *src = table + (size_t)row * 100 + ((it * 8) % 96 & ~(4 * SHARE - 1)) + 4 * (lane % SHARE);
            cp16(base + 16u * 128u * e, src);
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 1;\n" ::);
        acc += reinterpret_cast<const unsigned *>(smem)[tid * 4 + (it & 3)];
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    if (acc == 0x12345678u) *sink = acc;
}

template <int SHARE, int NPL>
void run(const float *table, const int *rows, int n_idx, unsigned long long *sink, int warps_per_sm) {
    const int iters = 2000, sms = 148;
    const int blocks = sms * warps_per_sm / 4;
    const size_t smem = 16 * 128 * NPL;
    cudaFuncSetAttribute(gather<SHARE, NPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<SHARE, NPL><<<blocks, 128, smem>>>(table, rows, n_idx, 50, sink);
    cudaEventRecord(a);
    gather<SHARE, NPL><<<blocks, 128, smem>>>(table, rows, n_idx, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cycles = ms * 1e-3 * clk * 1e3;
    const double req = (double)blocks * 4 * iters * NPL;       // warp instructions
    const double bytes = req * 32 * 16;
    printf("share %d npl %2d warps/SM %2d: %.3f ms  %.1f cycles per warp LDGSTS per SM  %.2f useful B/cycle/SM  %.2f TB/s useful\n",
           SHARE, NPL, warps_per_sm, ms, cycles / (req / sms), bytes / sms / cycles, bytes / (ms * 1e-3) / 1e12);
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
    for (int w : {8, 16, 32}) {
        run<1, 8>(table, rows, n_idx, sink, w);
        run<2, 8>(table, rows, n_idx, sink, w);
        run<4, 8>(table, rows, n_idx, sink, w);
        run<8, 8>(table, rows, n_idx, sink, w);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
