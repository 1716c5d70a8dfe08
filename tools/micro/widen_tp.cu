// Throughput of the pass's per-entry operations on one B200 SM set:
// f32->f64 conversion (F2F) vs an integer bit-widen, DFMA, the fp64
// reciprocal seed (MUFU.RCP64H) and an fp32 MUFU.RCP seed.  Rates are for the
// whole loop body (ops/clk/SM = loop bodies per clock per SM).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double widen_int(float f) {
    const unsigned b = __float_as_uint(f);
    const unsigned hi = b ? (b >> 3) + 0x38000000u : 0u;
    return __hiloint2double((int)hi, (int)(b << 29));
}

template <int MODE>
__global__ void k(const float *in, double *out, int iters) {
    float f[8];
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { f[i] = in[(threadIdx.x + i) & 255]; acc[i] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) acc[i] += (double)f[i];                 // F2F + DADD
            if (MODE == 1) acc[i] += widen_int(f[i]);              // int widen + DADD
            if (MODE == 2) acc[i] = fma(acc[i], 1.0000001, 0.5);   // DFMA only
            if (MODE == 3) {                                        // MUFU.RCP64H seed + DADD
                double r;
                asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(acc[i] + 1.5));
                acc[i] += r;
            }
            if (MODE == 4) acc[i] += (double)__frcp_rn((float)(acc[i] + 1.5));  // F2F + MUFU.RCP + F2F + DADD
            f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);       // keep f live/varying
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *in; double *out;
    cudaMalloc(&in, 256 * 4); cudaMemset(in, 0x3f, 256 * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char *names[5] = {"F2F.F64.F32 + DADD", "int widen + DADD", "DFMA", "RCP64H seed + 2 DADD",
                            "f32 rcp seed (2 F2F) + DADD"};
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, threads>>>(in, out, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(in, out, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(in, out, iters);
            if (mode == 3) k<3><<<blocks, threads>>>(in, out, iters);
            if (mode == 4) k<4><<<blocks, threads>>>(in, out, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters * 8;
            if (rep) printf("%-22s %8.3f ms  %.1f ops/clk/SM (at %d MHz nominal)\n", names[mode], ms,
                            ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
