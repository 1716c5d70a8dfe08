// Device-side synthetic corpus generator.
//
// The planted-topic model of synth.py (BASELINE.json "configs") drawn on the
// GPU, so that C5-sized inputs (480M nonzeros) are built where they are used
// instead of in host numpy:
//   phi_t ~ Dirichlet(0.05 * n * pop)     (pop: uniform or Zipf(s))
//   theta_j ~ Dirichlet(0.1)              (drawn per document, on the fly)
//   L_j ~ Poisson(mean) | lognormal(mean, sigma), >= 1
//   L_j tokens: topic ~ theta_j, feature ~ phi_topic;  V[f, j] = count
// Randomness is counter-based (Philox4x32-10, common.cuh) keyed by the seed:
// every draw is a pure function of (purpose, index, attempt), so the matrix
// is deterministic and independent of launch geometry -- but a different
// stream than numpy's, i.e. the same distribution, not the host generator's
// matrix.  Aggregation: one uint64 key doc * n + feature per token, CUB radix
// sort, run-length encode, then the CSC arrays.
#include <cub/cub.cuh>

#include "common.cuh"

namespace klnmf {
namespace {

enum Purpose : uint32_t { P_PHI = 1, P_LEN = 2, P_THETA = 3, P_TOKEN = 4 };

struct Rng {
    uint64_t seed;
    __device__ __forceinline__ void block(uint32_t a, uint32_t b, uint32_t purpose, uint32_t attempt,
                                          uint32_t (&w)[4]) const {
        w[0] = a;
        w[1] = b;
        w[2] = purpose;
        w[3] = attempt;
        philox4x32_10(w, (uint32_t)seed, (uint32_t)(seed >> 32));
    }
};

// uniform in (0, 1) from two words (53 bits)
__device__ __forceinline__ double unit(uint32_t hi, uint32_t lo) {
    const uint64_t v = ((uint64_t)(hi >> 5) << 26) | (uint64_t)(lo >> 6);  // 27 + 26 bits
    return ((double)v + 0.5) * (1.0 / 9007199254740992.0);
}

// Gamma(shape, 1): Marsaglia & Tsang (2000); shape < 1 through
// Gamma(shape + 1) * U^(1/shape).  Returns log of the sample (tiny shapes
// underflow in the linear domain).
__device__ double log_gamma_sample(const Rng &rng, uint32_t a, uint32_t b, uint32_t purpose, double shape) {
    const bool boost = shape < 1.0;
    const double al = boost ? shape + 1.0 : shape;
    const double d = al - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
    uint32_t w[4];
    for (uint32_t att = 0;; ++att) {
        rng.block(a, b, purpose, att, w);
        const double u1 = unit(w[0], w[1]), u2 = unit(w[2], w[3]);
        const double x = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);  // Box-Muller
        const double t = 1.0 + c * x;
        if (t <= 0.0) continue;
        const double v = t * t * t;
        rng.block(a, b, purpose, att | 0x80000000u, w);
        const double u = unit(w[0], w[1]);
        if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) {
            double lg = log(d * v);
            if (boost) lg += log(unit(w[2], w[3])) / shape;
            return lg;
        }
    }
}

// phi: one block per topic: Gamma draws, normalisation, inclusive CDF (fp64)
template <int NT>
__global__ void phi_cdf_kernel(Rng rng, int64_t n, double zipf, double zipf_norm, double *cdf) {
    const int t = blockIdx.x;
    double *row = cdf + (int64_t)t * n;
    __shared__ double sh[NT / 32];
    // log-weights, max-shifted before exponentiation for the normalisation
    double mx = -1e300;
    for (int64_t i = threadIdx.x; i < n; i += NT) {
        const double pop = zipf > 0.0 ? pow((double)(i + 1), -zipf) / zipf_norm : 1.0 / (double)n;
        const double lg = log_gamma_sample(rng, (uint32_t)t, (uint32_t)i, P_PHI, 0.05 * (double)n * pop);
        row[i] = lg;
        mx = fmax(mx, lg);
    }
    // block max
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = sh[0];
    for (int q = 1; q < NT / 32; ++q) mx = fmax(mx, sh[q]);
    __syncthreads();
    // weights and a chunked inclusive scan (fixed order: deterministic)
    typedef cub::BlockScan<double, NT> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ double carry;
    if (threadIdx.x == 0) carry = 0.0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += NT) {
        const int64_t i = base + threadIdx.x;
        const double w = i < n ? exp(row[i] - mx) : 0.0;
        double inc, total;
        Scan(tmp).InclusiveSum(w, inc, total);
        const double c0 = carry;
        if (i < n) row[i] = c0 + inc;
        __syncthreads();
        if (threadIdx.x == 0) carry = c0 + total;
        __syncthreads();
    }
    // normalise; the last entry is pinned to exactly 1 by the thread that owns
    // it (a separate store from another thread would race with this one)
    const double tot = carry;
    for (int64_t i = threadIdx.x; i < n; i += NT) row[i] = i == n - 1 ? 1.0 : row[i] / tot;
}

__global__ void lengths_kernel(Rng rng, int64_t m, int kind, double mean, double sigma, int64_t *len) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[4];
        int64_t L;
        if (kind == 0) {  // Poisson (Knuth; the configs use it for mean 200 only)
            const double lim = exp(-mean);
            double p = 1.0;
            L = -1;
            uint32_t att = 0;
            do {
                rng.block((uint32_t)j, (uint32_t)(j >> 32), P_LEN, att++, w);
                p *= unit(w[0], w[1]);
                ++L;
                if (p > lim) {
                    p *= unit(w[2], w[3]);
                    ++L;
                }
            } while (p > lim);
        } else {  // lognormal with the stated mean: mu = log(mean) - sigma^2 / 2
            rng.block((uint32_t)j, (uint32_t)(j >> 32), P_LEN, 0, w);
            const double z = sqrt(-2.0 * log(unit(w[0], w[1]))) * cospi(2.0 * unit(w[2], w[3]));
            const double mu = log(mean) - 0.5 * sigma * sigma;
            L = (int64_t)rint(exp(mu + sigma * z));
        }
        len[j] = L < 1 ? 1 : L;
    }
}

__device__ __forceinline__ int upper_bound(const double *a, int n, double x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// tokens: one warp per document: theta (T gammas) into a shared CDF, then
// the document's tokens as keys doc * n + feature
constexpr int TOK_WARPS = 4;
__global__ void __launch_bounds__(TOK_WARPS * 32)
    tokens_kernel(Rng rng, int64_t m, int64_t n, int T, const double *phi_cdf, const int64_t *offsets,
                  uint64_t *keys) {
    extern __shared__ double th_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *th = th_all + (size_t)warp * T;
    for (int64_t j = (int64_t)blockIdx.x * TOK_WARPS + warp; j < m; j += (int64_t)gridDim.x * TOK_WARPS) {
        double mx = -1e300;
        for (int t = lane; t < T; t += 32) {
            th[t] = log_gamma_sample(rng, (uint32_t)j, (uint32_t)t, P_THETA, 0.1);
            mx = fmax(mx, th[t]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, o));
        __syncwarp();
        if (lane == 0) {  // inclusive CDF, serial (T <= a few hundred)
            double c = 0.0;
            for (int t = 0; t < T; ++t) {
                c += exp(th[t] - mx);
                th[t] = c;
            }
            for (int t = 0; t < T; ++t) th[t] /= c;
            th[T - 1] = 1.0;
        }
        __syncwarp();
        const int64_t lo = offsets[j], L = offsets[j + 1] - lo;
        for (int64_t s = lane; s < L; s += 32) {
            uint32_t w[4];
            rng.block((uint32_t)j, (uint32_t)s, P_TOKEN, (uint32_t)(j >> 32), w);
            const int t = min(upper_bound(th, T, unit(w[0], w[1])), T - 1);
            const int64_t f = min((int64_t)upper_bound(phi_cdf + (int64_t)t * n, (int)n, unit(w[2], w[3])), n - 1);
            keys[lo + s] = (uint64_t)j * (uint64_t)n + (uint64_t)f;
        }
        __syncwarp();
    }
}

template <typename V>
__global__ void decode_kernel(const uint64_t *ukeys, const int32_t *counts, int64_t nnz, int64_t n, int32_t *rows,
                              V *vals, int64_t *col_of) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
        rows[q] = (int32_t)(ukeys[q] % (uint64_t)n);
        col_of[q] = (int64_t)(ukeys[q] / (uint64_t)n);
        vals[q] = (V)counts[q];
    }
}

__global__ void col_ptr_kernel(const int64_t *col_of, int64_t nnz, int64_t m, int64_t *col_ptr) {
    // col_ptr[c] = first q with col_of[q] >= c (col_of ascending)
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= m; c += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (col_of[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        col_ptr[c] = lo;
    }
}

int bits_for(uint64_t v) {
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

}  // namespace
}  // namespace klnmf

using namespace klnmf;

// Phase 1: phi CDFs, document lengths and token offsets; reports the token count.
// Phase 2 (klnmf_synth_build): tokens, sort, counts -> CSC.
extern "C" int klnmf_synth_build(uint64_t seed, int64_t n, int64_t m, int32_t topics, double zipf, int length_kind,
                                 double length_mean, double length_sigma, int fp32, int64_t *nnz_out,
                                 int64_t *col_ptr, int32_t **row_idx_out, void **values_out, void *stream) {
    // Allocates row_idx (int32[nnz]) and values (float/double[nnz]) with
    // cudaMallocAsync on `stream`; the caller frees them (klnmf_synth_free).
    cudaStream_t st = as_stream(stream);
    if (n < 1 || m < 1 || topics < 1) return set_error_msg(1, "klnmf_synth_build: bad shape");
    if ((double)n * (double)m >= 1.8e19) return set_error_msg(1, "klnmf_synth_build: n * m overflows the keys");
    Rng rng{seed};
    double zipf_norm = 0.0;
    if (zipf > 0.0)
        for (int64_t i = 1; i <= n; ++i) zipf_norm += pow((double)i, -zipf);
    double *phi = nullptr;
    int64_t *len = nullptr, *off = nullptr;
    KLNMF_CHECK(keep_async_pool());
    KLNMF_CHECK(cudaMallocAsync(&phi, sizeof(double) * (size_t)topics * (size_t)n, st));
    KLNMF_CHECK(cudaMallocAsync(&len, sizeof(int64_t) * (size_t)m, st));
    KLNMF_CHECK(cudaMallocAsync(&off, sizeof(int64_t) * (size_t)(m + 1), st));
    phi_cdf_kernel<256><<<topics, 256, 0, st>>>(rng, n, zipf, zipf_norm, phi);
    KLNMF_CHECK_LAUNCH("phi_cdf_kernel");
    lengths_kernel<<<148 * 8, 256, 0, st>>>(rng, m, length_kind, length_mean, length_sigma, len);
    KLNMF_CHECK_LAUNCH("lengths_kernel");
    // offsets = exclusive scan of lengths (off[0] = 0, off[m] = tokens)
    KLNMF_CHECK(cudaMemsetAsync(off, 0, sizeof(int64_t), st));
    size_t tb = 0;
    void *tmp = nullptr;
    KLNMF_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tb, len, off + 1, (int)m, st));
    KLNMF_CHECK(cudaMallocAsync(&tmp, tb, st));
    KLNMF_CHECK(cub::DeviceScan::InclusiveSum(tmp, tb, len, off + 1, (int)m, st));
    KLNMF_CHECK(cudaFreeAsync(tmp, st));
    int64_t tokens = 0;
    KLNMF_CHECK(cudaMemcpyAsync(&tokens, off + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));

    uint64_t *keys = nullptr, *keys_alt = nullptr;
    KLNMF_CHECK(cudaMallocAsync(&keys, sizeof(uint64_t) * (size_t)tokens, st));
    KLNMF_CHECK(cudaMallocAsync(&keys_alt, sizeof(uint64_t) * (size_t)tokens, st));
    const size_t tsm = sizeof(double) * (size_t)TOK_WARPS * (size_t)topics;
    if (tsm > 48 * 1024) KLNMF_CHECK(ensure_smem((const void *)tokens_kernel, tsm));
    tokens_kernel<<<148 * 16, TOK_WARPS * 32, tsm, st>>>(rng, m, n, topics, phi, off, keys);
    KLNMF_CHECK_LAUNCH("tokens_kernel");
    KLNMF_CHECK(cudaFreeAsync(phi, st));
    // sort keys (doc-major, feature-minor)
    const int end_bit = bits_for((uint64_t)m * (uint64_t)n);
    cub::DoubleBuffer<uint64_t> db(keys, keys_alt);
    tb = 0;
    KLNMF_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)tokens, 0, end_bit, st));
    KLNMF_CHECK(cudaMallocAsync(&tmp, tb, st));
    KLNMF_CHECK(cub::DeviceRadixSort::SortKeys(tmp, tb, db, (int64_t)tokens, 0, end_bit, st));
    KLNMF_CHECK(cudaFreeAsync(tmp, st));
    uint64_t *sorted = db.Current(), *ukeys = db.Alternate();
    int32_t *counts = nullptr;
    int64_t *d_nnz = nullptr;
    KLNMF_CHECK(cudaMallocAsync(&counts, sizeof(int32_t) * (size_t)tokens, st));
    KLNMF_CHECK(cudaMallocAsync(&d_nnz, sizeof(int64_t), st));
    tb = 0;
    KLNMF_CHECK(cub::DeviceRunLengthEncode::Encode(nullptr, tb, sorted, ukeys, counts, d_nnz, (int64_t)tokens, st));
    KLNMF_CHECK(cudaMallocAsync(&tmp, tb, st));
    KLNMF_CHECK(cub::DeviceRunLengthEncode::Encode(tmp, tb, sorted, ukeys, counts, d_nnz, (int64_t)tokens, st));
    KLNMF_CHECK(cudaFreeAsync(tmp, st));
    int64_t nnz = 0;
    KLNMF_CHECK(cudaMemcpyAsync(&nnz, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    if (nnz >= INT32_MAX) return set_error_msg(1, "klnmf_synth_build: nnz must be < 2^31");
    int32_t *rows = nullptr;
    void *vals = nullptr;
    int64_t *col_of = reinterpret_cast<int64_t *>(sorted);  // sorted keys are no longer needed
    KLNMF_CHECK(cudaMallocAsync(&rows, sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1), st));
    KLNMF_CHECK(cudaMallocAsync(&vals, (fp32 ? sizeof(float) : sizeof(double)) * (size_t)(nnz > 0 ? nnz : 1), st));
    if (fp32)
        decode_kernel<float><<<148 * 8, 256, 0, st>>>(ukeys, counts, nnz, n, rows, static_cast<float *>(vals), col_of);
    else
        decode_kernel<double><<<148 * 8, 256, 0, st>>>(ukeys, counts, nnz, n, rows, static_cast<double *>(vals),
                                                       col_of);
    KLNMF_CHECK_LAUNCH("decode_kernel");
    col_ptr_kernel<<<148 * 8, 256, 0, st>>>(col_of, nnz, m, col_ptr);
    KLNMF_CHECK_LAUNCH("col_ptr_kernel");
    KLNMF_CHECK(cudaFreeAsync(keys, st));
    KLNMF_CHECK(cudaFreeAsync(keys_alt, st));
    KLNMF_CHECK(cudaFreeAsync(counts, st));
    KLNMF_CHECK(cudaFreeAsync(d_nnz, st));
    KLNMF_CHECK(cudaFreeAsync(len, st));
    KLNMF_CHECK(cudaFreeAsync(off, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    *nnz_out = nnz;
    *row_idx_out = rows;
    *values_out = vals;
    return 0;
}

// Moves klnmf_synth_build's arrays into caller-owned buffers and frees them.
extern "C" int klnmf_synth_fetch(int32_t *rows, void *vals, int64_t nnz, int fp32, int32_t *rows_dst,
                                 void *vals_dst, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (nnz > 0) {
        KLNMF_CHECK(cudaMemcpyAsync(rows_dst, rows, sizeof(int32_t) * (size_t)nnz, cudaMemcpyDeviceToDevice, st));
        KLNMF_CHECK(cudaMemcpyAsync(vals_dst, vals, (fp32 ? sizeof(float) : sizeof(double)) * (size_t)nnz,
                                    cudaMemcpyDeviceToDevice, st));
    }
    KLNMF_CHECK(cudaFreeAsync(rows, st));
    KLNMF_CHECK(cudaFreeAsync(vals, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    return 0;
}
