// Factor-side device operations: layout conversion between the reference's
// (r, n) fp64 layout and the device's item-major visit-order layout, the fp32
// mode row sums (deterministic), factor statistics for the objective and
// sparsity log, and the initial maintained products of the fp32 mode.
//
// Reference anchors: DenseFactor (sparse.py:168-206: row_sums :194-196,
// sparsity :198-200), full_objective's regulariser sums (solver.py:229-233).
#include "common.cuh"

namespace klnmf {
namespace {

template <typename T, typename S = double>
__global__ void to_device_kernel(const S *src, int64_t r, int64_t n, const int32_t *order,
                                 int32_t rp, T *dst) {
    // dst[i, tt] = src[order[tt], i]; padding columns = 0
    const int64_t total = n * rp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / rp;
        const int tt = (int)(e - i * rp);
        T x = tt < r ? (T)src[(int64_t)order[tt] * n + i] : (T)0;
        // fp32 storage: subnormals flush to zero (the fp32 kernels widen
        // stored values with integer arithmetic, exact for zero and normals)
        if (sizeof(T) == 4 && x < (T)1.17549435e-38f) x = (T)0;
        dst[e] = x;
    }
}

template <typename T, typename D>
__global__ void from_device_kernel(const T *src, int64_t r, int64_t n, const int32_t *order,
                                   int32_t rp, D *dst) {
    const int64_t total = n * r;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / r;
        const int tt = (int)(e - i * r);
        dst[(int64_t)order[tt] * n + i] = (D)src[i * rp + tt];
    }
}

// fp32 row sums by position: each block sums a contiguous item range in fp64
// (thread = position, items in order), then one pass adds block partials in
// block order.  Fixed grid => deterministic and identical on every rank.
constexpr int RS_BLOCKS = 1024;

__global__ void row_sums_fast_partial(const float *fac, int64_t n_items, int32_t rp, double *partial) {
    const int64_t per = (n_items + RS_BLOCKS - 1) / RS_BLOCKS;
    const int64_t i0 = (int64_t)blockIdx.x * per;
    const int64_t i1 = min(n_items, i0 + per);
    for (int k = threadIdx.x; k < rp; k += blockDim.x) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int64_t i = i0;
        for (; i + 3 < i1; i += 4) {
            s0 += (double)__ldg(fac + i * rp + k);
            s1 += (double)__ldg(fac + (i + 1) * rp + k);
            s2 += (double)__ldg(fac + (i + 2) * rp + k);
            s3 += (double)__ldg(fac + (i + 3) * rp + k);
        }
        for (; i < i1; ++i) s0 += (double)__ldg(fac + i * rp + k);
        partial[(int64_t)blockIdx.x * rp + k] = (s0 + s1) + (s2 + s3);
    }
}

__global__ void row_sums_fast_final(const double *partial, int32_t rp, int32_t r, double *out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= rp) return;
    double s = 0.0;
    if (k < r)
        for (int b = 0; b < RS_BLOCKS; ++b) s += partial[(int64_t)b * rp + k];
    out[k] = s;
}

// sum x^2, sum x, zero count over the r real columns (fixed grid, fixed tree)
template <typename T, int NT>
__global__ void __launch_bounds__(NT) factor_stats_partial(const T *fac, int64_t n_items, int32_t rp,
                                                           int32_t r, double *partial) {
    __shared__ double sh[NT / 32];
    const int64_t total = n_items * rp;
    double s2 = 0.0, s1 = 0.0, zc = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * NT) {
        const int tt = (int)(e % rp);
        if (tt < r) {
            const double x = (double)fac[e];
            s2 += x * x;
            s1 += x;
            zc += (x == 0.0) ? 1.0 : 0.0;
        }
    }
    const double a = block_sum_det<NT>(s2, sh);
    const double b = block_sum_det<NT>(s1, sh);
    const double c = block_sum_det<NT>(zc, sh);
    if (threadIdx.x == 0) {
        partial[blockIdx.x * 3 + 0] = a;
        partial[blockIdx.x * 3 + 1] = b;
        partial[blockIdx.x * 3 + 2] = c;
    }
}

__global__ void factor_stats_final(const double *partial, int nb, double *out) {
    if (threadIdx.x < 3) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += partial[b * 3 + threadIdx.x];
        out[threadIdx.x] = s;
    }
}

// t[q] = sum_k fixed[i_q, pos_f(k)] * moving[j, pos_m(k)] in natural k order (fp64)
template <int NT>
__global__ void __launch_bounds__(NT) init_t_kernel(const int64_t *ptr, const int32_t *idx, int64_t n_mov,
                                                    int64_t nnz, const float *fixed, const float *moving,
                                                    int32_t rp, const int32_t *fpos, const int32_t *mpos,
                                                    int32_t r, double *t) {
    const int64_t q = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (q >= nnz) return;
    int64_t lo = 0, hi = n_mov;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ptr[mid + 1] <= q) lo = mid + 1; else hi = mid;
    }
    const float *a = fixed + (int64_t)idx[q] * rp;
    const float *b = moving + lo * rp;
    double d = 0.0;
    for (int k = 0; k < r; ++k) d = fma((double)__ldg(a + fpos[k]), (double)__ldg(b + mpos[k]), d);
    t[q] = d;
}

inline unsigned grid_for(int64_t total, int nt) {
    int64_t b = (total + nt - 1) / nt;
    if (b < 1) b = 1;
    if (b > 148 * 64) b = 148 * 64;
    return (unsigned)b;
}

}  // namespace
}  // namespace klnmf

using namespace klnmf;

extern "C" int klnmf_layout_to_device(const double *src, int64_t r, int64_t n, const int32_t *order,
                                      int32_t rp, void *dst, int fp32, void *stream) {
    const int64_t total = n * rp;
    if (total == 0) return 0;
    if (fp32)
        to_device_kernel<float><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(src, r, n, order, rp,
                                                                                    static_cast<float *>(dst));
    else
        to_device_kernel<double><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(src, r, n, order, rp,
                                                                                     static_cast<double *>(dst));
    KLNMF_CHECK_LAUNCH("to_device_kernel");
    return 0;
}

// the same from fp32 values already narrowed on the host (fp32 mode: half the
// PCIe bytes; host (float)x and device __double2float_rn round alike)
extern "C" int klnmf_layout_to_device_f32src(const float *src, int64_t r, int64_t n, const int32_t *order,
                                             int32_t rp, float *dst, void *stream) {
    const int64_t total = n * rp;
    if (total == 0) return 0;
    to_device_kernel<float, float><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(src, r, n, order, rp, dst);
    KLNMF_CHECK_LAUNCH("to_device_kernel");
    return 0;
}

extern "C" int klnmf_layout_from_device(const void *src, int64_t r, int64_t n, const int32_t *order,
                                        int32_t rp, int fp32, double *dst, void *stream) {
    const int64_t total = n * r;
    if (total == 0) return 0;
    if (fp32)
        from_device_kernel<float, double><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
            static_cast<const float *>(src), r, n, order, rp, dst);
    else
        from_device_kernel<double, double><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
            static_cast<const double *>(src), r, n, order, rp, dst);
    KLNMF_CHECK_LAUNCH("from_device_kernel");
    return 0;
}

extern "C" int klnmf_layout_from_device_f32(const float *src, int64_t r, int64_t n, const int32_t *order,
                                            int32_t rp, float *dst, void *stream) {
    const int64_t total = n * r;
    if (total == 0) return 0;
    from_device_kernel<float, float><<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(src, r, n, order, rp, dst);
    KLNMF_CHECK_LAUNCH("from_device_kernel");
    return 0;
}

// Chunk nonzero masks of a factor's rows (klnmf_solve_args_t.fixed_mask):
// one warp per row, lane c tests the 16-byte chunk c.
__global__ void chunk_masks_kernel(const float *fac, int64_t n_items, int32_t rp, int32_t r, uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (row >= n_items) return;
    bool nz = false;
    if (4 * lane < r) {
        const float4 v = *reinterpret_cast<const float4 *>(fac + row * rp + 4 * lane);
        nz = v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f;
    }
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) out[row] = r > 128 ? 0xffffffffu : m;
}

extern "C" int klnmf_chunk_masks(const float *fixed, int64_t n_fix, int32_t rp, int32_t r, uint32_t *out,
                                 void *stream) {
    if (n_fix <= 0) return 0;
    if (rp % 4 != 0) return set_error_msg(1, "klnmf_chunk_masks: rp must be a multiple of 4");
    const int wpb = 8;
    chunk_masks_kernel<<<(unsigned)((n_fix + wpb - 1) / wpb), 32 * wpb, 0, as_stream(stream)>>>(fixed, n_fix, rp, r, out);
    KLNMF_CHECK_LAUNCH("klnmf_chunk_masks");
    return 0;
}

extern "C" int klnmf_row_sums_fast(const float *fac, int64_t n_items, int32_t rp, int32_t r,
                                   double *out, void *stream) {
    cudaStream_t st = as_stream(stream);
    double *partial = nullptr;
    KLNMF_CHECK(keep_async_pool());
    KLNMF_CHECK(cudaMallocAsync(&partial, sizeof(double) * (size_t)RS_BLOCKS * (size_t)rp, st));
    const int nt = rp < 128 ? ((rp + 31) / 32) * 32 : 128;
    row_sums_fast_partial<<<RS_BLOCKS, nt, 0, st>>>(fac, n_items, rp, partial);
    KLNMF_CHECK_LAUNCH("row_sums_fast_partial");
    row_sums_fast_final<<<(rp + 127) / 128, 128, 0, st>>>(partial, rp, r, out);
    KLNMF_CHECK_LAUNCH("row_sums_fast_final");
    KLNMF_CHECK(cudaFreeAsync(partial, st));
    return 0;
}

extern "C" int klnmf_factor_stats(const void *fac, int64_t n_items, int32_t rp, int32_t r, int fp32,
                                  double *out_host, void *stream) {
    cudaStream_t st = as_stream(stream);
    constexpr int NT = 256, NB = 512;
    double *partial = nullptr;
    KLNMF_CHECK(keep_async_pool());
    KLNMF_CHECK(cudaMallocAsync(&partial, sizeof(double) * (NB * 3 + 3), st));
    if (fp32)
        factor_stats_partial<float, NT><<<NB, NT, 0, st>>>(static_cast<const float *>(fac), n_items, rp, r, partial);
    else
        factor_stats_partial<double, NT><<<NB, NT, 0, st>>>(static_cast<const double *>(fac), n_items, rp, r, partial);
    KLNMF_CHECK_LAUNCH("factor_stats_partial");
    factor_stats_final<<<1, 32, 0, st>>>(partial, NB, partial + NB * 3);
    KLNMF_CHECK_LAUNCH("factor_stats_final");
    KLNMF_CHECK(cudaMemcpyAsync(out_host, partial + NB * 3, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaFreeAsync(partial, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    return 0;
}

// KL data term from the maintained products (fp32 mode): fixed grid, each
// block sums a fixed contiguous range in a fixed tree, then one warp sums the
// block partials in order -- deterministic for a given nnz.
constexpr int KL_BLOCKS = 1184, KL_NT = 256;  // 8 x 148 SMs
// tmap (may be NULL): t of entry q is t[tmap[q]] -- the products stored in
// the other orientation, summed in val's (canonical) entry order
__global__ void kl_t_partial(const float *val, const double *t, const int32_t *tmap, int64_t nnz, double eps,
                             double *partial) {
    __shared__ double sh[KL_NT / 32];
    const int64_t per = (nnz + KL_BLOCKS - 1) / KL_BLOCKS;
    const int64_t lo = (int64_t)blockIdx.x * per, hi = min(nnz, lo + per);
    double s = 0.0;
    for (int64_t q = lo + threadIdx.x; q < hi; q += KL_NT) {
        const double v = (double)val[q];
        const double tq = tmap ? t[tmap[q]] : t[q];
        s += v * log(v / (tq + eps)) - v;  // _kernels.py:158
    }
    const double b = block_sum_det<KL_NT>(s, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = b;
}
__global__ void kl_t_final(const double *partial, double *out) {
    double s = 0.0;
    for (int b = threadIdx.x; b < KL_BLOCKS; b += 32) s += partial[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL_MASK, s, o);
    if (threadIdx.x == 0) *out = s;
}

extern "C" int klnmf_kl_data_term_t(const float *val, const double *t, int64_t nnz, double eps_div,
                                    double *out_host, void *stream) {
    return klnmf_kl_data_term_t_mapped(val, t, nullptr, nnz, eps_div, out_host, stream);
}

extern "C" int klnmf_kl_data_term_t_mapped(const float *val, const double *t, const int32_t *tmap, int64_t nnz,
                                           double eps_div, double *out_host, void *stream) {
    cudaStream_t st = as_stream(stream);
    double *partial = nullptr;
    KLNMF_CHECK(keep_async_pool());
    KLNMF_CHECK(cudaMallocAsync(&partial, sizeof(double) * (KL_BLOCKS + 1), st));
    kl_t_partial<<<KL_BLOCKS, KL_NT, 0, st>>>(val, t, tmap, nnz, eps_div, partial);
    KLNMF_CHECK_LAUNCH("kl_t_partial");
    kl_t_final<<<1, 32, 0, st>>>(partial, partial + KL_BLOCKS);
    KLNMF_CHECK_LAUNCH("kl_t_final");
    KLNMF_CHECK(cudaMemcpyAsync(out_host, partial + KL_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaFreeAsync(partial, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int klnmf_init_t(const klnmf_side_t *side, const float *fixed, const float *moving, int32_t rp,
                            const int32_t *fixed_pos, const int32_t *moving_pos, int32_t r, double *t,
                            void *stream) {
    constexpr int NT = 256;
    if (side->nnz == 0) return 0;
    const int64_t blocks = (side->nnz + NT - 1) / NT;
    init_t_kernel<NT><<<(unsigned)blocks, NT, 0, as_stream(stream)>>>(side->ptr, side->idx, side->n_mov, side->nnz,
                                                                      fixed, moving, rp, fixed_pos, moving_pos, r, t);
    KLNMF_CHECK_LAUNCH("init_t_kernel");
    return 0;
}
