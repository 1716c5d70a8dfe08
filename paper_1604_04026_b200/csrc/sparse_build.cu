// Device-side sparse structure construction (north-star (a)):
//   * COO -> CSC   (SparseMatrix.from_coo, sparse.py:92-124: lexsort by
//                   (col, row), duplicate detection, col_ptr from counts)
//   * CSC -> CSC of the transpose (= CSR of V) with both entry maps
//                  (SparseMatrix.transpose, sparse.py:146-154: stable argsort
//                   of row indices, so rows ascending then columns ascending)
//   * nnz bucketing of subproblems (largest first) for the solver kernels.
// Sorting is CUB's stable LSD radix sort; everything stays on the device.
#include <cub/cub.cuh>

#include "common.cuh"

namespace klnmf {
namespace {

// expand ptr into the owning segment of every entry
__global__ void expand_segments(const int64_t *ptr, int64_t n_seg, int32_t *seg_of) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_seg;
         j += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t q = ptr[j]; q < ptr[j + 1]; ++q) seg_of[q] = (int32_t)j;
    }
}

__global__ void iota_i32(int32_t *a, int64_t n) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        a[q] = (int32_t)q;
}

template <typename V>
__global__ void gather_transpose(const int32_t *map_t2o, const int32_t *seg_of, const V *val, int64_t nnz,
                                 int32_t *idx_t, V *val_t, int32_t *map_o2t) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t src = map_t2o[q];
        idx_t[q] = seg_of[src];
        val_t[q] = val[src];
        if (map_o2t) map_o2t[src] = (int32_t)q;
    }
}

// ptr[i] = lower_bound(sorted_keys, i) for i in [0, n]
template <typename K>
__global__ void ptr_from_sorted(const K *keys, int64_t nnz, int64_t n, int64_t *ptr) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)keys[mid] < i) lo = mid + 1; else hi = mid;
        }
        ptr[i] = lo;
    }
}

__global__ void make_coo_keys(const int32_t *rows, const int32_t *cols, int64_t nnz, int64_t n_rows,
                              uint64_t *keys) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x)
        keys[q] = (uint64_t)cols[q] * (uint64_t)n_rows + (uint64_t)rows[q];
}

template <typename V>
__global__ void split_coo_keys(const uint64_t *keys, const int32_t *perm, const V *vals_in, int64_t nnz,
                               int64_t n_rows, int32_t *idx, int32_t *col_of, V *val, int32_t *dup_flag) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[q];
        idx[q] = (int32_t)(k % (uint64_t)n_rows);
        col_of[q] = (int32_t)(k / (uint64_t)n_rows);
        val[q] = vals_in[perm[q]];
        if (q > 0 && keys[q - 1] == k) atomicExch(dup_flag, 1);
    }
}

__global__ void segment_sizes(const int64_t *ptr, int64_t j_lo, int64_t n, int64_t *sizes, int32_t *ids) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        sizes[q] = ptr[j_lo + q + 1] - ptr[j_lo + q];
        ids[q] = (int32_t)(j_lo + q);
    }
}

// counts of items (sorted by size descending) per bucket (bounds ascending)
__global__ void bucket_counts(const int64_t *sorted_sizes, int64_t n, const int64_t *bounds, int nb,
                              int64_t *counts) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    // bucket b holds sizes in (bounds[b-1], bounds[b]]; sizes are descending
    for (int b = 0; b < nb; ++b) {
        const int64_t lo_excl = b == 0 ? -1 : bounds[b - 1];
        const int64_t hi_incl = bounds[b];
        // count elements with lo_excl < s <= hi_incl via binary searches on descending data
        int64_t lo = 0, hi = n;  // first index with s <= hi_incl
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sorted_sizes[mid] > hi_incl) lo = mid + 1; else hi = mid;
        }
        const int64_t a = lo;
        lo = 0; hi = n;  // first index with s <= lo_excl
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sorted_sizes[mid] > lo_excl) lo = mid + 1; else hi = mid;
        }
        counts[b] = lo - a;
    }
}

constexpr int KMAX_BUCKETS = 64;  // size buckets of one side (the fp32 kernel ladder)

inline unsigned grid_for(int64_t total, int nt) {
    int64_t b = (total + nt - 1) / nt;
    if (b < 1) b = 1;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)b;
}

inline int bits_for(int64_t n) {
    int b = 1;
    while (b < 63 && ((int64_t)1 << b) <= n) ++b;
    return b;
}

template <typename V>
int transpose_impl(const int64_t *ptr, const int32_t *idx, const V *val, int64_t n_rows, int64_t n_cols,
                   int64_t nnz, int64_t *ptr_t, int32_t *idx_t, V *val_t, int32_t *map_t2o, int32_t *map_o2t,
                   cudaStream_t st) {
    KLNMF_CHECK(keep_async_pool());
    if (nnz == 0) {
        KLNMF_CHECK(cudaMemsetAsync(ptr_t, 0, sizeof(int64_t) * (size_t)(n_rows + 1), st));
        return 0;
    }
    int32_t *seg_of = nullptr, *iota = nullptr, *keys_out = nullptr;
    KLNMF_CHECK(cudaMallocAsync(&seg_of, sizeof(int32_t) * (size_t)nnz, st));
    KLNMF_CHECK(cudaMallocAsync(&iota, sizeof(int32_t) * (size_t)nnz, st));
    KLNMF_CHECK(cudaMallocAsync(&keys_out, sizeof(int32_t) * (size_t)nnz, st));
    expand_segments<<<grid_for(n_cols, 256), 256, 0, st>>>(ptr, n_cols, seg_of);
    iota_i32<<<grid_for(nnz, 256), 256, 0, st>>>(iota, nnz);
    KLNMF_CHECK_LAUNCH("expand_segments");
    size_t tmp_bytes = 0;
    const int end_bit = bits_for(n_rows);
    KLNMF_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, idx, keys_out, iota, map_t2o, (int)nnz, 0,
                                                end_bit, st));
    void *tmp = nullptr;
    KLNMF_CHECK(cudaMallocAsync(&tmp, tmp_bytes, st));
    KLNMF_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, idx, keys_out, iota, map_t2o, (int)nnz, 0,
                                                end_bit, st));
    gather_transpose<V><<<grid_for(nnz, 256), 256, 0, st>>>(map_t2o, seg_of, val, nnz, idx_t, val_t, map_o2t);
    ptr_from_sorted<int32_t><<<grid_for(n_rows + 1, 256), 256, 0, st>>>(keys_out, nnz, n_rows, ptr_t);
    KLNMF_CHECK_LAUNCH("gather_transpose");
    KLNMF_CHECK(cudaFreeAsync(tmp, st));
    KLNMF_CHECK(cudaFreeAsync(seg_of, st));
    KLNMF_CHECK(cudaFreeAsync(iota, st));
    KLNMF_CHECK(cudaFreeAsync(keys_out, st));
    return 0;
}

template <typename V>
int coo_impl(const int32_t *rows, const int32_t *cols, const V *vals, int64_t nnz, int64_t n_rows, int64_t n_cols,
             int64_t *ptr, int32_t *idx, V *val, int32_t *dup_flag, cudaStream_t st) {
    KLNMF_CHECK(keep_async_pool());
    KLNMF_CHECK(cudaMemsetAsync(dup_flag, 0, sizeof(int32_t), st));
    if (nnz == 0) {
        KLNMF_CHECK(cudaMemsetAsync(ptr, 0, sizeof(int64_t) * (size_t)(n_cols + 1), st));
        return 0;
    }
    uint64_t *keys = nullptr, *keys_sorted = nullptr;
    int32_t *iota = nullptr, *perm = nullptr, *col_of = nullptr;
    KLNMF_CHECK(cudaMallocAsync(&keys, sizeof(uint64_t) * (size_t)nnz, st));
    KLNMF_CHECK(cudaMallocAsync(&keys_sorted, sizeof(uint64_t) * (size_t)nnz, st));
    KLNMF_CHECK(cudaMallocAsync(&iota, sizeof(int32_t) * (size_t)nnz, st));
    KLNMF_CHECK(cudaMallocAsync(&perm, sizeof(int32_t) * (size_t)nnz, st));
    KLNMF_CHECK(cudaMallocAsync(&col_of, sizeof(int32_t) * (size_t)nnz, st));
    make_coo_keys<<<grid_for(nnz, 256), 256, 0, st>>>(rows, cols, nnz, n_rows, keys);
    iota_i32<<<grid_for(nnz, 256), 256, 0, st>>>(iota, nnz);
    KLNMF_CHECK_LAUNCH("make_coo_keys");
    const int end_bit = bits_for(n_rows * n_cols);
    size_t tmp_bytes = 0;
    KLNMF_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_sorted, iota, perm, (int)nnz, 0,
                                                end_bit, st));
    void *tmp = nullptr;
    KLNMF_CHECK(cudaMallocAsync(&tmp, tmp_bytes, st));
    KLNMF_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_sorted, iota, perm, (int)nnz, 0,
                                                end_bit, st));
    split_coo_keys<V><<<grid_for(nnz, 256), 256, 0, st>>>(keys_sorted, perm, vals, nnz, n_rows, idx, col_of, val,
                                                          dup_flag);
    ptr_from_sorted<int32_t><<<grid_for(n_cols + 1, 256), 256, 0, st>>>(col_of, nnz, n_cols, ptr);
    KLNMF_CHECK_LAUNCH("split_coo_keys");
    KLNMF_CHECK(cudaFreeAsync(tmp, st));
    KLNMF_CHECK(cudaFreeAsync(keys, st));
    KLNMF_CHECK(cudaFreeAsync(keys_sorted, st));
    KLNMF_CHECK(cudaFreeAsync(iota, st));
    KLNMF_CHECK(cudaFreeAsync(perm, st));
    KLNMF_CHECK(cudaFreeAsync(col_of, st));
    return 0;
}

}  // namespace
}  // namespace klnmf

using namespace klnmf;

extern "C" int klnmf_transpose(const int64_t *ptr, const int32_t *idx, const void *val, int val_bytes,
                               int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t *ptr_t, int32_t *idx_t,
                               void *val_t, int32_t *map_t2o, int32_t *map_o2t, void *stream) {
    if (nnz >= INT32_MAX) return set_error_msg(1, "klnmf_transpose: nnz must be < 2^31");
    cudaStream_t st = as_stream(stream);
    if (val_bytes == 4)
        return transpose_impl<float>(ptr, idx, static_cast<const float *>(val), n_rows, n_cols, nnz, ptr_t, idx_t,
                                     static_cast<float *>(val_t), map_t2o, map_o2t, st);
    if (val_bytes == 8)
        return transpose_impl<double>(ptr, idx, static_cast<const double *>(val), n_rows, n_cols, nnz, ptr_t, idx_t,
                                      static_cast<double *>(val_t), map_t2o, map_o2t, st);
    return set_error_msg(1, "klnmf_transpose: val_bytes must be 4 or 8");
}

extern "C" int klnmf_coo_to_csc(const int32_t *rows, const int32_t *cols, const void *vals, int val_bytes,
                                int64_t nnz, int64_t n_rows, int64_t n_cols, int64_t *ptr, int32_t *idx, void *val,
                                int32_t *dup_flag, void *stream) {
    if (nnz >= INT32_MAX) return set_error_msg(1, "klnmf_coo_to_csc: nnz must be < 2^31");
    cudaStream_t st = as_stream(stream);
    if (val_bytes == 4)
        return coo_impl<float>(rows, cols, static_cast<const float *>(vals), nnz, n_rows, n_cols, ptr, idx,
                               static_cast<float *>(val), dup_flag, st);
    if (val_bytes == 8)
        return coo_impl<double>(rows, cols, static_cast<const double *>(vals), nnz, n_rows, n_cols, ptr, idx,
                                static_cast<double *>(val), dup_flag, st);
    return set_error_msg(1, "klnmf_coo_to_csc: val_bytes must be 4 or 8");
}

extern "C" int klnmf_bucketize(const int64_t *ptr, int64_t j_lo, int64_t j_hi, const int64_t *bounds, int n_bounds,
                               int32_t *items, int64_t *bucket_count_host, void *stream) {
    cudaStream_t st = as_stream(stream);
    const int64_t n = j_hi - j_lo;
    if (n_bounds < 1 || n_bounds > KMAX_BUCKETS)
        return set_error_msg(1, "klnmf_bucketize: 1 <= n_bounds <= 64");
    if (n <= 0) {
        for (int b = 0; b < n_bounds; ++b) bucket_count_host[b] = 0;
        return 0;
    }
    int64_t *sizes = nullptr, *sizes_sorted = nullptr, *dbounds = nullptr, *dcounts = nullptr;
    int32_t *ids = nullptr;
    KLNMF_CHECK(keep_async_pool());
    KLNMF_CHECK(cudaMallocAsync(&sizes, sizeof(int64_t) * (size_t)n, st));
    KLNMF_CHECK(cudaMallocAsync(&sizes_sorted, sizeof(int64_t) * (size_t)n, st));
    KLNMF_CHECK(cudaMallocAsync(&ids, sizeof(int32_t) * (size_t)n, st));
    KLNMF_CHECK(cudaMallocAsync(&dbounds, sizeof(int64_t) * 2 * KMAX_BUCKETS, st));
    dcounts = dbounds + KMAX_BUCKETS;
    KLNMF_CHECK(cudaMemcpyAsync(dbounds, bounds, sizeof(int64_t) * (size_t)n_bounds, cudaMemcpyHostToDevice, st));
    segment_sizes<<<grid_for(n, 256), 256, 0, st>>>(ptr, j_lo, n, sizes, ids);
    KLNMF_CHECK_LAUNCH("segment_sizes");
    size_t tmp_bytes = 0;
    KLNMF_CHECK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, sizes, sizes_sorted, ids, items,
                                                          (int)n, 0, 64, st));
    void *tmp = nullptr;
    KLNMF_CHECK(cudaMallocAsync(&tmp, tmp_bytes, st));
    KLNMF_CHECK(cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, sizes, sizes_sorted, ids, items, (int)n,
                                                          0, 64, st));
    bucket_counts<<<1, 1, 0, st>>>(sizes_sorted, n, dbounds, n_bounds, dcounts);
    KLNMF_CHECK_LAUNCH("bucket_counts");
    KLNMF_CHECK(cudaMemcpyAsync(bucket_count_host, dcounts, sizeof(int64_t) * (size_t)n_bounds,
                                cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaFreeAsync(tmp, st));
    KLNMF_CHECK(cudaFreeAsync(sizes, st));
    KLNMF_CHECK(cudaFreeAsync(sizes_sorted, st));
    KLNMF_CHECK(cudaFreeAsync(ids, st));
    KLNMF_CHECK(cudaFreeAsync(dbounds, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    return 0;
}
