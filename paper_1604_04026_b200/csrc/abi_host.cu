// C-ABI plumbing and the host-pointer drop-in entry points.
//
// klnmf_sweep_range / klnmf_kl_data_term / klnmf_row_sums take the exact
// arguments of the reference's native functions (_kernels.py:123-160,
// sparse.py:194-196) as host arrays in the reference layout, stage them on the
// device, run the fp64 exact-mode kernels and copy the results back.  They are
// what a maintainer binds with ctypes in place of the numba kernels
// (INTEGRATION.md).  Every call is self-contained (own stream, own buffers).
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace klnmf {

static thread_local char g_err[512] = "";

int set_error(cudaError_t err, const char *where) {
    snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorString(err), cudaGetErrorName(err));
    (void)cudaGetLastError();  // a failed API call must not surface again at the next launch check
    return (int)err;
}

int set_error_msg(int code, const char *msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

cudaError_t ensure_smem(const void *fn, size_t bytes) {
    struct Entry {
        const void *fn;
        size_t bytes;
    };
    static Entry cache[256];
    static int n = 0;
    static std::mutex mu;  // host drop-ins run concurrently on the reference's worker threads
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const void *key = static_cast<const char *>(fn) + dev;  // attributes are per device
    for (int i = 0; i < n; ++i)
        if (cache[i].fn == key) {
            if (cache[i].bytes >= bytes) return cudaSuccess;
            const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
            if (e == cudaSuccess) cache[i].bytes = bytes;
            return e;
        }
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess && n < 256) cache[n++] = Entry{key, bytes};
    return e;
}

int row_sums_ref_layout(const double *fac_dev, int64_t r, int64_t n, double *out_dev, cudaStream_t st);

namespace {

__global__ void i64_to_i32(const int64_t *src, int64_t n, int32_t *dst) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        dst[q] = (int32_t)src[q];
}

__global__ void iota_from(int32_t *dst, int64_t n, int64_t start) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        dst[q] = (int32_t)(start + q);
}

inline unsigned grid_for(int64_t total) {
    int64_t b = (total + 255) / 256;
    if (b < 1) b = 1;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)b;
}

// RAII bundle of device allocations for one host call.
struct DevBufs {
    std::vector<void *> ptrs;
    cudaStream_t st = nullptr;
    ~DevBufs() {
        for (void *p : ptrs) cudaFree(p);
        if (st) cudaStreamDestroy(st);
    }
    template <typename T>
    cudaError_t alloc(T **p, size_t count) {
        void *q = nullptr;
        cudaError_t e = cudaMalloc(&q, count * sizeof(T) + 16);
        if (e == cudaSuccess) ptrs.push_back(q);
        *p = static_cast<T *>(q);
        return e;
    }
};

inline int32_t round_rp(int64_t r) { return (int32_t)((r + 3) / 4 * 4); }

// Columns j_lo..j_hi-1 of an (r, n) C-order fp64 array: one strided copy
// (r rows of (j_hi-j_lo) values, pitch n).  The device buffer is full-size;
// its other columns are zeroed on upload so the layout transform reads no
// uninitialised memory.
cudaError_t copy_columns(double *dst, const double *src, int64_t r, int64_t n, int64_t j_lo, int64_t j_hi,
                         cudaMemcpyKind kind, cudaStream_t st) {
    if (r <= 0 || j_hi <= j_lo) return cudaSuccess;
    if (kind == cudaMemcpyHostToDevice && j_hi - j_lo < n) {
        const cudaError_t e = cudaMemsetAsync(dst, 0, sizeof(double) * (size_t)r * (size_t)n, st);
        if (e != cudaSuccess) return e;
    }
    const size_t pitch = sizeof(double) * (size_t)n;
    return cudaMemcpy2DAsync(dst + j_lo, pitch, src + j_lo, pitch, sizeof(double) * (size_t)(j_hi - j_lo),
                             (size_t)r, kind, st);
}

}  // namespace
}  // namespace klnmf

using namespace klnmf;

extern "C" int klnmf_abi_version(void) { return KLNMF_ABI_VERSION; }
extern "C" int klnmf_sizeof_solve_args(void) { return (int)sizeof(klnmf_solve_args_t); }
extern "C" int klnmf_sizeof_side(void) { return (int)sizeof(klnmf_side_t); }

extern "C" const char *klnmf_last_error(void) { return g_err; }

extern "C" int klnmf_chunk_order(uint64_t seed, uint32_t iter, uint32_t item, uint32_t side, int32_t nchunks,
                                 uint8_t *order) {
    if (nchunks < 0 || nchunks > klnmf::MAX_CHUNKS) return set_error_msg(1, "klnmf_chunk_order: 0 <= nchunks <= 64");
    klnmf::chunk_order(seed, iter, item, side, nchunks, order);
    return 0;
}

extern "C" int klnmf_chunk_perm4(uint64_t seed, uint32_t iter, uint32_t item, uint32_t side, int32_t pos,
                                 uint8_t *perm) {
    if (pos < 0 || pos >= klnmf::MAX_CHUNKS) return set_error_msg(1, "klnmf_chunk_perm4: 0 <= pos < 64");
    const uint32_t p = klnmf::chunk_perm4(seed, iter, item, side, pos);
    for (int c = 0; c < 4; ++c) perm[c] = (uint8_t)((p >> (2 * c)) & 3u);
    return 0;
}

extern "C" int klnmf_event_create(void **event) {
    cudaEvent_t ev;
    KLNMF_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    *event = ev;
    return 0;
}

extern "C" int klnmf_event_destroy(void *event) {
    if (event) KLNMF_CHECK(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
    return 0;
}

// --- CUDA IPC (fused sharded exchange) ---
// The allocation base of a device pointer comes from the driver's
// cuMemGetAddressRange, reached through the runtime's entry-point query so the
// library needs no link-time libcuda.
typedef int (*GetAddressRangeFn)(unsigned long long *base, size_t *size, unsigned long long ptr);

extern "C" int klnmf_ipc_export(const void *ptr, void *handle, int64_t *offset) {
    static GetAddressRangeFn range = nullptr;
    if (!range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        KLNMF_CHECK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn)
            return set_error_msg(1, "klnmf_ipc_export: cuMemGetAddressRange is not available");
        range = reinterpret_cast<GetAddressRangeFn>(fn);
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0)
        return set_error_msg(1, "klnmf_ipc_export: not a device allocation");
    cudaIpcMemHandle_t h;
    KLNMF_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
    memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((unsigned long long)(uintptr_t)ptr - base);
    return 0;
}

extern "C" int klnmf_ipc_open(const void *handle, void **base) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    KLNMF_CHECK(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
    return 0;
}

extern "C" int klnmf_ipc_close(void *base) {
    if (base) KLNMF_CHECK(cudaIpcCloseMemHandle(base));
    return 0;
}

extern "C" int klnmf_stream_wait(void *stream, void *event) {
    KLNMF_CHECK(cudaStreamWaitEvent(as_stream(stream), static_cast<cudaEvent_t>(event), 0));
    return 0;
}

extern "C" int klnmf_event_record(void *event, void *stream, int external) {
    cudaEvent_t ev = static_cast<cudaEvent_t>(event);
    if (external)
        KLNMF_CHECK(cudaEventRecordWithFlags(ev, as_stream(stream), cudaEventRecordExternal));
    else
        KLNMF_CHECK(cudaEventRecord(ev, as_stream(stream)));
    return 0;
}

// Shared body of the exact host drop-ins: stage the oriented CSC, the fixed
// factor and the moving columns in the device layout (visit order `ids`),
// then either solve (max_passes passes) or, with kkt_out, evaluate the KKT
// violations at the given moving columns; results return in the reference
// layout.
static int exact_host_call(const int64_t *col_ptr, const int64_t *row_idx, const double *values, const double *at,
                           const double *sum_a, double *moving, int64_t j_lo, int64_t j_hi, const int64_t *ids,
                           double alpha, double beta, double eps_grad, double eps_x, double eps_div,
                           int64_t inner_cap, int64_t max_passes, int64_t r, int64_t n_fix, int64_t n_mov,
                           int64_t *stats, double *kkt_out, const char *who) {
    if (r < 1 || n_fix < 0 || n_mov < 0 || j_lo < 0 || j_hi > n_mov || max_passes < 1)
        return set_error_msg(1, (std::string(who) + ": bad shape, column range or pass count").c_str());
    if (j_hi <= j_lo) return 0;
    // ids must be a permutation of 0..r-1 (solver.py:287 draws rng.permutation(r))
    std::vector<int32_t> order(r), nat(r, -1);
    for (int64_t t = 0; t < r; ++t) {
        const int64_t k = ids ? ids[t] : t;
        if (k < 0 || k >= r || nat[k] >= 0)
            return set_error_msg(1, (std::string(who) + ": ids must be a permutation").c_str());
        order[t] = (int32_t)k;
        nat[k] = (int32_t)t;
    }
    const int64_t nnz = col_ptr[n_mov];
    if (nnz >= INT32_MAX) return set_error_msg(1, "klnmf_sweep_range: nnz must be < 2^31");
    const int32_t rp = round_rp(r);
    std::vector<double> sum_pos(rp, 0.0);
    std::vector<int32_t> ident(rp);
    for (int64_t t = 0; t < r; ++t) sum_pos[t] = sum_a[order[t]];
    for (int t = 0; t < rp; ++t) ident[t] = t;

    DevBufs B;
    KLNMF_CHECK(cudaStreamCreateWithFlags(&B.st, cudaStreamNonBlocking));
    cudaStream_t st = B.st;
    int64_t *d_ptr, *d_row64;
    int32_t *d_idx, *d_order, *d_nat, *d_ident, *d_items;
    double *d_val, *d_at, *d_mov_ref, *d_fixed, *d_moving, *d_sum, *d_scratch;
    unsigned long long *d_stats;
    KLNMF_CHECK(B.alloc(&d_ptr, n_mov + 1));
    KLNMF_CHECK(B.alloc(&d_row64, nnz));
    KLNMF_CHECK(B.alloc(&d_idx, nnz));
    KLNMF_CHECK(B.alloc(&d_val, nnz));
    KLNMF_CHECK(B.alloc(&d_at, r * n_fix));
    KLNMF_CHECK(B.alloc(&d_mov_ref, r * n_mov));
    KLNMF_CHECK(B.alloc(&d_fixed, (int64_t)rp * n_fix));
    KLNMF_CHECK(B.alloc(&d_moving, (int64_t)rp * n_mov));
    KLNMF_CHECK(B.alloc(&d_sum, rp));
    KLNMF_CHECK(B.alloc(&d_scratch, nnz));
    KLNMF_CHECK(B.alloc(&d_order, rp));
    KLNMF_CHECK(B.alloc(&d_nat, rp));
    KLNMF_CHECK(B.alloc(&d_ident, rp));
    KLNMF_CHECK(B.alloc(&d_items, j_hi - j_lo));
    KLNMF_CHECK(B.alloc(&d_stats, KLNMF_STATS_LEN));

    KLNMF_CHECK(cudaMemcpyAsync(d_ptr, col_ptr, sizeof(int64_t) * (n_mov + 1), cudaMemcpyHostToDevice, st));
    if (nnz > 0) {
        KLNMF_CHECK(cudaMemcpyAsync(d_row64, row_idx, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
        KLNMF_CHECK(cudaMemcpyAsync(d_val, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
        i64_to_i32<<<grid_for(nnz), 256, 0, st>>>(d_row64, nnz, d_idx);
        KLNMF_CHECK_LAUNCH("i64_to_i32");
    }
    if (r * n_fix > 0)
        KLNMF_CHECK(cudaMemcpyAsync(d_at, at, sizeof(double) * r * n_fix, cudaMemcpyHostToDevice, st));
    // Only columns j_lo..j_hi-1 of `moving` belong to this call: the reference
    // runs disjoint column ranges concurrently on worker threads
    // (solver.py:207-214), so the other columns are neither read nor written.
    KLNMF_CHECK(copy_columns(d_mov_ref, moving, r, n_mov, j_lo, j_hi, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(cudaMemcpyAsync(d_order, order.data(), sizeof(int32_t) * r, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(cudaMemcpyAsync(d_nat, nat.data(), sizeof(int32_t) * r, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(cudaMemcpyAsync(d_ident, ident.data(), sizeof(int32_t) * rp, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(cudaMemcpyAsync(d_sum, sum_pos.data(), sizeof(double) * rp, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * KLNMF_STATS_LEN, st));
    iota_from<<<grid_for(j_hi - j_lo), 256, 0, st>>>(d_items, j_hi - j_lo, j_lo);
    KLNMF_CHECK_LAUNCH("iota_from");
    int rc = klnmf_layout_to_device(d_at, r, n_fix, d_order, rp, d_fixed, 0, st);
    if (rc) return rc;
    rc = klnmf_layout_to_device(d_mov_ref, r, n_mov, d_order, rp, d_moving, 0, st);
    if (rc) return rc;

    klnmf_solve_args_t a = {};  // shared coordinate order (the reference ids)
    memset(&a, 0, sizeof(a));
    a.side.ptr = d_ptr;
    a.side.idx = d_idx;
    a.side.val = d_val;
    a.side.n_fix = n_fix;
    a.side.n_mov = n_mov;
    a.side.nnz = nnz;
    a.fixed = d_fixed;
    a.moving = d_moving;
    a.sum_pos = d_sum;
    a.perm_in = d_ident;
    a.perm_out = d_ident;
    a.nat_pos = d_nat;
    a.items = d_items;
    a.n_items = j_hi - j_lo;
    a.scratch = d_scratch;
    a.r = (int32_t)r;
    a.rp = rp;
    a.alpha = alpha;
    a.beta = beta;
    a.eps_grad = eps_grad;
    a.eps_x = eps_x;
    a.eps_div = eps_div;
    a.inner_cap = inner_cap;
    a.stats = d_stats;
    a.max_passes = (int32_t)max_passes;
    if (kkt_out) {
        double *d_kkt;
        KLNMF_CHECK(B.alloc(&d_kkt, (int64_t)rp * n_mov));
        KLNMF_CHECK(cudaMemsetAsync(d_kkt, 0, sizeof(double) * (size_t)rp * (size_t)n_mov, st));
        rc = klnmf_kkt_exact(&a, d_kkt, st);
        if (rc) return rc;
        rc = klnmf_layout_from_device(d_kkt, r, n_mov, d_order, rp, 0, d_mov_ref, st);
        if (rc) return rc;
        if (r * n_mov > 0)
            KLNMF_CHECK(cudaMemcpyAsync(kkt_out, d_mov_ref, sizeof(double) * r * n_mov, cudaMemcpyDeviceToHost, st));
        KLNMF_CHECK(cudaStreamSynchronize(st));
        return 0;
    }
    rc = klnmf_solve_exact(&a, st);
    if (rc) return rc;
    rc = klnmf_layout_from_device(d_moving, r, n_mov, d_order, rp, 0, d_mov_ref, st);
    if (rc) return rc;
    unsigned long long hs[KLNMF_STATS_LEN];
    KLNMF_CHECK(copy_columns(moving, d_mov_ref, r, n_mov, j_lo, j_hi, cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaMemcpyAsync(hs, d_stats, sizeof(hs), cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    for (int q = 0; q < KLNMF_STATS_LEN; ++q) stats[q] += (int64_t)hs[q];
    return 0;
}

extern "C" int klnmf_sweep_range(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                                 const double *at, const double *sum_a, double *moving, int64_t j_lo, int64_t j_hi,
                                 const int64_t *ids, double alpha, double beta, double eps_grad, double eps_x,
                                 double eps_div, int64_t inner_cap, int64_t r, int64_t n_fix, int64_t n_mov,
                                 int64_t *stats) {
    return exact_host_call(col_ptr, row_idx, values, at, sum_a, moving, j_lo, j_hi, ids, alpha, beta, eps_grad,
                           eps_x, eps_div, inner_cap, 1, r, n_fix, n_mov, stats, nullptr, "klnmf_sweep_range");
}

extern "C" int klnmf_sweep_range_passes(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                                        const double *at, const double *sum_a, double *moving, int64_t j_lo,
                                        int64_t j_hi, const int64_t *ids, double alpha, double beta,
                                        double eps_grad, double eps_x, double eps_div, int64_t inner_cap,
                                        int64_t max_passes, int64_t r, int64_t n_fix, int64_t n_mov,
                                        int64_t *stats) {
    return exact_host_call(col_ptr, row_idx, values, at, sum_a, moving, j_lo, j_hi, ids, alpha, beta, eps_grad,
                           eps_x, eps_div, inner_cap, max_passes, r, n_fix, n_mov, stats, nullptr,
                           "klnmf_sweep_range_passes");
}

extern "C" int klnmf_kkt_violation(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                                   const double *at, const double *sum_a, const double *x, double alpha, double beta,
                                   double eps_grad, double eps_x, double eps_div, int64_t r, int64_t n_fix,
                                   int64_t n_mov, double *out) {
    int64_t stats[KLNMF_STATS_LEN] = {0, 0, 0, 0};
    return exact_host_call(col_ptr, row_idx, values, at, sum_a, const_cast<double *>(x), 0, n_mov, nullptr, alpha,
                           beta, eps_grad, eps_x, eps_div, 1, 1, r, n_fix, n_mov, stats, out, "klnmf_kkt_violation");
}

extern "C" int klnmf_mu_update_range(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                                     const double *fixed, double *moving, const double *sum_fixed, double eps_mu,
                                     int64_t j_lo, int64_t j_hi, int64_t r, int64_t n_fix, int64_t n_mov) {
    if (r < 1 || n_fix < 0 || n_mov < 0 || j_lo < 0 || j_hi > n_mov)
        return set_error_msg(1, "klnmf_mu_update_range: bad shape or column range");
    if (j_hi <= j_lo) return 0;
    const int64_t nnz = col_ptr[n_mov];
    if (nnz >= INT32_MAX) return set_error_msg(1, "klnmf_mu_update_range: nnz must be < 2^31");
    const int32_t rp = round_rp(r);
    std::vector<int32_t> ident(rp);
    for (int t = 0; t < rp; ++t) ident[t] = t;
    std::vector<double> sum_pad(rp, 0.0);
    for (int64_t k = 0; k < r; ++k) sum_pad[k] = sum_fixed[k];
    DevBufs B;
    KLNMF_CHECK(cudaStreamCreateWithFlags(&B.st, cudaStreamNonBlocking));
    cudaStream_t st = B.st;
    int64_t *d_ptr, *d_row64;
    int32_t *d_idx, *d_ident, *d_items;
    double *d_val, *d_fix_ref, *d_mov_ref, *d_fixed, *d_moving, *d_sum, *d_ratio;
    KLNMF_CHECK(B.alloc(&d_ptr, n_mov + 1));
    KLNMF_CHECK(B.alloc(&d_row64, nnz));
    KLNMF_CHECK(B.alloc(&d_idx, nnz));
    KLNMF_CHECK(B.alloc(&d_val, nnz));
    KLNMF_CHECK(B.alloc(&d_ratio, nnz));
    KLNMF_CHECK(B.alloc(&d_fix_ref, r * n_fix));
    KLNMF_CHECK(B.alloc(&d_mov_ref, r * n_mov));
    KLNMF_CHECK(B.alloc(&d_fixed, (int64_t)rp * n_fix));
    KLNMF_CHECK(B.alloc(&d_moving, (int64_t)rp * n_mov));
    KLNMF_CHECK(B.alloc(&d_sum, rp));
    KLNMF_CHECK(B.alloc(&d_ident, rp));
    KLNMF_CHECK(B.alloc(&d_items, j_hi - j_lo));
    KLNMF_CHECK(cudaMemcpyAsync(d_ptr, col_ptr, sizeof(int64_t) * (n_mov + 1), cudaMemcpyHostToDevice, st));
    if (nnz > 0) {
        KLNMF_CHECK(cudaMemcpyAsync(d_row64, row_idx, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
        KLNMF_CHECK(cudaMemcpyAsync(d_val, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
        i64_to_i32<<<grid_for(nnz), 256, 0, st>>>(d_row64, nnz, d_idx);
        KLNMF_CHECK_LAUNCH("i64_to_i32");
    }
    if (r * n_fix > 0)
        KLNMF_CHECK(cudaMemcpyAsync(d_fix_ref, fixed, sizeof(double) * r * n_fix, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(copy_columns(d_mov_ref, moving, r, n_mov, j_lo, j_hi, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(cudaMemcpyAsync(d_ident, ident.data(), sizeof(int32_t) * rp, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(cudaMemcpyAsync(d_sum, sum_pad.data(), sizeof(double) * rp, cudaMemcpyHostToDevice, st));
    iota_from<<<grid_for(j_hi - j_lo), 256, 0, st>>>(d_items, j_hi - j_lo, j_lo);
    KLNMF_CHECK_LAUNCH("iota_from");
    int rc = klnmf_layout_to_device(d_fix_ref, r, n_fix, d_ident, rp, d_fixed, 0, st);
    if (rc) return rc;
    rc = klnmf_layout_to_device(d_mov_ref, r, n_mov, d_ident, rp, d_moving, 0, st);
    if (rc) return rc;
    klnmf_side_t side = {d_ptr, d_idx, d_val, n_fix, n_mov, nnz};
    rc = klnmf_mu_update_dev(&side, d_fixed, d_moving, d_sum, (int32_t)r, rp, eps_mu, d_items, j_hi - j_lo, d_ratio,
                             st);
    if (rc) return rc;
    rc = klnmf_layout_from_device(d_moving, r, n_mov, d_ident, rp, 0, d_mov_ref, st);
    if (rc) return rc;
    KLNMF_CHECK(copy_columns(moving, d_mov_ref, r, n_mov, j_lo, j_hi, cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int klnmf_kl_data_term(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                                  const double *w, const double *f, double eps_div, int64_t r, int64_t n_rows,
                                  int64_t n_cols, double *out) {
    if (r < 1 || n_rows < 0 || n_cols < 0) return set_error_msg(1, "klnmf_kl_data_term: bad shape");
    const int64_t nnz = col_ptr[n_cols];
    if (nnz >= INT32_MAX) return set_error_msg(1, "klnmf_kl_data_term: nnz must be < 2^31");
    const int32_t rp = round_rp(r);
    std::vector<int32_t> ident(rp);
    for (int t = 0; t < rp; ++t) ident[t] = t;
    DevBufs B;
    KLNMF_CHECK(cudaStreamCreateWithFlags(&B.st, cudaStreamNonBlocking));
    cudaStream_t st = B.st;
    int64_t *d_ptr, *d_row64;
    int32_t *d_idx, *d_ident;
    double *d_val, *d_w, *d_f, *d_wl, *d_fl;
    KLNMF_CHECK(B.alloc(&d_ptr, n_cols + 1));
    KLNMF_CHECK(B.alloc(&d_row64, nnz));
    KLNMF_CHECK(B.alloc(&d_idx, nnz));
    KLNMF_CHECK(B.alloc(&d_val, nnz));
    KLNMF_CHECK(B.alloc(&d_w, r * n_rows));
    KLNMF_CHECK(B.alloc(&d_f, r * n_cols));
    KLNMF_CHECK(B.alloc(&d_wl, (int64_t)rp * n_rows));
    KLNMF_CHECK(B.alloc(&d_fl, (int64_t)rp * n_cols));
    KLNMF_CHECK(B.alloc(&d_ident, rp));
    KLNMF_CHECK(cudaMemcpyAsync(d_ptr, col_ptr, sizeof(int64_t) * (n_cols + 1), cudaMemcpyHostToDevice, st));
    if (nnz > 0) {
        KLNMF_CHECK(cudaMemcpyAsync(d_row64, row_idx, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
        KLNMF_CHECK(cudaMemcpyAsync(d_val, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
        i64_to_i32<<<grid_for(nnz), 256, 0, st>>>(d_row64, nnz, d_idx);
        KLNMF_CHECK_LAUNCH("i64_to_i32");
    }
    if (r * n_rows > 0) KLNMF_CHECK(cudaMemcpyAsync(d_w, w, sizeof(double) * r * n_rows, cudaMemcpyHostToDevice, st));
    if (r * n_cols > 0) KLNMF_CHECK(cudaMemcpyAsync(d_f, f, sizeof(double) * r * n_cols, cudaMemcpyHostToDevice, st));
    KLNMF_CHECK(cudaMemcpyAsync(d_ident, ident.data(), sizeof(int32_t) * rp, cudaMemcpyHostToDevice, st));
    int rc = klnmf_layout_to_device(d_w, r, n_rows, d_ident, rp, d_wl, 0, st);
    if (rc) return rc;
    rc = klnmf_layout_to_device(d_f, r, n_cols, d_ident, rp, d_fl, 0, st);
    if (rc) return rc;
    klnmf_side_t side;
    side.ptr = d_ptr;
    side.idx = d_idx;
    side.val = d_val;
    side.n_fix = n_rows;
    side.n_mov = n_cols;
    side.nnz = nnz;
    return klnmf_kl_data_term_dev(&side, d_wl, d_fl, rp, d_ident, d_ident, (int32_t)r, 0, eps_div, out, st);
}

extern "C" int klnmf_row_sums(const double *factor, int64_t r, int64_t n, double *out) {
    if (r < 0 || n < 0) return set_error_msg(1, "klnmf_row_sums: bad shape");
    if (r == 0) return 0;
    DevBufs B;
    KLNMF_CHECK(cudaStreamCreateWithFlags(&B.st, cudaStreamNonBlocking));
    cudaStream_t st = B.st;
    double *d_fac, *d_out;
    KLNMF_CHECK(B.alloc(&d_fac, r * n));
    KLNMF_CHECK(B.alloc(&d_out, r));
    if (r * n > 0) KLNMF_CHECK(cudaMemcpyAsync(d_fac, factor, sizeof(double) * r * n, cudaMemcpyHostToDevice, st));
    int rc = row_sums_ref_layout(d_fac, r, n, d_out, st);
    if (rc) return rc;
    KLNMF_CHECK(cudaMemcpyAsync(out, d_out, sizeof(double) * r, cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    return 0;
}
