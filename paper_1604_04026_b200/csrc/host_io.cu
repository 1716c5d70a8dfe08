// Host <-> device transfers of the plan's bulk arrays (native I/O path).
//
// V arrives from the reference API as int64 row indices and fp64 values
// (sparse.py:71-73) while the device keeps int32 / fp32 (fp32 mode).  The
// narrowing (and, on the way back, the widening of fp32 factors to the fp64
// arrays the API returns) runs on host threads straight into / out of two
// reusable pinned staging buffers, overlapped with the copies of the other
// buffer -- instead of a pageable copy of the wide arrays followed by a
// device-side cast.
#include <algorithm>
#include <mutex>
#include <atomic>
#include <thread>
#include <vector>

#include "common.cuh"

namespace klnmf {
namespace {

constexpr size_t STAGE_BYTES = 32u << 20;  // per staging buffer

struct Staging {
    void *buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int device = -1;
};
Staging g_stage;
std::mutex g_stage_mu;

cudaError_t staging(Staging *&out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (g_stage.device != dev) {
        for (int i = 0; i < 2; ++i) {
            if (g_stage.buf[i]) cudaFreeHost(g_stage.buf[i]);
            if (g_stage.done[i]) cudaEventDestroy(g_stage.done[i]);
            g_stage.buf[i] = nullptr;
            g_stage.done[i] = nullptr;
        }
        for (int i = 0; i < 2; ++i) {
            if ((e = cudaHostAlloc(&g_stage.buf[i], STAGE_BYTES, cudaHostAllocDefault)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&g_stage.done[i], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        g_stage.device = dev;
    }
    out = &g_stage;
    return cudaSuccess;
}

int n_threads() {
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(16u, hc ? hc : 1u));
}

// f(lo, hi) over [0, n) split across threads
template <typename F>
void parallel_for(int64_t n, F &&f) {
    const int nt = (int)std::min<int64_t>(n_threads(), std::max<int64_t>(1, n / (1 << 16)));
    if (nt <= 1) {
        f((int64_t)0, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t per = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        const int64_t lo = std::min(n, t * per), hi = std::min(n, lo + per);
        th.emplace_back([&f, lo, hi] { f(lo, hi); });
    }
    for (auto &x : th) x.join();
}

}  // namespace
}  // namespace klnmf

using namespace klnmf;

// dst_dev[i] = (Dst)src_host[i] for i < n, through pinned staging.
template <typename Src, typename Dst>
static int upload_narrow(const Src *src, int64_t n, Dst *dst_dev, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g_stage_mu);
    Staging *S = nullptr;
    KLNMF_CHECK(staging(S));
    const int64_t per_chunk = (int64_t)(STAGE_BYTES / sizeof(Dst));
    int b = 0;
    for (int64_t off = 0; off < n; off += per_chunk, b ^= 1) {
        const int64_t cnt = std::min(per_chunk, n - off);
        KLNMF_CHECK(cudaEventSynchronize(S->done[b]));  // the copy that last used this buffer is done
        Dst *stage = static_cast<Dst *>(S->buf[b]);
        parallel_for(cnt, [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; ++i) stage[i] = (Dst)src[off + i];
        });
        KLNMF_CHECK(cudaMemcpyAsync(dst_dev + off, stage, sizeof(Dst) * (size_t)cnt, cudaMemcpyHostToDevice, st));
        KLNMF_CHECK(cudaEventRecord(S->done[b], st));
    }
    KLNMF_CHECK(cudaEventSynchronize(S->done[0]));
    KLNMF_CHECK(cudaEventSynchronize(S->done[1]));
    return 0;
}

// min and max of a host array on the host threads (the fp32 mode's range
// check of V before anything is uploaded; numpy's single-threaded min()/max()
// took 50 ms of a C4 plan build).  NaN compares false and is skipped.
extern "C" int klnmf_host_minmax_f64(const double *src_host, int64_t n, double *lo_out, double *hi_out) {
    if (n <= 0) return set_error_msg(1, "klnmf_host_minmax_f64: empty array");
    const int nt = n_threads();
    std::vector<double> lo((size_t)nt + 1, src_host[0]), hi((size_t)nt + 1, src_host[0]);
    std::atomic<int> slot{0};
    parallel_for(n, [&](int64_t a, int64_t b) {
        double l = src_host[a], h = src_host[a];
        for (int64_t i = a; i < b; ++i) {
            const double v = src_host[i];
            l = v < l ? v : l;
            h = v > h ? v : h;
        }
        const int k = slot.fetch_add(1);
        lo[(size_t)k] = l;
        hi[(size_t)k] = h;
    });
    double l = lo[0], h = hi[0];
    for (int k = 0; k < slot.load(); ++k) {
        l = lo[(size_t)k] < l ? lo[(size_t)k] : l;
        h = hi[(size_t)k] > h ? hi[(size_t)k] : h;
    }
    *lo_out = l;
    *hi_out = h;
    return 0;
}

extern "C" int klnmf_upload_i64_as_i32(const int64_t *src_host, int64_t n, int32_t *dst_dev, void *stream) {
    return upload_narrow<int64_t, int32_t>(src_host, n, dst_dev, as_stream(stream));
}

extern "C" int klnmf_upload_f64_as_f32(const double *src_host, int64_t n, float *dst_dev, void *stream) {
    return upload_narrow<double, float>(src_host, n, dst_dev, as_stream(stream));
}

extern "C" int klnmf_upload_f64(const double *src_host, int64_t n, double *dst_dev, void *stream) {
    return upload_narrow<double, double>(src_host, n, dst_dev, as_stream(stream));
}

// dst_host[i] = (double)src_dev[i], through pinned staging: the copy of
// chunk c+1 overlaps the widening of chunk c.
template <typename Src>
static int download_widen(const Src *src_dev, int64_t n, double *dst, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g_stage_mu);
    Staging *S = nullptr;
    KLNMF_CHECK(staging(S));
    const int64_t per_chunk = (int64_t)(STAGE_BYTES / sizeof(Src));
    const int64_t n_chunks = (n + per_chunk - 1) / per_chunk;
    auto enqueue = [&](int64_t c) -> int {
        const int64_t off = c * per_chunk, cnt = std::min(per_chunk, n - off);
        KLNMF_CHECK(cudaMemcpyAsync(S->buf[c & 1], src_dev + off, sizeof(Src) * (size_t)cnt, cudaMemcpyDeviceToHost,
                                    st));
        KLNMF_CHECK(cudaEventRecord(S->done[c & 1], st));
        return 0;
    };
    if (n_chunks > 0 && enqueue(0)) return 1;
    for (int64_t c = 0; c < n_chunks; ++c) {
        KLNMF_CHECK(cudaEventSynchronize(S->done[c & 1]));
        if (c + 1 < n_chunks && enqueue(c + 1)) return 1;
        const int64_t off = c * per_chunk, cnt = std::min(per_chunk, n - off);
        const Src *stage = static_cast<const Src *>(S->buf[c & 1]);
        parallel_for(cnt, [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; ++i) dst[off + i] = (double)stage[i];
        });
    }
    return 0;
}

extern "C" int klnmf_download_f32_as_f64(const float *src_dev, int64_t n, double *dst_host, void *stream) {
    return download_widen<float>(src_dev, n, dst_host, as_stream(stream));
}

extern "C" int klnmf_download_f64(const double *src_dev, int64_t n, double *dst_host, void *stream) {
    return download_widen<double>(src_dev, n, dst_host, as_stream(stream));
}
