// fp64 exact mode: bit-identical restatement of the reference numba kernels.
//
// Compiled with -fmad=false AND written with explicit __d*_rn intrinsics: the
// reference's numba kernels contain no FMA and no fast-math (SURVEY.md
// finding 3), reductions run strictly in entry order, and division is IEEE.
//
//   solve_exact_kernel   _kernels.sweep_range + solve_column + _grad_hess +
//                        compute_ax (_kernels.py:24-144), max_passes = 1, with
//                        the maintained product kept on the column support
//                        only (bitwise identical, SURVEY.md finding 2)
//   row_sums_pairwise    DenseFactor.row_sums (sparse.py:194-196): numpy
//                        pairwise summation, bit-identical
//   kl_terms_kernel      _kernels.kl_data_term (_kernels.py:147-160), per-entry
//                        terms in the reference's operation order; the final sum
//                        is a fixed-order tree (deterministic, not serial)
//
// Layout: one warp owns one subproblem (a column of the oriented matrix).  The
// per-coordinate gradient reduction is serial in entry order: lanes compute the
// entry terms in parallel, then every lane folds the 32 terms of each chunk in
// order via shuffles, so g/h are identical on all lanes and equal to the
// reference's left-to-right sum.
#include "common.cuh"

namespace klnmf {

namespace {

constexpr int EXACT_WPB = 4;  // warps (subproblems) per block

struct ExactState {
    const int32_t *vi;
    const double *vv;
    double *t;
    int64_t s;
};

// _grad_hess (_kernels.py:24-36), serial over entries in index order.
__device__ __forceinline__ void exact_grad_hess(const klnmf_solve_args_t &a, const double *fixed,
                                                const ExactState &st, int tt, double x,
                                                double *g_out, double *h_out, int lane) {
    // g = sum_a[k] + alpha * x_k + beta ; h = alpha
    double g = __dadd_rn(__dadd_rn(a.sum_pos[tt], __dmul_rn(a.alpha, x)), a.beta);
    double h = a.alpha;
    const int64_t rp = a.rp;
    for (int64_t base = 0; base < st.s; base += 32) {
        const int64_t p = base + lane;
        double tg = 0.0, th = 0.0;
        bool nz = false;
        if (p < st.s) {
            const double av = __ldg(fixed + (int64_t)st.vi[p] * rp + tt);
            if (av != 0.0) {
                const double q = __ddiv_rn(av, __dadd_rn(st.t[p], a.eps_div));
                tg = __dmul_rn(st.vv[p], q);   // v * q
                th = __dmul_rn(tg, q);         // (v * q) * q
                nz = true;
            }
        }
        const unsigned m = __ballot_sync(FULL_MASK, nz);
        const int cnt = (int)min((int64_t)32, st.s - base);
        for (int l = 0; l < cnt; ++l) {
            const double tgl = __shfl_sync(FULL_MASK, tg, l);
            const double thl = __shfl_sync(FULL_MASK, th, l);
            if ((m >> l) & 1u) {
                g = __dsub_rn(g, tgl);
                h = __dadd_rn(h, thl);
            }
        }
    }
    *g_out = g;
    *h_out = h;
}

// ax += delta * at[k]; clamp at 0 (_kernels.py:86-90, :103-106), on the support.
__device__ __forceinline__ void exact_update(const klnmf_solve_args_t &a, const double *fixed,
                                             const ExactState &st, int tt, double delta, int lane) {
    const int64_t rp = a.rp;
    for (int64_t p = lane; p < st.s; p += 32) {
        const double av = __ldg(fixed + (int64_t)st.vi[p] * rp + tt);
        double tn = __dadd_rn(st.t[p], __dmul_rn(delta, av));
        if (tn < 0.0) tn = 0.0;
        st.t[p] = tn;
    }
}

__global__ void __launch_bounds__(EXACT_WPB * 32) solve_exact_kernel(const klnmf_solve_args_t a) {
    extern __shared__ double xs_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t slot = (int64_t)blockIdx.x * EXACT_WPB + warp;
    if (slot >= a.n_items) return;  // warp-uniform
    const int r = a.r, rp = a.rp;
    double *xs = xs_all + (int64_t)warp * rp;
    const double *fixed = static_cast<const double *>(a.fixed);
    double *moving = static_cast<double *>(a.moving);
    const int64_t j = a.items ? a.items[slot] : slot;
    const int64_t lo = a.side.ptr[j];
    ExactState st;
    st.s = a.side.ptr[j + 1] - lo;
    st.vi = a.side.idx + lo;
    st.vv = static_cast<const double *>(a.side.val) + lo;
    st.t = a.scratch + lo;

    // x <- moving[:, j] (sweep_range, _kernels.py:135-136), re-ordered to visit order
    for (int k = lane; k < r; k += 32) xs[k] = moving[j * rp + a.perm_in[k]];
    __syncwarp();

    // compute_ax (_kernels.py:39-50): natural k order, exact zeros of x skipped
    for (int64_t p = lane; p < st.s; p += 32) {
        const double *row = fixed + (int64_t)st.vi[p] * rp;
        double acc = 0.0;
        for (int k = 0; k < r; ++k) {
            const int pos = a.nat_pos[k];
            const double xk = xs[pos];
            if (xk != 0.0) acc = __dadd_rn(acc, __dmul_rn(xk, __ldg(row + pos)));
        }
        st.t[p] = acc;
    }
    __syncwarp();

    unsigned long long n_cap = 0, n_deg = 0, n_inner = 0, n_pass = 0;
    const double eg = a.eps_grad;
    const int max_passes = a.max_passes > 0 ? a.max_passes : 1;
    // solve_column body (_kernels.py:70-120): passes until one moves nothing
    for (int pass = 0; pass < max_passes; ++pass) {
      ++n_pass;
      bool moved = false;
      for (int tt = 0; tt < r; ++tt) {
        double x = xs[tt];
        const double x_enter = x;
        double g, h;
        exact_grad_hess(a, fixed, st, tt, x, &g, &h, lane);
        int64_t inner = 0;
        while ((g < -eg) || (fabs(g) > eg && x > eg)) {
            if (h <= 0.0) {
                if (g > 0.0) {
                    const double delta = -x;
                    if (delta != 0.0) {
                        exact_update(a, fixed, st, tt, delta, lane);
                        x = 0.0;
                    }
                } else {
                    ++n_deg;
                }
                break;
            }
            double target = __dsub_rn(x, __ddiv_rn(g, h));
            if (target < 0.0) target = 0.0;
            const double delta = __dsub_rn(target, x);
            exact_update(a, fixed, st, tt, delta, lane);
            const double xs_old = x;
            x = __dadd_rn(xs_old, delta);
            ++inner;
            ++n_inner;
            if (fabs(delta) < __dmul_rn(a.eps_x, xs_old)) break;
            if (inner >= a.inner_cap) {
                ++n_cap;
                break;
            }
            __syncwarp();
            exact_grad_hess(a, fixed, st, tt, x, &g, &h, lane);
        }
        __syncwarp();
        if (lane == 0) xs[tt] = x;
        __syncwarp();
        if (x != x_enter) moved = true;  // warp-uniform: every lane holds the same x
      }
      if (!moved) break;
    }
    // moving[:, j] <- x (_kernels.py:143-144), written in the next visit order
    for (int k = lane; k < r; k += 32) moving[j * rp + a.perm_out[k]] = xs[k];
    if (lane == 0 && a.stats) {
        if (n_cap) atomicAdd(a.stats + KLNMF_STAT_CAP_HITS, n_cap);
        if (n_deg) atomicAdd(a.stats + KLNMF_STAT_DEGENERATE, n_deg);
        if (n_inner) atomicAdd(a.stats + KLNMF_STAT_INNER_ITERS, n_inner);
        atomicAdd(a.stats + KLNMF_STAT_PASSES, n_pass);
    }
}

// kkt_violation (_kernels.py:176-190) of every subproblem at its current x:
// compute_ax, then per coordinate (natural order) the exact gradient and
// Hessian diagonal and the reference's violation measure; out is (n_mov, rp)
// by position.
__global__ void __launch_bounds__(EXACT_WPB * 32) kkt_exact_kernel(const klnmf_solve_args_t a, double *out) {
    extern __shared__ double xs_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t slot = (int64_t)blockIdx.x * EXACT_WPB + warp;
    if (slot >= a.n_items) return;
    const int r = a.r, rp = a.rp;
    double *xs = xs_all + (int64_t)warp * rp;
    const double *fixed = static_cast<const double *>(a.fixed);
    const double *moving = static_cast<const double *>(a.moving);
    const int64_t j = a.items ? a.items[slot] : slot;
    const int64_t lo = a.side.ptr[j];
    ExactState st;
    st.s = a.side.ptr[j + 1] - lo;
    st.vi = a.side.idx + lo;
    st.vv = static_cast<const double *>(a.side.val) + lo;
    st.t = a.scratch + lo;
    for (int k = lane; k < r; k += 32) xs[k] = moving[j * rp + a.perm_in[k]];
    __syncwarp();
    for (int64_t p = lane; p < st.s; p += 32) {
        const double *row = fixed + (int64_t)st.vi[p] * rp;
        double acc = 0.0;
        for (int k = 0; k < r; ++k) {
            const int pos = a.nat_pos[k];
            const double xk = xs[pos];
            if (xk != 0.0) acc = __dadd_rn(acc, __dmul_rn(xk, __ldg(row + pos)));
        }
        st.t[p] = acc;
    }
    __syncwarp();
    const double eg = a.eps_grad;
    for (int tt = 0; tt < r; ++tt) {
        const double x = xs[tt];
        double g, h;
        exact_grad_hess(a, fixed, st, tt, x, &g, &h, lane);
        double v;
        if (x <= eg) {
            v = fmax(0.0, __dsub_rn(-g, eg));
        } else {
            const double scale = fmax(eg, __dmul_rn(__dmul_rn(a.eps_x, x), h));
            v = fmax(0.0, __dsub_rn(fabs(g), scale));
        }
        if (lane == 0) out[j * rp + tt] = v;
    }
}

// mu_update_range (_kernels.py:193-214) for every listed subproblem, bit for
// bit: lanes compute the per-entry data ratios (serial r-dots, natural k
// order), then each lane owns coordinates and folds the entries in order.
// Factors are (n, rp) item-major in natural order; ratio is nnz scratch.
__global__ void __launch_bounds__(EXACT_WPB * 32) mu_exact_kernel(const klnmf_side_t side, const double *fixed,
                                                                  double *moving, const double *sum_fixed, int r,
                                                                  int rp, double eps_mu, const int32_t *items,
                                                                  int64_t n_items, double *ratio) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t slot = (int64_t)blockIdx.x * EXACT_WPB + warp;
    if (slot >= n_items) return;
    const int64_t j = items ? items[slot] : slot;
    const int64_t lo = side.ptr[j], s = side.ptr[j + 1] - lo;
    const int32_t *idx = side.idx + lo;
    const double *val = static_cast<const double *>(side.val) + lo;
    double *mj = moving + j * rp;
    for (int64_t p = lane; p < s; p += 32) {
        const double *row = fixed + (int64_t)idx[p] * rp;
        double d = 0.0;
        for (int k = 0; k < r; ++k) d = __dadd_rn(d, __dmul_rn(row[k], mj[k]));
        ratio[lo + p] = __ddiv_rn(val[p], __dadd_rn(d, eps_mu));
    }
    __syncwarp();
    for (int k = lane; k < r; k += 32) {
        double num = 0.0;
        for (int64_t p = 0; p < s; ++p) num = __dadd_rn(num, __dmul_rn(fixed[(int64_t)idx[p] * rp + k], ratio[lo + p]));
        mj[k] = __ddiv_rn(__dmul_rn(mj[k], __dadd_rn(num, eps_mu)), __dadd_rn(sum_fixed[k], eps_mu));
    }
}

// numpy pairwise_sum leaf (n <= 128), loops_utils.h.src
__device__ double pw_leaf(const double *a, int64_t n, int64_t stride) {
    if (n < 8) {
        double res = 0.;
        for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = a[q * stride];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], a[(i + q) * stride]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
    return res;
}

// Iterative form of numpy's recursion: n <= 128 is a leaf, otherwise split at
// n2 = n/2 - (n/2)%8 and return left + right.
__device__ double pw_sum(const double *a, int64_t n, int64_t stride) {
    int64_t off[64], len[64];
    double left[64];
    int state[64];
    int sp = 0;
    off[0] = 0;
    len[0] = n;
    state[0] = 0;
    for (;;) {
        if (len[sp] <= 128) {
            double v = pw_leaf(a + off[sp] * stride, len[sp], stride);
            --sp;
            for (;;) {
                if (sp < 0) return v;
                if (state[sp] == 0) {  // left child done: remember it, descend right
                    left[sp] = v;
                    state[sp] = 1;
                    int64_t n2 = len[sp] / 2;
                    n2 -= n2 % 8;
                    off[sp + 1] = off[sp] + n2;
                    len[sp + 1] = len[sp] - n2;
                    state[sp + 1] = 0;
                    ++sp;
                    break;
                }
                v = __dadd_rn(left[sp], v);  // right child done
                --sp;
            }
        } else {
            int64_t n2 = len[sp] / 2;
            n2 -= n2 % 8;
            off[sp + 1] = off[sp];
            len[sp + 1] = n2;
            state[sp + 1] = 0;
            ++sp;
        }
    }
}

__global__ void row_sums_pairwise_kernel(const double *fac, int64_t n_items, int64_t stride,
                                         int64_t col_stride, int32_t r, double *out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= r) return;
    out[k] = pw_sum(fac + (int64_t)k * col_stride, n_items, stride);
}

// kl_data_term per-entry terms (_kernels.py:152-159): d accumulated in natural
// k order with mul-then-add, then v*log(v/(d+eps)) - v; block sums in a fixed tree.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) kl_terms_kernel(const int64_t *ptr, const int32_t *idx,
                                                      const T *val, int64_t n_cols, int64_t nnz,
                                                      const T *w, const T *f, int32_t rp,
                                                      const int32_t *wpos, const int32_t *fpos,
                                                      int32_t r, double eps, double *partial) {
    __shared__ double sh[NT / 32];
    const int64_t q = (int64_t)blockIdx.x * NT + threadIdx.x;
    double term = 0.0;
    if (q < nnz) {
        // column of entry q: upper_bound(ptr, q) - 1
        int64_t lo = 0, hi = n_cols;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ptr[mid + 1] <= q) lo = mid + 1; else hi = mid;
        }
        const int64_t j = lo;
        const int64_t i = idx[q];
        double d = 0.0;
        for (int k = 0; k < r; ++k)
            d = __dadd_rn(d, __dmul_rn((double)w[i * rp + wpos[k]], (double)f[j * rp + fpos[k]]));
        const double v = (double)val[q];
        term = __dsub_rn(__dmul_rn(v, log(__ddiv_rn(v, __dadd_rn(d, eps)))), v);
    }
    const double tot = block_sum_det<NT>(term, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void sum_partials_kernel(const double *partial, int64_t n, double *out) {
    // single thread, fixed order
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s = __dadd_rn(s, partial[i]);
        out[0] = s;
    }
}

}  // namespace

}  // namespace klnmf

using namespace klnmf;

extern "C" int klnmf_kkt_exact(const klnmf_solve_args_t *args, double *out, void *stream) {
    if (args->n_items <= 0) return 0;
    const int64_t blocks = (args->n_items + EXACT_WPB - 1) / EXACT_WPB;
    const size_t smem = sizeof(double) * (size_t)EXACT_WPB * (size_t)args->rp;
    if (smem > 48 * 1024) KLNMF_CHECK(ensure_smem((const void *)kkt_exact_kernel, smem));
    kkt_exact_kernel<<<(unsigned)blocks, EXACT_WPB * 32, smem, as_stream(stream)>>>(*args, out);
    KLNMF_CHECK_LAUNCH("kkt_exact_kernel");
    return 0;
}

extern "C" int klnmf_mu_update_dev(const klnmf_side_t *side, const double *fixed, double *moving,
                                   const double *sum_fixed, int32_t r, int32_t rp, double eps_mu,
                                   const int32_t *items, int64_t n_items, double *ratio_scratch, void *stream) {
    if (n_items <= 0) return 0;
    const int64_t blocks = (n_items + EXACT_WPB - 1) / EXACT_WPB;
    mu_exact_kernel<<<(unsigned)blocks, EXACT_WPB * 32, 0, as_stream(stream)>>>(*side, fixed, moving, sum_fixed, r,
                                                                               rp, eps_mu, items, n_items,
                                                                               ratio_scratch);
    KLNMF_CHECK_LAUNCH("mu_exact_kernel");
    return 0;
}

extern "C" int klnmf_solve_exact(const klnmf_solve_args_t *args, void *stream) {
    if (args->n_items <= 0) return 0;
    if (args->order_mode != KLNMF_ORDER_SHARED)
        return set_error_msg(1, "klnmf_solve_exact: the exact mode visits the shared (reference) order only");
    if (args->n_peers != 0)
        return set_error_msg(1, "klnmf_solve_exact: the fused peer exchange is an fp32-mode path (exact mode all-gathers)");
    const int64_t blocks = (args->n_items + EXACT_WPB - 1) / EXACT_WPB;
    const size_t smem = sizeof(double) * (size_t)EXACT_WPB * (size_t)args->rp;
    if (smem > 48 * 1024) KLNMF_CHECK(ensure_smem((const void *)solve_exact_kernel, smem));
    solve_exact_kernel<<<(unsigned)blocks, EXACT_WPB * 32, smem, as_stream(stream)>>>(*args);
    KLNMF_CHECK_LAUNCH("solve_exact_kernel");
    return 0;
}

extern "C" int klnmf_row_sums_exact(const double *fac, int64_t n_items, int32_t rp, int32_t r,
                                    double *out, void *stream) {
    if (r <= 0) return 0;
    row_sums_pairwise_kernel<<<(r + 31) / 32, 32, 0, as_stream(stream)>>>(fac, n_items, rp, 1, r, out);
    KLNMF_CHECK_LAUNCH("row_sums_pairwise_kernel");
    return 0;
}

// Reference-layout pairwise row sums (factor (r, n) C-order) on device memory.
namespace klnmf {
int row_sums_ref_layout(const double *fac_dev, int64_t r, int64_t n, double *out_dev, cudaStream_t st) {
    if (r <= 0) return 0;
    row_sums_pairwise_kernel<<<(unsigned)((r + 31) / 32), 32, 0, st>>>(fac_dev, n, 1, n, (int32_t)r, out_dev);
    KLNMF_CHECK_LAUNCH("row_sums_pairwise_kernel");
    return 0;
}
}  // namespace klnmf

extern "C" int klnmf_kl_data_term_dev(const klnmf_side_t *csc, const void *w, const void *f,
                                      int32_t rp, const int32_t *wpos, const int32_t *fpos,
                                      int32_t r, int fp32, double eps_div, double *out_host,
                                      void *stream) {
    cudaStream_t st = as_stream(stream);
    constexpr int NT = 256;
    const int64_t nnz = csc->nnz;
    const int64_t blocks = nnz > 0 ? (nnz + NT - 1) / NT : 1;
    double *partial = nullptr;
    KLNMF_CHECK(keep_async_pool());
    KLNMF_CHECK(cudaMallocAsync(&partial, sizeof(double) * (size_t)(blocks + 1), st));
    if (nnz > 0) {
        if (fp32)
            kl_terms_kernel<float, NT><<<(unsigned)blocks, NT, 0, st>>>(
                csc->ptr, csc->idx, static_cast<const float *>(csc->val), csc->n_mov, nnz,
                static_cast<const float *>(w), static_cast<const float *>(f), rp, wpos, fpos, r,
                eps_div, partial);
        else
            kl_terms_kernel<double, NT><<<(unsigned)blocks, NT, 0, st>>>(
                csc->ptr, csc->idx, static_cast<const double *>(csc->val), csc->n_mov, nnz,
                static_cast<const double *>(w), static_cast<const double *>(f), rp, wpos, fpos, r,
                eps_div, partial);
        KLNMF_CHECK_LAUNCH("kl_terms_kernel");
    } else {
        KLNMF_CHECK(cudaMemsetAsync(partial, 0, sizeof(double), st));
    }
    sum_partials_kernel<<<1, 32, 0, st>>>(partial, nnz > 0 ? blocks : 1, partial + blocks);
    KLNMF_CHECK_LAUNCH("sum_partials_kernel");
    KLNMF_CHECK(cudaMemcpyAsync(out_host, partial + blocks, sizeof(double), cudaMemcpyDeviceToHost, st));
    KLNMF_CHECK(cudaFreeAsync(partial, st));
    KLNMF_CHECK(cudaStreamSynchronize(st));
    return 0;
}
