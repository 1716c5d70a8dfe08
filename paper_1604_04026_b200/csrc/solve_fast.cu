// fp32-storage / fp64-arithmetic subproblem solver (throughput mode).
//
// Algorithm: the reference's solve_column with max_passes = 1
// (_kernels.py:53-120, driven by sweep_range :123-144), restated for the
// device:
//   * the maintained product t is kept on the column support S only and is
//     CARRIED between half-steps (t at entry (i,j) is <W_i, F_j> for both
//     sides), so no subproblem recomputes it from the fixed factor;
//   * per entry the kernel keeps u = v/(t+eps) and z = u/(t+eps) so that
//     _grad_hess (_kernels.py:24-36) becomes g = sum_a + alpha*x + beta -
//     sum(u*a), h = alpha + sum(z*a*a): one FMA pair per (entry, coordinate)
//     and one reciprocal per entry per Newton step (instead of one division
//     per (entry, coordinate)); entries with a == 0 are skipped exactly as the
//     reference does;
//   * every Newton step rounds the coordinate to fp32 (the storage type), so
//     t stays consistent with the stored factors;
//   * coordinates are visited in storage order (the factors are stored in the
//     iteration's visit order), so each subproblem streams its gathered rows
//     of the fixed factor front to back in 16-byte chunks of 4 coordinates.
//
// Kernel family (one launch per nnz bucket, largest subproblems first):
//   solve_fast_kernel<L, NPL, NT>   L lanes per subproblem (L <= 32: 32/L
//       subproblems per warp, lock-step over coordinates; L > 32: one
//       subproblem per block), NPL entries per lane held in registers.
//   solve_fast_stream_kernel<NT>    one block per subproblem, any size,
//       per-entry state in global scratch (the long rows of the W-side).
#include "common.cuh"

namespace klnmf {
namespace {

template <int L, int NT>
struct Group {
    static_assert((L & (L - 1)) == 0, "L must be a power of two");
    static_assert(L <= 32 || L == NT, "multi-warp groups span the whole block");
    static constexpr int NW = NT / 32;
    static_assert(NW >= 1, "at least one warp");

    __device__ __forceinline__ static void reduce2(double &x, double &y, double *red, int &buf) {
        if constexpr (L <= 32) {
#pragma unroll
            for (int o = L / 2; o > 0; o >>= 1) {
                x += __shfl_xor_sync(FULL_MASK, x, o);
                y += __shfl_xor_sync(FULL_MASK, y, o);
            }
        } else {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                x += __shfl_xor_sync(FULL_MASK, x, o);
                y += __shfl_xor_sync(FULL_MASK, y, o);
            }
            const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
            double *r = red + buf * NW * 2;
            if (lane == 0) {
                r[2 * w] = x;
                r[2 * w + 1] = y;
            }
            __syncthreads();
            double sx = 0.0, sy = 0.0;
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                sx += r[2 * i];
                sy += r[2 * i + 1];
            }
            x = sx;
            y = sy;
            buf ^= 1;  // double buffer: one barrier per reduction is enough
        }
    }
    __device__ __forceinline__ static bool any(bool p) {
        if constexpr (L <= 32) return __any_sync(FULL_MASK, p);
        else return p;  // block-uniform by construction
    }
    __device__ __forceinline__ static void sync() {
        if constexpr (L <= 32) __syncwarp();
        else __syncthreads();
    }
};

struct Counters {
    unsigned n_inner = 0, n_cap = 0, n_deg = 0;
};

// Newton logic of one coordinate step (_kernels.py:78-115), fp32-rounded x.
// Returns the applied delta; clears `active` when the inner loop ends and sets
// `again` when it needs another gradient evaluation.
__device__ __forceinline__ double newton_step(double g, double h, double &x, int &inner, bool &active,
                                              bool &again, const klnmf_solve_args_t &a, Counters &cnt) {
    double delta = 0.0;
    again = false;
    if (h <= 0.0) {
        // zero curvature: positive slope sends the coordinate to the bound
        if (g > 0.0) {
            if (x != 0.0) {
                delta = -x;
                x = 0.0;
            }
        } else {
            ++cnt.n_deg;
        }
        active = false;
        return delta;
    }
    double target = x - g / h;
    if (target < 0.0) target = 0.0;
    const double xn = (double)__double2float_rn(target);
    delta = xn - x;
    const double xo = x;
    x = xn;
    ++inner;
    ++cnt.n_inner;
    if (fabs(delta) < a.eps_x * xo) {
        active = false;
    } else if (inner >= a.inner_cap) {
        ++cnt.n_cap;
        active = false;
    } else {
        again = true;
    }
    return delta;
}

__device__ __forceinline__ bool enters(double g, double x, double eg) {
    return (g < -eg) || (fabs(g) > eg && x > eg);
}

template <int L, int NPL, int NT>
__global__ void __launch_bounds__(NT) solve_fast_kernel(const klnmf_solve_args_t a) {
    using G = Group<L, NT>;
    constexpr int GPB = (L <= 32) ? NT / L : 1;
    extern __shared__ float xs_all[];
    __shared__ double red[(L > 32) ? 2 * (NT / 32) * 2 : 2];

    const int tid = threadIdx.x;
    const int grp = (L <= 32) ? tid / L : 0;
    const int gl = (L <= 32) ? (tid & (L - 1)) : tid;
    const int rp = a.rp, r = a.r;
    const int rps = rp | 1;
    float *xs = xs_all + grp * rps;
    const int64_t slot = (int64_t)blockIdx.x * GPB + grp;
    const bool valid = slot < a.n_items;
    if constexpr (L > 32) {
        if (!valid) return;
    } else {
        if (!__any_sync(FULL_MASK, valid)) return;
    }

    const float *fixed = static_cast<const float *>(a.fixed);
    float *moving = static_cast<float *>(a.moving);
    const float *val = static_cast<const float *>(a.side.val);
    const int64_t j = valid ? (int64_t)a.items[slot] : 0;
    const int64_t lo = valid ? a.side.ptr[j] : 0;
    const int s = valid ? (int)(a.side.ptr[j + 1] - lo) : 0;

    for (int k = gl; k < r; k += L) xs[k] = valid ? moving[j * rp + a.perm_in[k]] : 0.f;

    double t[NPL], u[NPL], z[NPL];
    float v[NPL];
    int off[NPL];
#pragma unroll
    for (int e = 0; e < NPL; ++e) {
        const int p = gl + e * L;
        if (p < s) {
            const int64_t q = lo + p;
            off[e] = a.side.idx[q] * rp;
            v[e] = val[q];
            const double tq = a.t_in[a.tmap ? (int64_t)a.tmap[q] : q];
            t[e] = tq;
            const double ri = 1.0 / (tq + a.eps_div);
            u[e] = (double)v[e] * ri;
            z[e] = u[e] * ri;
        } else {
            off[e] = -1;
            v[e] = 0.f;
            t[e] = 0.0;
            u[e] = 0.0;
            z[e] = 0.0;
        }
    }
    G::sync();

    Counters cnt;
    int buf = 0;
    const double eg = a.eps_grad;

    for (int c = 0; c < r; c += 4) {
        float4 A[NPL];
#pragma unroll
        for (int e = 0; e < NPL; ++e)
            A[e] = off[e] >= 0 ? ldg_f4(fixed + off[e] + c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            const int tt = c + cc;
            if (tt >= r) break;  // uniform
            double ad[NPL];
#pragma unroll
            for (int e = 0; e < NPL; ++e) ad[e] = (double)f4_get(A[e], cc);
            const double sa = a.sum_pos[tt];
            double x = (double)xs[tt];

            auto eval = [&](double xv, double &g, double &h) {
                double gp = 0.0, hp = 0.0;
#pragma unroll
                for (int e = 0; e < NPL; ++e) {
                    if (ad[e] != 0.0) {
                        gp = fma(u[e], ad[e], gp);
                        hp = fma(z[e] * ad[e], ad[e], hp);
                    }
                }
                G::reduce2(gp, hp, red, buf);
                g = (sa + a.alpha * xv + a.beta) - gp;
                h = a.alpha + hp;
            };

            double g, h;
            eval(x, g, h);
            int inner = 0;
            bool active = valid && enters(g, x, eg);
            while (G::any(active)) {
                bool again = false;
                double delta = 0.0;
                if (active) delta = newton_step(g, h, x, inner, active, again, a, cnt);
                if (delta != 0.0) {
#pragma unroll
                    for (int e = 0; e < NPL; ++e) {
                        if (ad[e] != 0.0) {
                            double tn = fma(delta, ad[e], t[e]);
                            if (tn < 0.0) tn = 0.0;
                            t[e] = tn;
                            const double ri = 1.0 / (tn + a.eps_div);
                            u[e] = (double)v[e] * ri;
                            z[e] = u[e] * ri;
                        }
                    }
                }
                if (G::any(again)) {
                    double g2, h2;
                    eval(x, g2, h2);
                    if (again) {
                        g = g2;
                        h = h2;
                    }
                }
            }
            if (gl == 0 && valid) xs[tt] = (float)x;
        }
    }
    G::sync();
    if (valid) {
        for (int k = gl; k < r; k += L) moving[j * rp + a.perm_out[k]] = xs[k];
#pragma unroll
        for (int e = 0; e < NPL; ++e)
            if (off[e] >= 0) a.t_out[lo + gl + e * L] = t[e];
    }
    if (a.stats) {
        unsigned ci = (gl == 0 && valid) ? cnt.n_inner : 0u;
        unsigned cc_ = (gl == 0 && valid) ? cnt.n_cap : 0u;
        unsigned cd = (gl == 0 && valid) ? cnt.n_deg : 0u;
        unsigned cp = (gl == 0 && valid) ? 1u : 0u;
        if constexpr (L <= 32) {
            ci = __reduce_add_sync(FULL_MASK, ci);
            cc_ = __reduce_add_sync(FULL_MASK, cc_);
            cd = __reduce_add_sync(FULL_MASK, cd);
            cp = __reduce_add_sync(FULL_MASK, cp);
            if ((tid & 31) != 0) return;
        } else {
            if (tid != 0) return;
        }
        if (ci) atomicAdd(a.stats + KLNMF_STAT_INNER_ITERS, (unsigned long long)ci);
        if (cc_) atomicAdd(a.stats + KLNMF_STAT_CAP_HITS, (unsigned long long)cc_);
        if (cd) atomicAdd(a.stats + KLNMF_STAT_DEGENERATE, (unsigned long long)cd);
        if (cp) atomicAdd(a.stats + KLNMF_STAT_PASSES, (unsigned long long)cp);
    }
}

// Any-size subproblem, one block each; per-entry t/u/z live in global memory
// (t in t_out, u and z in scratch), each thread owning entries p = tid mod NT.
template <int NT>
__global__ void __launch_bounds__(NT) solve_fast_stream_kernel(const klnmf_solve_args_t a) {
    using G = Group<NT, NT>;
    extern __shared__ float xs[];
    __shared__ double red[2 * (NT / 32) * 2];
    const int tid = threadIdx.x;
    const int64_t slot = blockIdx.x;
    if (slot >= a.n_items) return;
    const int rp = a.rp, r = a.r;
    const float *fixed = static_cast<const float *>(a.fixed);
    float *moving = static_cast<float *>(a.moving);
    const float *val = static_cast<const float *>(a.side.val);
    const int64_t j = a.items[slot];
    const int64_t lo = a.side.ptr[j];
    const int64_t s = a.side.ptr[j + 1] - lo;
    double *T = a.t_out + lo;
    double *U = a.scratch + lo;
    double *Z = a.scratch + a.side.nnz + lo;
    const int32_t *vi = a.side.idx + lo;
    const float *vv = val + lo;

    for (int k = tid; k < r; k += NT) xs[k] = moving[j * rp + a.perm_in[k]];
    for (int64_t p = tid; p < s; p += NT) {
        const int64_t q = lo + p;
        const double tq = a.t_in[a.tmap ? (int64_t)a.tmap[q] : q];
        T[p] = tq;
        const double ri = 1.0 / (tq + a.eps_div);
        const double uu = (double)vv[p] * ri;
        U[p] = uu;
        Z[p] = uu * ri;
    }
    __syncthreads();

    Counters cnt;
    int buf = 0;
    const double eg = a.eps_grad;
    for (int tt = 0; tt < r; ++tt) {
        const double sa = a.sum_pos[tt];
        double x = (double)xs[tt];
        auto eval = [&](double xv, double &g, double &h) {
            double gp = 0.0, hp = 0.0;
            for (int64_t p = tid; p < s; p += NT) {
                const double av = (double)__ldg(fixed + (int64_t)vi[p] * rp + tt);
                if (av != 0.0) {
                    gp = fma(U[p], av, gp);
                    hp = fma(Z[p] * av, av, hp);
                }
            }
            G::reduce2(gp, hp, red, buf);
            g = (sa + a.alpha * xv + a.beta) - gp;
            h = a.alpha + hp;
        };
        double g, h;
        eval(x, g, h);
        int inner = 0;
        bool active = enters(g, x, eg);
        while (active) {
            bool again = false;
            const double delta = newton_step(g, h, x, inner, active, again, a, cnt);
            if (delta != 0.0) {
                for (int64_t p = tid; p < s; p += NT) {
                    const double av = (double)__ldg(fixed + (int64_t)vi[p] * rp + tt);
                    if (av != 0.0) {
                        double tn = fma(delta, av, T[p]);
                        if (tn < 0.0) tn = 0.0;
                        T[p] = tn;
                        const double ri = 1.0 / (tn + a.eps_div);
                        const double uu = (double)vv[p] * ri;
                        U[p] = uu;
                        Z[p] = uu * ri;
                    }
                }
            }
            if (again) eval(x, g, h);
        }
        if (tid == 0) xs[tt] = (float)x;
    }
    __syncthreads();
    for (int k = tid; k < r; k += NT) moving[j * rp + a.perm_out[k]] = xs[k];
    if (tid == 0 && a.stats) {
        if (cnt.n_inner) atomicAdd(a.stats + KLNMF_STAT_INNER_ITERS, (unsigned long long)cnt.n_inner);
        if (cnt.n_cap) atomicAdd(a.stats + KLNMF_STAT_CAP_HITS, (unsigned long long)cnt.n_cap);
        if (cnt.n_deg) atomicAdd(a.stats + KLNMF_STAT_DEGENERATE, (unsigned long long)cnt.n_deg);
        atomicAdd(a.stats + KLNMF_STAT_PASSES, 1ull);
    }
}

struct FastKernel {
    int lanes, npl, nt;
    int64_t capacity;  // -1 = unbounded
    void (*fn)(const klnmf_solve_args_t);
    int gpb;  // subproblems per block
};

#define FK(L, NPL, NT) {L, NPL, NT, (int64_t)(L) * (NPL), solve_fast_kernel<L, NPL, NT>, ((L) <= 32 ? (NT) / (L) : 1)}
const FastKernel kFast[] = {
    FK(1, 4, 128),  FK(2, 4, 128),  FK(4, 4, 128),   FK(8, 4, 128),   FK(8, 8, 128),
    FK(16, 8, 128), FK(32, 8, 128), FK(64, 8, 64),   FK(128, 8, 128), FK(256, 8, 256),
    {512, 0, 512, -1, solve_fast_stream_kernel<512>, 1},
};
#undef FK
constexpr int kNumFast = sizeof(kFast) / sizeof(kFast[0]);

}  // namespace
}  // namespace klnmf

using namespace klnmf;

extern "C" int klnmf_fast_kernel_count(void) { return kNumFast; }

extern "C" int klnmf_fast_kernel_info(int kernel_id, int64_t *capacity, int32_t *lanes, int32_t *npl) {
    if (kernel_id < 0 || kernel_id >= kNumFast) return set_error_msg(1, "klnmf_fast_kernel_info: bad kernel id");
    *capacity = kFast[kernel_id].capacity;
    *lanes = kFast[kernel_id].lanes;
    *npl = kFast[kernel_id].npl;
    return 0;
}

extern "C" int klnmf_solve_fast(const klnmf_solve_args_t *args, int kernel_id, void *stream) {
    if (kernel_id < 0 || kernel_id >= kNumFast) return set_error_msg(1, "klnmf_solve_fast: bad kernel id");
    if (args->n_items <= 0) return 0;
    if (args->rp % 4 != 0) return set_error_msg(1, "klnmf_solve_fast: rp must be a multiple of 4");
    const FastKernel &k = kFast[kernel_id];
    if (k.capacity < 0 && args->scratch == nullptr)
        return set_error_msg(1, "klnmf_solve_fast: the streaming kernel needs 2*nnz doubles of scratch");
    const int64_t blocks = (args->n_items + k.gpb - 1) / k.gpb;
    const size_t smem = sizeof(float) * (size_t)k.gpb * (size_t)(args->rp | 1);
    if (smem > 48 * 1024) {
        KLNMF_CHECK(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k.fn<<<(unsigned)blocks, k.nt, smem, as_stream(stream)>>>(*args);
    KLNMF_CHECK_LAUNCH("solve_fast_kernel");
    return 0;
}
