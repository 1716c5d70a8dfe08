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
//     sum(u*a), h = alpha + sum(z*a*a); entries with a == 0 are skipped as in
//     the reference;
//   * every Newton step rounds the coordinate to fp32 (the storage type), so
//     t stays consistent with the stored factors;
//   * coordinates are visited in storage order (factors are stored in the
//     iteration's visit order), 4 at a time: one pass over the subproblem's
//     entries produces the partial (g, h) sums of the next 4 coordinates
//     ("speculative" batch), one transposed reduction combines all 8 values,
//     and the coordinates are then consumed in order.  A coordinate that moves
//     changes t, so the remaining coordinates of the batch are re-evaluated:
//     every gradient is computed on exactly the t the sequential reference
//     would see.  At steady state ~5% of visits move (C4), so most batches
//     need a single pass;
//   * the gathered fixed-factor rows stream through a per-thread cp.async
//     ring in shared memory (16 B = 4 coordinates per entry per stage); each
//     thread only reads the copies it issued, so no barrier is needed.
//
// Kernels (one launch per nnz bucket, largest subproblems first):
//   solve_warp_kernel<L, NPL>   L <= 32 lanes per subproblem, 32/L subproblems
//       per warp in lock-step, NPL entries per lane in registers.
//   solve_block_kernel<NT, NPL> one subproblem per block (NT threads).
//   solve_stream_kernel<NT>     any size, one block per subproblem, per-entry
//       state in global memory (long rows of the W side).
#include <cooperative_groups.h>
#include <cstdio>
#include <type_traits>

#include "common.cuh"

namespace klnmf {
namespace {

constexpr int C = 4;       // coordinates per batch (16 B of fp32 per entry)
constexpr int NV = 2 * C;  // reduced values per pass: g partials then h partials
constexpr int STAGES = 3;  // cp.async ring depth
constexpr int KMAX_RP = 256;  // largest padded rank of the fp32 kernels (row sums staged in smem)

// Compile-time loop: f(std::integral_constant<int, I>) for I in [I0, N).
template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

// Adds one entry's contribution to a coordinate's (g, h) partial sums.
// The reference skips a == 0 (_kernels.py:32).  With eps_div > 0, u and z are
// finite, so an a == 0 term adds exactly +0.0 and the (if-converted, select-
// heavy) guard is dropped; GUARD keeps it for eps_div == 0, where u may be inf.
template <bool GUARD>
__device__ __forceinline__ void accum(double &g, double &h, double u, double z, double av) {
    if (!GUARD || av != 0.0) {
        g = fma(u, av, g);
        h = fma(z * av, av, h);
    }
}

struct Counters {
    unsigned n_inner = 0, n_cap = 0, n_deg = 0;
};

__device__ __forceinline__ bool enters(double g, double x, double eg) {
    return (g < -eg) || (fabs(g) > eg && x > eg);
}

// One Newton step of the inner loop (_kernels.py:78-115), x rounded to fp32.
// Returns the applied delta; clears `active` when the loop ends, sets `again`
// when the loop needs a fresh gradient.
__device__ __forceinline__ double newton_step(double g, double h, double &x, int &inner, bool &active,
                                              bool &again, const klnmf_solve_args_t &a, Counters &cnt) {
    double delta = 0.0;
    again = false;
    if (h <= 0.0) {
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

// 1/x: MUFU approximation refined by one Newton step (relative error ~1e-14,
// far below the fp32 storage rounding of this mode); x == 0 (only possible
// with eps_div == 0) returns inf like the IEEE division.
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    return x == 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : r;
}

// Move of the visited coordinate by delta at an entry with a != 0: the
// maintained product and its derived u = v/(t+eps), z = u/(t+eps).  The clamp
// at 0 is the reference's (_kernels.py:105-106).
__device__ __forceinline__ void entry_update(double delta, double av, float v, double eps, double &t, double &u,
                                             double &z) {
    const double tn = fmax(fma(delta, av, t), 0.0);
    t = tn;
    const double ri = fast_rcp(tn + eps);
    u = (double)v * ri;
    z = u * ri;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 16 : 0;  // zero-fill when the entry does not exist
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Transposed reduction of NV values across the L lanes of a group: after it
// each lane holds KEEP totals; lane_of(i)/slot_of(i) locate value i.
template <int L>
struct TReduce {
    static constexpr int NL = (L == 1) ? 0 : (L == 2) ? 1 : (L == 4) ? 2 : (L == 8) ? 3 : (L == 16) ? 4 : 5;
    static constexpr int HL = NL < 3 ? NL : 3;  // halving levels (NV = 8 = 2^3)
    static constexpr int KEEP = NV >> HL;       // values per lane afterwards

    __device__ __forceinline__ static void run(double (&v)[NV], int gl) {
        int cur = NV;
#pragma unroll
        for (int lvl = 0; lvl < NL; ++lvl) {
            const int o = L >> (lvl + 1);
            if (lvl < HL) {
                const bool up = (gl & o) != 0;
                const int half = cur >> 1;
#pragma unroll
                for (int i = 0; i < NV / 2; ++i) {
                    if (i < half) {
                        const double send = up ? v[i] : v[i + half];
                        const double keep = up ? v[i + half] : v[i];
                        v[i] = keep + __shfl_xor_sync(FULL_MASK, send, o);
                    }
                }
                cur = half;
            } else {
                v[0] += __shfl_xor_sync(FULL_MASK, v[0], o);
            }
        }
    }
    __host__ __device__ static constexpr int lane_of(int i) { return (i / KEEP) << (NL - HL); }
    __host__ __device__ static constexpr int slot_of(int i) { return i % KEEP; }
};

template <int L>
__device__ __forceinline__ double fetch(const double (&v)[NV], int i) {
    using R = TReduce<L>;
    if constexpr (L == 1) {
        return v[i];
    } else {
        double val = v[0];
#pragma unroll
        for (int s = 1; s < R::KEEP; ++s)
            if (s == R::slot_of(i)) val = v[s];
        return __shfl_sync(FULL_MASK, val, R::lane_of(i), L);
    }
}

// ---------------------------------------------------------------------------
// Warp kernel: groups of L <= 32 lanes, 32/L subproblems per warp in lock-step.
template <int L, int NPL>
__global__ void __launch_bounds__(128) solve_warp_kernel(const klnmf_solve_args_t a) {
    constexpr int NT = 128;
    constexpr int GPB = NT / L;  // groups per block
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4 *ring = reinterpret_cast<float4 *>(smem_raw);                 // [STAGES][NPL][NT]
    float *xs_all = reinterpret_cast<float *>(ring + STAGES * NPL * NT);  // [GPB][2][rps]

    const int tid = threadIdx.x;
    const int grp = tid / L;
    const int gl = tid & (L - 1);
    const int rp = a.rp, r = a.r;
    const int rps = rp | 1;
    // xs: the row as read (never written during the sweep), xo: the result.
    // Separate buffers: without a per-coordinate barrier, overwriting xs[tt]
    // could race with a lagging lane still reading the old value.
    float *xs = xs_all + grp * 2 * rps;
    float *xo = xs + rps;
    const int64_t slot = (int64_t)blockIdx.x * GPB + grp;
    const bool valid = slot < a.n_items;
    __shared__ double ssum[KMAX_RP];  // fixed-factor row sums by position
    for (int k = tid; k < r; k += NT) ssum[k] = a.sum_pos[k];
    __syncthreads();
    if (!__any_sync(FULL_MASK, valid)) return;

    const float *fixed = static_cast<const float *>(a.fixed);
    float *moving = static_cast<float *>(a.moving);
    const float *val = static_cast<const float *>(a.side.val);
    const int64_t j = valid ? (int64_t)a.items[slot] : 0;
    const int64_t lo = valid ? a.side.ptr[j] : 0;
    const int s = valid ? (int)(a.side.ptr[j + 1] - lo) : 0;

    for (int k = gl; k < r; k += L) xs[k] = valid ? moving[j * rp + a.perm_in[k]] : 0.f;

    double t[NPL], u[NPL], z[NPL];
    float v[NPL];
    int off[NPL];  // row offset of the entry in the fixed factor, -1 = none
#pragma unroll
    for (int e = 0; e < NPL; ++e) {
        const int p = gl + e * L;
        if (p < s) {
            const int64_t q = lo + p;
            off[e] = a.side.idx[q] * rp;
            v[e] = val[q];
            const double tq = a.t_in[a.tmap ? (int64_t)a.tmap[q] : q];
            t[e] = tq;
            const double ri = fast_rcp(tq + a.eps_div);
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
    const int nchunks = (r + C - 1) / C;
    // prologue: STAGES-1 chunks in flight
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nchunks) {
#pragma unroll
            for (int e = 0; e < NPL; ++e)
                cp_async16(&ring[(st * NPL + e) * NT + tid], off[e] >= 0 ? fixed + off[e] + st * C : fixed, off[e] >= 0);
        }
        cp_commit();
    }
    __syncwarp();

    Counters cnt;
    const double eg = a.eps_grad, eps = a.eps_div, alpha = a.alpha;

    for (int ch = 0; ch < nchunks; ++ch) {
        // issue chunk ch + STAGES - 1, then wait for chunk ch
        {
            const int nx = ch + STAGES - 1;
            if (nx < nchunks) {
                const int st = nx % STAGES;
#pragma unroll
                for (int e = 0; e < NPL; ++e)
                    cp_async16(&ring[(st * NPL + e) * NT + tid], off[e] >= 0 ? fixed + off[e] + nx * C : fixed,
                               off[e] >= 0);
            }
            cp_commit();
            cp_wait<STAGES - 1>();
        }
        const float4 *Ach = ring + (ch % STAGES) * NPL * NT + tid;  // own slots of this stage

        double red[NV];
        bool fresh = false;  // partials valid for the current t
        static_for<0, C>([&](auto cc_c) {  // compile-time coordinate index
            constexpr int cc = decltype(cc_c)::value;
            const int tt = ch * C + cc;
            if (tt >= r) return;
            if (__any_sync(FULL_MASK, !fresh)) {
                // pass: partial sums of coordinates cc..C-1 on the current t
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
                auto pass = [&](auto guard) {
#pragma unroll
                    for (int e = 0; e < NPL; ++e) {
                        const float4 a4 = Ach[e * NT];
#pragma unroll
                        for (int q = cc; q < C; ++q)
                            accum<decltype(guard)::value>(red[q], red[C + q], u[e], z[e], (double)f4_get(a4, q));
                    }
                };
                if (eps > 0.0) pass(std::false_type{});
                else pass(std::true_type{});
                TReduce<L>::run(red, gl);
                fresh = true;
            }
            const double gp = fetch<L>(red, cc);
            const double hp = fetch<L>(red, C + cc);
            double x = (double)xs[tt];
            const double base = ssum[tt];
            double g = (base + alpha * x + a.beta) - gp;
            double h = alpha + hp;
            int inner = 0;
            bool active = valid && enters(g, x, eg);
            bool moved = false;
            while (__any_sync(FULL_MASK, active)) {
                bool again = false;
                double delta = 0.0;
                if (active) delta = newton_step(g, h, x, inner, active, again, a, cnt);
                if (delta != 0.0) {
                    moved = true;
#pragma unroll
                    for (int e = 0; e < NPL; ++e) {
                        const double av = (double)reinterpret_cast<const float *>(Ach + e * NT)[cc];
                        if (av != 0.0) entry_update(delta, av, v[e], eps, t[e], u[e], z[e]);
                    }
                }
                if (__any_sync(FULL_MASK, again)) {
                    double g2 = 0.0, h2 = 0.0;
#pragma unroll
                    for (int e = 0; e < NPL; ++e) {
                        const double av = (double)reinterpret_cast<const float *>(Ach + e * NT)[cc];
                        if (av != 0.0) {
                            g2 = fma(u[e], av, g2);
                            h2 = fma(z[e] * av, av, h2);
                        }
                    }
#pragma unroll
                    for (int o = L / 2; o > 0; o >>= 1) {
                        g2 += __shfl_xor_sync(FULL_MASK, g2, o);
                        h2 += __shfl_xor_sync(FULL_MASK, h2, o);
                    }
                    if (again) {
                        g = (base + alpha * x + a.beta) - g2;
                        h = alpha + h2;
                        active = enters(g, x, eg);  // _kernels.py:78
                    }
                }
            }
            if (moved) fresh = false;
            if (gl == 0 && valid) xo[tt] = (float)x;
        });
    }
    cp_wait<0>();
    __syncwarp();
    if (valid) {
        for (int k = gl; k < r; k += L) moving[j * rp + a.perm_out[k]] = xo[k];
#pragma unroll
        for (int e = 0; e < NPL; ++e)
            if (off[e] >= 0) a.t_out[lo + gl + e * L] = t[e];
    }
    if (a.stats) {
        const bool lead = gl == 0 && valid;
        const unsigned ci = __reduce_add_sync(FULL_MASK, lead ? cnt.n_inner : 0u);
        const unsigned cc_ = __reduce_add_sync(FULL_MASK, lead ? cnt.n_cap : 0u);
        const unsigned cd = __reduce_add_sync(FULL_MASK, lead ? cnt.n_deg : 0u);
        const unsigned cp = __reduce_add_sync(FULL_MASK, lead ? 1u : 0u);
        if ((tid & 31) == 0) {
            if (ci) atomicAdd(a.stats + KLNMF_STAT_INNER_ITERS, (unsigned long long)ci);
            if (cc_) atomicAdd(a.stats + KLNMF_STAT_CAP_HITS, (unsigned long long)cc_);
            if (cd) atomicAdd(a.stats + KLNMF_STAT_DEGENERATE, (unsigned long long)cd);
            if (cp) atomicAdd(a.stats + KLNMF_STAT_PASSES, (unsigned long long)cp);
        }
    }
}

// ---------------------------------------------------------------------------
// Block-wide reduction of NV values: warp transposed reduce, then per-warp
// totals through shared memory (double-buffered, one barrier per reduction);
// every thread ends with all NV totals (identical, fixed order).
template <int NT>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double *sred, int &buf) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    TReduce<32>::run(v, lane);
    double *r = sred + buf * NW * NV;
    // lane (i << 2) holds total i of this warp
    if ((lane & 3) == 0) r[w * NV + (lane >> 2)] = v[0];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) s += r[q * NV + i];
        v[i] = s;
    }
    buf ^= 1;
}

template <int NT>
__device__ __forceinline__ void block_reduce2(double &g, double &h, double *sred, int &buf) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        g += __shfl_xor_sync(FULL_MASK, g, o);
        h += __shfl_xor_sync(FULL_MASK, h, o);
    }
    double *r = sred + buf * NW * NV;
    if (lane == 0) {
        r[w * NV] = g;
        r[w * NV + 1] = h;
    }
    __syncthreads();
    double sg = 0.0, sh = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
        sg += r[q * NV];
        sh += r[q * NV + 1];
    }
    g = sg;
    h = sh;
    buf ^= 1;
}

// One subproblem per block, NPL register entries per thread.
template <int NT, int NPL>
__global__ void __launch_bounds__(NT) solve_block_kernel(const klnmf_solve_args_t a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4 *ring = reinterpret_cast<float4 *>(smem_raw);             // [STAGES][NPL][NT]
    float *xs = reinterpret_cast<float *>(ring + STAGES * NPL * NT);  // [2][rps]: input row, result
    float *xo = xs + (a.rp | 1);
    __shared__ double sred[2 * (NT / 32) * NV];

    const int tid = threadIdx.x;
    const int64_t slot = blockIdx.x;
    if (slot >= a.n_items) return;
    const int rp = a.rp, r = a.r;
    const float *fixed = static_cast<const float *>(a.fixed);
    float *moving = static_cast<float *>(a.moving);
    const float *val = static_cast<const float *>(a.side.val);
    const int64_t j = a.items[slot];
    const int64_t lo = a.side.ptr[j];
    const int s = (int)(a.side.ptr[j + 1] - lo);

    __shared__ double ssum[KMAX_RP];
    for (int k = tid; k < r; k += NT) ssum[k] = a.sum_pos[k];
    for (int k = tid; k < r; k += NT) xs[k] = moving[j * rp + a.perm_in[k]];

    double t[NPL], u[NPL], z[NPL];
    float v[NPL];
    int off[NPL];  // row offset of the entry in the fixed factor, -1 = none
#pragma unroll
    for (int e = 0; e < NPL; ++e) {
        const int p = tid + e * NT;
        if (p < s) {
            const int64_t q = lo + p;
            off[e] = a.side.idx[q] * rp;
            v[e] = val[q];
            const double tq = a.t_in[a.tmap ? (int64_t)a.tmap[q] : q];
            t[e] = tq;
            const double ri = fast_rcp(tq + a.eps_div);
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
    const int nchunks = (r + C - 1) / C;
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nchunks) {
#pragma unroll
            for (int e = 0; e < NPL; ++e)
                cp_async16(&ring[(st * NPL + e) * NT + tid], off[e] >= 0 ? fixed + off[e] + st * C : fixed, off[e] >= 0);
        }
        cp_commit();
    }
    __syncthreads();

    Counters cnt;
    int buf = 0;
    const double eg = a.eps_grad, eps = a.eps_div, alpha = a.alpha;
    for (int ch = 0; ch < nchunks; ++ch) {
        {
            const int nx = ch + STAGES - 1;
            if (nx < nchunks) {
                const int st = nx % STAGES;
#pragma unroll
                for (int e = 0; e < NPL; ++e)
                    cp_async16(&ring[(st * NPL + e) * NT + tid], off[e] >= 0 ? fixed + off[e] + nx * C : fixed,
                               off[e] >= 0);
            }
            cp_commit();
            cp_wait<STAGES - 1>();
        }
        const float4 *Ach = ring + (ch % STAGES) * NPL * NT + tid;  // own slots of this stage

        double red[NV];
        bool fresh = false;
        static_for<0, C>([&](auto cc_c) {  // compile-time coordinate index
            constexpr int cc = decltype(cc_c)::value;
            const int tt = ch * C + cc;
            if (tt >= r) return;
            if (!fresh) {
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
                auto pass = [&](auto guard) {
#pragma unroll
                    for (int e = 0; e < NPL; ++e) {
                        const float4 a4 = Ach[e * NT];
#pragma unroll
                        for (int q = cc; q < C; ++q)
                            accum<decltype(guard)::value>(red[q], red[C + q], u[e], z[e], (double)f4_get(a4, q));
                    }
                };
                if (eps > 0.0) pass(std::false_type{});
                else pass(std::true_type{});
                block_reduce<NT>(red, sred, buf);
                fresh = true;
            }
            double x = (double)xs[tt];
            const double base = ssum[tt];
            double g = (base + alpha * x + a.beta) - red[cc];
            double h = alpha + red[C + cc];
            int inner = 0;
            bool active = enters(g, x, eg);
            bool moved = false;
            while (active) {  // block-uniform
                bool again = false;
                const double delta = newton_step(g, h, x, inner, active, again, a, cnt);
                if (delta != 0.0) {
                    moved = true;
#pragma unroll
                    for (int e = 0; e < NPL; ++e) {
                        const double av = (double)reinterpret_cast<const float *>(Ach + e * NT)[cc];
                        if (av != 0.0) entry_update(delta, av, v[e], eps, t[e], u[e], z[e]);
                    }
                }
                if (again) {
                    double g2 = 0.0, h2 = 0.0;
#pragma unroll
                    for (int e = 0; e < NPL; ++e) {
                        const double av = (double)reinterpret_cast<const float *>(Ach + e * NT)[cc];
                        if (av != 0.0) {
                            g2 = fma(u[e], av, g2);
                            h2 = fma(z[e] * av, av, h2);
                        }
                    }
                    block_reduce2<NT>(g2, h2, sred, buf);
                    g = (base + alpha * x + a.beta) - g2;
                    h = alpha + h2;
                    active = enters(g, x, eg);
                }
            }
            if (moved) fresh = false;
            if (tid == 0) xo[tt] = (float)x;
        });
    }
    cp_wait<0>();
    __syncthreads();
    for (int k = tid; k < r; k += NT) moving[j * rp + a.perm_out[k]] = xo[k];
#pragma unroll
    for (int e = 0; e < NPL; ++e)
        if (off[e] >= 0) a.t_out[lo + tid + e * NT] = t[e];
    if (tid == 0 && a.stats) {
        if (cnt.n_inner) atomicAdd(a.stats + KLNMF_STAT_INNER_ITERS, (unsigned long long)cnt.n_inner);
        if (cnt.n_cap) atomicAdd(a.stats + KLNMF_STAT_CAP_HITS, (unsigned long long)cnt.n_cap);
        if (cnt.n_deg) atomicAdd(a.stats + KLNMF_STAT_DEGENERATE, (unsigned long long)cnt.n_deg);
        atomicAdd(a.stats + KLNMF_STAT_PASSES, 1ull);
    }
}

// ---------------------------------------------------------------------------
// Long subproblems (the W side's popular rows): one subproblem per thread-block
// CLUSTER of k CTAs (k = 1..16).  Each CTA owns a contiguous slice of the
// entries and keeps their state ON CHIP -- NR entries per thread in
// registers, NS in shared memory; only entries beyond the cluster's capacity
// spill to global memory (t_out / scratch).  At the start of every 4-coordinate
// chunk each thread cp.async-gathers the chunk of its resident entries into
// shared memory once; every pass and every move of that chunk then reads it
// from there (no re-gathers, no scattered scalar loads).  Partial sums are
// reduced warp -> CTA (shared memory) -> cluster (DSMEM, fixed CTA order), so
// every CTA sees identical (g, h) and runs the same Newton logic.
namespace cg = cooperative_groups;

constexpr int CL_NT = 512, CL_NR = 8, CL_NS = 4;
constexpr int CL_NE = CL_NR + CL_NS;  // resident entries per thread

struct ClusterRed {
    double wred[2][CL_NT / 32][NV];
    double cpart[2][NV];
    double tot[2][NV];
};

// Sum of NV values over the cluster; every thread of every CTA gets the same
// totals (warp transposed reduce, fixed-order CTA sum, fixed-order cluster
// sum).  Double-buffered: one cluster barrier and two CTA barriers per call.
__device__ __forceinline__ void cluster_reduce(double (&v)[NV], ClusterRed &R, int &buf, cg::cluster_group &cl,
                                               int k) {
    constexpr int NW = CL_NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    TReduce<32>::run(v, lane);
    if ((lane & 3) == 0) R.wred[buf][w][lane >> 2] = v[0];
    __syncthreads();
    if (w == 0 && lane < NV) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) s += R.wred[buf][q][lane];
        R.cpart[buf][lane] = s;
    }
    if (k > 1) {
        cl.sync();
        if (w == 0 && lane < NV) {
            double s = 0.0;
            for (int c = 0; c < k; ++c) s += cl.map_shared_rank(&R.cpart[buf][0], c)[lane];
            R.tot[buf][lane] = s;
        }
    } else if (w == 0 && lane < NV) {
        R.tot[buf][lane] = R.cpart[buf][lane];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = R.tot[buf][i];
    buf ^= 1;
}

// One subproblem's slice on one CTA: rank cq of the k CTAs sharing it.
// `reduce(v)` sums NV values over the k CTAs (identical result in all).
template <int NT, int NR, int NS, typename ReduceFn>
__device__ __forceinline__ void solve_slice(const klnmf_solve_args_t &a, int64_t slot, int cq, int k,
                                            ReduceFn &&reduce, unsigned char *smem_raw, const double *ssum) {
    static_assert(NT == CL_NT && NR + NS == CL_NE, "buffers are sized for CL_NT / CL_NE");
    float4 *cache = reinterpret_cast<float4 *>(smem_raw);    // [NR+NS][NT]: current chunk
    double *Ts = reinterpret_cast<double *>(cache + (NR + NS) * NT);  // [NS][NT]
    double *Us = Ts + NS * NT;
    double *Zs = Us + NS * NT;
    int2 *VO = reinterpret_cast<int2 *>(Zs + NS * NT);    // (float bits of v, row offset)
    float *xs = reinterpret_cast<float *>(VO + NS * NT);  // [2][rps]: input row, result
    float *xo = xs + (a.rp | 1);

    const int tid = threadIdx.x;
    const int rp = a.rp, r = a.r;
    const float *fixed = static_cast<const float *>(a.fixed);
    float *moving = static_cast<float *>(a.moving);
    const float *val = static_cast<const float *>(a.side.val);
    const int64_t j = a.items[slot];
    const int64_t lo = a.side.ptr[j];
    const int64_t s = a.side.ptr[j + 1] - lo;
    const int64_t per = (s + k - 1) / k;
    const int64_t c0 = min(s, (int64_t)cq * per);
    const int64_t cn = min(s, c0 + per) - c0;  // entries of this CTA
    const int64_t base = lo + c0;              // global entry index of local entry 0
    const double eps = a.eps_div, eg = a.eps_grad, alpha = a.alpha;
    double *Tg = a.t_out + base;  // spilled entries: t in t_out, u/z in scratch
    double *Ug = a.scratch + base;
    double *Zg = a.scratch + a.side.nnz + base;

    for (int kk = tid; kk < r; kk += NT) xs[kk] = moving[j * rp + a.perm_in[kk]];

    double t[NR], u[NR], z[NR];
    float v[NR];
    int off[NR];
#pragma unroll
    for (int e = 0; e < NR; ++e) {
        const int64_t i = tid + (int64_t)e * NT;
        if (i < cn) {
            const int64_t g = base + i;
            off[e] = a.side.idx[g] * rp;
            v[e] = val[g];
            const double tq = a.t_in[a.tmap ? (int64_t)a.tmap[g] : g];
            t[e] = tq;
            const double ri = fast_rcp(tq + eps);
            u[e] = (double)v[e] * ri;
            z[e] = u[e] * ri;
        } else {
            off[e] = -1;
            v[e] = 0.f;
            t[e] = u[e] = z[e] = 0.0;
        }
    }
#pragma unroll
    for (int e = 0; e < NS; ++e) {
        const int64_t i = tid + (int64_t)(NR + e) * NT;
        const int si = e * NT + tid;
        if (i < cn) {
            const int64_t g = base + i;
            const float vv = val[g];
            VO[si] = make_int2(__float_as_int(vv), a.side.idx[g] * rp);
            const double tq = a.t_in[a.tmap ? (int64_t)a.tmap[g] : g];
            const double ri = fast_rcp(tq + eps);
            Ts[si] = tq;
            Us[si] = (double)vv * ri;
            Zs[si] = Us[si] * ri;
        } else {
            VO[si] = make_int2(0, -1);
            Ts[si] = Us[si] = Zs[si] = 0.0;
        }
    }
    int offs[NS];  // row offsets of the shared-memory entries (for the gathers)
#pragma unroll
    for (int e = 0; e < NS; ++e) offs[e] = VO[e * NT + tid].y;
    const int64_t spill0 = (int64_t)(NR + NS) * NT;  // first spilled local entry
    for (int64_t i = spill0 + tid; i < cn; i += NT) {
        const int64_t g = base + i;
        const double tq = a.t_in[a.tmap ? (int64_t)a.tmap[g] : g];
        const double ri = fast_rcp(tq + eps);
        Tg[i] = tq;
        Ug[i] = (double)val[g] * ri;
        Zg[i] = Ug[i] * ri;
    }
    __syncthreads();

    Counters cnt;
    const int nchunks = (r + C - 1) / C;
    for (int ch = 0; ch < nchunks; ++ch) {
        // gather this chunk of every resident entry once (own slots only)
#pragma unroll
        for (int e = 0; e < NR; ++e)
            cp_async16(&cache[e * NT + tid], off[e] >= 0 ? fixed + off[e] + ch * C : fixed, off[e] >= 0);
#pragma unroll
        for (int e = 0; e < NS; ++e)
            cp_async16(&cache[(NR + e) * NT + tid], offs[e] >= 0 ? fixed + offs[e] + ch * C : fixed, offs[e] >= 0);
        cp_commit();
        cp_wait<0>();

        double red[NV];
        bool fresh = false;
        static_for<0, C>([&](auto cc_c) {  // compile-time coordinate index
            constexpr int cc = decltype(cc_c)::value;
            const int tt = ch * C + cc;
            if (tt >= r) return;
            if (!fresh) {
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
                auto pass = [&](auto guard) {
                    auto acc = [&](const float4 &a4, double uu, double zz) {
#pragma unroll
                        for (int qq = cc; qq < C; ++qq)
                            accum<decltype(guard)::value>(red[qq], red[C + qq], uu, zz, (double)f4_get(a4, qq));
                    };
#pragma unroll
                    for (int e = 0; e < NR; ++e) acc(cache[e * NT + tid], u[e], z[e]);  // absent: u = z = 0
#pragma unroll
                    for (int e = 0; e < NS; ++e) acc(cache[(NR + e) * NT + tid], Us[e * NT + tid], Zs[e * NT + tid]);
                    for (int64_t i = spill0 + tid; i < cn; i += NT)
                        acc(ldg_f4(fixed + (int64_t)a.side.idx[base + i] * rp + ch * C), Ug[i], Zg[i]);
                };
                if (eps > 0.0) pass(std::false_type{});
                else pass(std::true_type{});
                reduce(red);
                fresh = true;
            }
            double x = (double)xs[tt];
            const double sa = ssum[tt];
            double g = (sa + alpha * x + a.beta) - red[cc];
            double h = alpha + red[C + cc];
            int inner = 0;
            bool active = enters(g, x, eg);
            bool moved = false;
            while (active) {  // uniform over the cluster
                bool again = false;
                const double delta = newton_step(g, h, x, inner, active, again, a, cnt);
                double ev[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i) ev[i] = 0.0;
                // apply the move (and, if the loop continues, re-evaluate this coordinate)
                if (delta != 0.0 || again) {
                    if (delta != 0.0) moved = true;
#pragma unroll
                    for (int e = 0; e < NR; ++e) {
                        const double av = (double)f4_get(cache[e * NT + tid], cc);
                        if (off[e] >= 0 && av != 0.0) {
                            if (delta != 0.0) entry_update(delta, av, v[e], eps, t[e], u[e], z[e]);
                            ev[0] = fma(u[e], av, ev[0]);
                            ev[1] = fma(z[e] * av, av, ev[1]);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < NS; ++e) {
                        const int si = e * NT + tid;
                        const double av = (double)f4_get(cache[(NR + e) * NT + tid], cc);
                        if (offs[e] >= 0 && av != 0.0) {
                            double tn = Ts[si], uu = Us[si], zz = Zs[si];
                            if (delta != 0.0) {
                                entry_update(delta, av, __int_as_float(VO[si].x), eps, tn, uu, zz);
                                Ts[si] = tn;
                                Us[si] = uu;
                                Zs[si] = zz;
                            }
                            ev[0] = fma(uu, av, ev[0]);
                            ev[1] = fma(zz * av, av, ev[1]);
                        }
                    }
                    for (int64_t i = spill0 + tid; i < cn; i += NT) {
                        const double av = (double)__ldg(fixed + (int64_t)a.side.idx[base + i] * rp + tt);
                        if (av != 0.0) {
                            double tn = Tg[i], uu = Ug[i], zz = Zg[i];
                            if (delta != 0.0) {
                                entry_update(delta, av, val[base + i], eps, tn, uu, zz);
                                Tg[i] = tn;
                                Ug[i] = uu;
                                Zg[i] = zz;
                            }
                            ev[0] = fma(uu, av, ev[0]);
                            ev[1] = fma(zz * av, av, ev[1]);
                        }
                    }
                }
                if (again) {
                    reduce(ev);
                    g = (sa + alpha * x + a.beta) - ev[0];
                    h = alpha + ev[1];
                    active = enters(g, x, eg);  // _kernels.py:78
                }
            }
            if (moved) fresh = false;
            if (tid == 0) xo[tt] = (float)x;
        });
    }
    __syncthreads();
    if (cq == 0)
        for (int kk = tid; kk < r; kk += NT) moving[j * rp + a.perm_out[kk]] = xo[kk];
#pragma unroll
    for (int e = 0; e < NR; ++e)
        if (off[e] >= 0) a.t_out[base + tid + (int64_t)e * NT] = t[e];
#pragma unroll
    for (int e = 0; e < NS; ++e) {
        const int si = e * NT + tid;
        if (offs[e] >= 0) a.t_out[base + tid + (int64_t)(NR + e) * NT] = Ts[si];
    }
    if (cq == 0 && tid == 0 && a.stats) {
        if (cnt.n_inner) atomicAdd(a.stats + KLNMF_STAT_INNER_ITERS, (unsigned long long)cnt.n_inner);
        if (cnt.n_cap) atomicAdd(a.stats + KLNMF_STAT_CAP_HITS, (unsigned long long)cnt.n_cap);
        if (cnt.n_deg) atomicAdd(a.stats + KLNMF_STAT_DEGENERATE, (unsigned long long)cnt.n_deg);
        atomicAdd(a.stats + KLNMF_STAT_PASSES, 1ull);
    }
}

template <int NT, int NR, int NS>
__global__ void __launch_bounds__(NT, 1) solve_cluster_kernel(const klnmf_solve_args_t a) {
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.num_blocks();
    const int cq = (int)cl.block_rank();
    const int64_t slot = blockIdx.x / k;
    if (slot >= a.n_items) return;  // uniform over the cluster
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ ClusterRed R;
    __shared__ double ssum[KMAX_RP];
    for (int kk = threadIdx.x; kk < a.r; kk += NT) ssum[kk] = a.sum_pos[kk];
    int buf = 0;
    solve_slice<NT, NR, NS>(
        a, slot, cq, k, [&](double (&v)[NV]) { cluster_reduce(v, R, buf, cl, k); }, smem_raw, ssum);
    if (k > 1) cl.sync();  // peers may still read this CTA's shared memory
}

// ---------------------------------------------------------------------------
// Rows too long for one 16-CTA cluster: a persistent COOPERATIVE kernel (all
// CTAs co-resident, one per SM).  A host-built schedule packs the rows into
// waves; a row spans as many CTAs as its entries need, so all per-entry state
// stays on chip.  The per-pass reduction of a row group goes through global
// memory: each CTA publishes its partial sums, bumps the group's monotonic
// counter and waits until all G members of the round have arrived.  Waits
// only point to rows of the same or an earlier wave, all CTAs are resident,
// so the schedule cannot deadlock.
struct CoopGroup {
    double *slots;       // [2][G][NV] partials, double-buffered by round parity
    unsigned *counter;   // arrivals, G per round
    int G, rank;
    unsigned round;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void coop_reduce(double (&v)[NV], ClusterRed &R, int &buf, CoopGroup &g) {
    constexpr int NW = CL_NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    TReduce<32>::run(v, lane);
    if ((lane & 3) == 0) R.wred[buf][w][lane >> 2] = v[0];
    __syncthreads();
    if (w == 0) {
        double part = 0.0;
        if (lane < NV) {
#pragma unroll
            for (int q = 0; q < NW; ++q) part += R.wred[buf][q][lane];
        }
        if (g.G > 1) {
            double *cur = g.slots + (size_t)(g.round & 1) * g.G * NV;
            if (lane < NV) {
                __stcg(cur + (size_t)g.rank * NV + lane, part);
                __threadfence();
            }
            __syncwarp();
            const unsigned target = (unsigned)g.G * (g.round + 1);
            if (lane == 0) {
                atomicAdd(g.counter, 1u);
                while (ld_acquire(g.counter) < target) __nanosleep(64);
            }
            __syncwarp();
            if (lane < NV) {
                (void)ld_acquire(g.counter);
                double s = 0.0;
                for (int c = 0; c < g.G; ++c) s += __ldcg(cur + (size_t)c * NV + lane);
                R.tot[buf][lane] = s;
            }
        } else if (lane < NV) {
            R.tot[buf][lane] = part;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = R.tot[buf][i];
    buf ^= 1;
    ++g.round;
}

// schedule: [n_waves][gridDim.x] int4 (item slot or -1, rank, G, group id);
// sync: per group, a 128-byte counter line then 2*CL_MAXG*NV doubles.
constexpr int CL_MAXG = 256;
constexpr size_t COOP_GROUP_BYTES = 128 + 2 * CL_MAXG * NV * sizeof(double);

template <int NT, int NR, int NS>
__global__ void __launch_bounds__(NT, 1) solve_coop_kernel(const klnmf_solve_args_t a, const int4 *schedule,
                                                           int n_waves, unsigned char *sync) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ ClusterRed R;
    __shared__ double ssum[KMAX_RP];
    for (int kk = threadIdx.x; kk < a.r; kk += NT) ssum[kk] = a.sum_pos[kk];
    int buf = 0;
    for (int wv = 0; wv < n_waves; ++wv) {
        const int4 job = schedule[(size_t)wv * gridDim.x + blockIdx.x];
        if (job.x < 0) continue;
        unsigned char *gb = sync + (size_t)job.w * COOP_GROUP_BYTES;
        CoopGroup g{reinterpret_cast<double *>(gb + 128), reinterpret_cast<unsigned *>(gb), job.z, job.y, 0u};
        __syncthreads();  // shared buffers of the previous row are no longer read
        solve_slice<NT, NR, NS>(
            a, job.x, job.y, job.z, [&](double (&v)[NV]) { coop_reduce(v, R, buf, g); }, smem_raw, ssum);
    }
}

struct FastKernel {
    int lanes, npl, nt;
    int64_t capacity;  // -1 = unbounded
    void (*fn)(const klnmf_solve_args_t);
    int gpb;           // subproblems per block
    int ring_entries;  // float4 ring slots per thread and stage (NPL)
    int cluster;       // CTAs per subproblem (cluster kernel), 0 = plain launch
};

#define WK(L, NPL) {L, NPL, 128, (int64_t)(L) * (NPL), solve_warp_kernel<L, NPL>, 128 / (L), NPL, 0}
#define BK(NT, NPL) {NT, NPL, NT, (int64_t)(NT) * (NPL), solve_block_kernel<NT, NPL>, 1, NPL, 0}
#define CK(K, CAP)                                                                                        \
    {CL_NT * (K), CL_NR + CL_NS, CL_NT, (CAP), solve_cluster_kernel<CL_NT, CL_NR, CL_NS>, 1, 0, (K)}
const FastKernel kFast[] = {
    WK(1, 4),  WK(2, 4),  WK(4, 4),   WK(8, 4),   WK(8, 8),   WK(16, 8),
    WK(32, 8), BK(64, 8), BK(128, 8), BK(256, 8), BK(512, 8),
    CK(1, (int64_t)CL_NT * (CL_NR + CL_NS)),     CK(2, 2ll * CL_NT * (CL_NR + CL_NS)),
    CK(4, 4ll * CL_NT * (CL_NR + CL_NS)),        CK(8, 8ll * CL_NT * (CL_NR + CL_NS)),
    CK(16, 16ll * CL_NT * (CL_NR + CL_NS)),
    // unbounded: the cooperative long-row kernel (klnmf_solve_coop, schedule built by the caller)
    {CL_NT, CL_NR + CL_NS, CL_NT, -1, nullptr, 1, 0, -1},
};
#undef WK
#undef BK
#undef CK
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
    if (args->rp > KMAX_RP) return set_error_msg(1, "klnmf_solve_fast: rank above 256 is not supported in fp32 mode");
    const FastKernel &k = kFast[kernel_id];
    if (k.cluster < 0) return set_error_msg(1, "klnmf_solve_fast: the long-row bucket runs through klnmf_solve_coop");
    const size_t xrow = 2 * sizeof(float) * (size_t)k.gpb * (size_t)(args->rp | 1) + 16;
    if (k.cluster > 0) {
        if (args->scratch == nullptr)
            return set_error_msg(1, "klnmf_solve_fast: the cluster kernel needs 2*nnz doubles of scratch");
        const size_t smem = (size_t)CL_NE * CL_NT * sizeof(float4) +
                            (size_t)CL_NS * CL_NT * (3 * sizeof(double) + sizeof(int2)) + xrow;
        KLNMF_CHECK(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (k.cluster > 8)
            KLNMF_CHECK(cudaFuncSetAttribute(k.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(args->n_items * k.cluster), 1, 1);
        cfg.blockDim = dim3((unsigned)k.nt, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = as_stream(stream);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)k.cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        KLNMF_CHECK(cudaLaunchKernelEx(&cfg, k.fn, *args));
        return 0;
    }
    const int64_t blocks = (args->n_items + k.gpb - 1) / k.gpb;
    const size_t ring = sizeof(float4) * (size_t)STAGES * (size_t)k.ring_entries * (size_t)k.nt;
    const size_t smem = ring + xrow;
    if (smem > 48 * 1024) {
        KLNMF_CHECK(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k.fn<<<(unsigned)blocks, k.nt, smem, as_stream(stream)>>>(*args);
    KLNMF_CHECK_LAUNCH("klnmf_solve_fast");
    return 0;
}

namespace klnmf {
namespace {
inline size_t coop_smem(int rp) {
    return (size_t)CL_NE * CL_NT * sizeof(float4) + (size_t)CL_NS * CL_NT * (3 * sizeof(double) + sizeof(int2)) +
           2 * sizeof(float) * (size_t)(rp | 1) + 16;
}
}  // namespace
}  // namespace klnmf

extern "C" int klnmf_coop_info(int32_t rp, int64_t *entries_per_cta, int32_t *n_ctas, int64_t *sync_bytes_per_group) {
    auto fn = solve_coop_kernel<CL_NT, CL_NR, CL_NS>;
    const size_t smem = coop_smem(rp);
    KLNMF_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, per_sm = 0;
    KLNMF_CHECK(cudaGetDevice(&dev));
    KLNMF_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    KLNMF_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, CL_NT, smem));
    *entries_per_cta = (int64_t)CL_NT * CL_NE;
    *n_ctas = sms * per_sm < CL_MAXG ? sms * per_sm : CL_MAXG;
    *sync_bytes_per_group = (int64_t)COOP_GROUP_BYTES;
    return 0;
}

extern "C" int klnmf_solve_coop(const klnmf_solve_args_t *args, const void *schedule, int32_t n_waves,
                                int32_t n_ctas, void *sync, int64_t n_groups, void *stream) {
    if (n_waves <= 0 || args->n_items <= 0) return 0;
    if (args->rp > KMAX_RP) return set_error_msg(1, "klnmf_solve_coop: rank above 256 is not supported");
    if (args->scratch == nullptr) return set_error_msg(1, "klnmf_solve_coop: needs 2*nnz doubles of scratch");
    cudaStream_t st = as_stream(stream);
    auto fn = solve_coop_kernel<CL_NT, CL_NR, CL_NS>;
    const size_t smem = coop_smem(args->rp);
    KLNMF_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    KLNMF_CHECK(cudaMemsetAsync(sync, 0, (size_t)n_groups * COOP_GROUP_BYTES, st));
    klnmf_solve_args_t a = *args;
    const int4 *sched = static_cast<const int4 *>(schedule);
    unsigned char *sy = static_cast<unsigned char *>(sync);
    int nw = n_waves;
    void *kargs[] = {&a, &sched, &nw, &sy};
    KLNMF_CHECK(cudaLaunchCooperativeKernel((const void *)fn, dim3((unsigned)n_ctas), dim3(CL_NT), kargs, smem, st));
    return 0;
}
