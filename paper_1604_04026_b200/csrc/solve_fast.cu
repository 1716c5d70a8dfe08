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
#include <cstdio>

#include "common.cuh"

namespace klnmf {
namespace {

constexpr int C = 4;       // coordinates per batch (16 B of fp32 per entry)
constexpr int NV = 2 * C;  // reduced values per pass: g partials then h partials
constexpr int STAGES = 3;  // cp.async ring depth

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

__device__ __forceinline__ void entry_update(double delta, double av, float v, double eps, double &t, double &u,
                                             double &z) {
    double tn = fma(delta, av, t);
    if (tn < 0.0) tn = 0.0;
    t = tn;
    const double ri = 1.0 / (tn + eps);
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
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
            const int tt = ch * C + cc;
            if (tt >= r) break;  // uniform
            if (__any_sync(FULL_MASK, !fresh)) {
                // pass: partial sums of coordinates cc..C-1 on the current t
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
#pragma unroll
                for (int e = 0; e < NPL; ++e) {
                    const float4 a4 = Ach[e * NT];
#pragma unroll
                    for (int q = cc; q < C; ++q) {
                        const double av = (double)f4_get(a4, q);
                        if (av != 0.0) {
                            red[q] = fma(u[e], av, red[q]);
                            red[C + q] = fma(z[e] * av, av, red[C + q]);
                        }
                    }
                }
                TReduce<L>::run(red, gl);
                fresh = true;
            }
            const double gp = fetch<L>(red, cc);
            const double hp = fetch<L>(red, C + cc);
            double x = (double)xs[tt];
            const double base = a.sum_pos[tt];
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
        }
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
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
            const int tt = ch * C + cc;
            if (tt >= r) break;
            if (!fresh) {
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
#pragma unroll
                for (int e = 0; e < NPL; ++e) {
                    const float4 a4 = Ach[e * NT];
#pragma unroll
                    for (int q = cc; q < C; ++q) {
                        const double av = (double)f4_get(a4, q);
                        if (av != 0.0) {
                            red[q] = fma(u[e], av, red[q]);
                            red[C + q] = fma(z[e] * av, av, red[C + q]);
                        }
                    }
                }
                block_reduce<NT>(red, sred, buf);
                fresh = true;
            }
            double x = (double)xs[tt];
            const double base = a.sum_pos[tt];
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
        }
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
// Any-size subproblem, one block each; per-entry t/u/z in global memory (t in
// t_out, u and z in scratch), each thread owning entries p = tid mod NT.  Same
// batched scheme: a pass streams every entry once (its 16-byte chunk of the
// fixed row and its u/z); the final move of the previous coordinate is
// applied inside the next pass.
template <int NT>
__global__ void __launch_bounds__(NT) solve_stream_kernel(const klnmf_solve_args_t a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *xs = reinterpret_cast<float *>(smem_raw);  // [2][rps]: input row, result
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
    const int64_t s = a.side.ptr[j + 1] - lo;
    double *T = a.t_out + lo;
    double *U = a.scratch + lo;
    double *Z = a.scratch + a.side.nnz + lo;
    const int32_t *vi = a.side.idx + lo;
    const float *vv = val + lo;
    const double eps = a.eps_div, eg = a.eps_grad, alpha = a.alpha;

    for (int k = tid; k < r; k += NT) xs[k] = moving[j * rp + a.perm_in[k]];
    for (int64_t p = tid; p < s; p += NT) {
        const int64_t q = lo + p;
        const double tq = a.t_in[a.tmap ? (int64_t)a.tmap[q] : q];
        T[p] = tq;
        const double ri = 1.0 / (tq + eps);
        const double uu = (double)vv[p] * ri;
        U[p] = uu;
        Z[p] = uu * ri;
    }
    __syncthreads();

    Counters cnt;
    int buf = 0;
    const int nchunks = (r + C - 1) / C;
    for (int ch = 0; ch < nchunks; ++ch) {
        double red[NV];
        bool fresh = false;
        double pend_delta = 0.0;  // final move of the previous coordinate, not yet applied
        int pend_q = 0;
        for (int cc = 0; cc < C; ++cc) {
            const int tt = ch * C + cc;
            if (tt >= r) break;
            if (!fresh) {
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
                for (int64_t p = tid; p < s; p += NT) {
                    const float4 A4 = ldg_f4(fixed + (int64_t)vi[p] * rp + ch * C);
                    double uu = U[p], zz = Z[p];
                    if (pend_delta != 0.0) {
                        const double av = (double)f4_get(A4, pend_q);
                        if (av != 0.0) {
                            double tn = T[p];
                            entry_update(pend_delta, av, vv[p], eps, tn, uu, zz);
                            T[p] = tn;
                            U[p] = uu;
                            Z[p] = zz;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < C; ++q) {
                        if (q >= cc) {
                            const double av = (double)f4_get(A4, q);
                            if (av != 0.0) {
                                red[q] = fma(uu, av, red[q]);
                                red[C + q] = fma(zz * av, av, red[C + q]);
                            }
                        }
                    }
                }
                pend_delta = 0.0;
                block_reduce<NT>(red, sred, buf);
                fresh = true;
            }
            double x = (double)xs[tt];
            const double base = a.sum_pos[tt];
            double g = (base + alpha * x + a.beta) - red[cc];
            double h = alpha + red[C + cc];
            int inner = 0;
            bool active = enters(g, x, eg);
            bool moved = false;
            while (active) {
                bool again = false;
                const double delta = newton_step(g, h, x, inner, active, again, a, cnt);
                if (delta != 0.0) moved = true;
                if (again) {
                    // apply this step now and re-evaluate the same coordinate
                    double g2 = 0.0, h2 = 0.0;
                    for (int64_t p = tid; p < s; p += NT) {
                        const double av = (double)__ldg(fixed + (int64_t)vi[p] * rp + tt);
                        double uu = U[p], zz = Z[p];
                        if (av != 0.0) {
                            if (delta != 0.0) {
                                double tn = T[p];
                                entry_update(delta, av, vv[p], eps, tn, uu, zz);
                                T[p] = tn;
                                U[p] = uu;
                                Z[p] = zz;
                            }
                            g2 = fma(uu, av, g2);
                            h2 = fma(zz * av, av, h2);
                        }
                    }
                    block_reduce2<NT>(g2, h2, sred, buf);
                    g = (base + alpha * x + a.beta) - g2;
                    h = alpha + h2;
                    active = enters(g, x, eg);
                } else if (delta != 0.0) {
                    // the loop ends on this step: fuse its update into the next pass
                    pend_delta = delta;
                    pend_q = cc;
                }
            }
            if (moved) fresh = false;
            if (tid == 0) xo[tt] = (float)x;
        }
        if (pend_delta != 0.0) {
            for (int64_t p = tid; p < s; p += NT) {
                const double av = (double)__ldg(fixed + (int64_t)vi[p] * rp + ch * C + pend_q);
                if (av != 0.0) {
                    double tn = T[p], uu = U[p], zz = Z[p];
                    entry_update(pend_delta, av, vv[p], eps, tn, uu, zz);
                    T[p] = tn;
                    U[p] = uu;
                    Z[p] = zz;
                }
            }
        }
    }
    __syncthreads();
    for (int k = tid; k < r; k += NT) moving[j * rp + a.perm_out[k]] = xo[k];
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
    int gpb;           // subproblems per block
    int ring_entries;  // float4 ring slots per thread and stage (NPL)
};

#define WK(L, NPL) {L, NPL, 128, (int64_t)(L) * (NPL), solve_warp_kernel<L, NPL>, 128 / (L), NPL}
#define BK(NT, NPL) {NT, NPL, NT, (int64_t)(NT) * (NPL), solve_block_kernel<NT, NPL>, 1, NPL}
const FastKernel kFast[] = {
    WK(1, 4),  WK(2, 4),   WK(4, 4),   WK(8, 4),   WK(8, 8),   WK(16, 8),
    WK(32, 8), BK(64, 8),  BK(128, 8), BK(256, 8), BK(512, 8),
    {1024, 0, 1024, -1, solve_stream_kernel<1024>, 1, 0},
};
#undef WK
#undef BK
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
    const size_t ring = sizeof(float4) * (size_t)STAGES * (size_t)k.ring_entries * (size_t)k.nt;
    const size_t smem = ring + 2 * sizeof(float) * (size_t)k.gpb * (size_t)(args->rp | 1) + 16;
    if (smem > 48 * 1024) {
        KLNMF_CHECK(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k.fn<<<(unsigned)blocks, k.nt, smem, as_stream(stream)>>>(*args);
    KLNMF_CHECK_LAUNCH("klnmf_solve_fast");
    return 0;
}
