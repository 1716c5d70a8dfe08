// fp32-storage / fp64-arithmetic subproblem solver (throughput mode).
//
// Algorithm: the reference's solve_column with max_passes = 1
// (_kernels.py:53-120, driven by sweep_range :123-144), restated for the
// device:
//   * the maintained product t is kept on the column support S only and is
//     CARRIED between half-steps (t at entry (i,j) is <W_i, F_j> for both
//     sides), so no subproblem recomputes it from the fixed factor;
//   * per entry the kernel keeps only u = v/(t+eps) and vi = 1/v (16 bytes):
//     _grad_hess (_kernels.py:24-36) becomes g = sum_a + alpha*x + beta -
//     sum(u*a), h = alpha + sum(z*a*a) with z = u/(t+eps) = u*u*vi, and a move
//     t' = t + delta*a (clamped at 0, _kernels.py:105-106) becomes
//     u' = u / (1 + delta*a*u*vi); t = 1/(u*vi) - eps is written back once at
//     the end.  The compact state is what sets how many entries stay on chip;
//   * every Newton step rounds the coordinate to fp32 (the storage type), so
//     t stays consistent with the stored factors;
//   * coordinates are visited in storage order (factors are stored in the
//     iteration's visit order), 4 at a time: one pass over the subproblem's
//     entries produces the partial (g, h) sums of the remaining coordinates
//     of the chunk ("speculative" batch), one transposed reduction combines
//     them, and the coordinates are then consumed in order.  A coordinate that
//     moves changes t, so the rest of the chunk is re-evaluated: every
//     gradient is computed on exactly the t the sequential reference sees;
//   * the gathered fixed-factor rows are staged in shared memory once per
//     chunk (cp.async; each thread reads only the copies it issued);
//   * code size matters: the coordinate loop is a runtime loop whose chunk
//     components and reduced sums are read from shared memory by index, so
//     the Newton/update code exists once per kernel and stays in the
//     instruction cache.
// eps_div > 0 is required (u is finite); the exact mode covers eps_div = 0.
//
// Kernels (one launch per nnz bucket, largest subproblems first):
//   solve_warp_kernel<L, NPL>    L <= 32 lanes per subproblem, 32/L
//       subproblems per warp in lock-step, NPL entries per lane in registers.
//   solve_block_kernel<NT, NPL>  one subproblem per block of NT threads.
//   solve_cluster_kernel         one subproblem per thread-block cluster of
//       k <= 16 CTAs (state in registers + shared memory, DSMEM reductions).
//   solve_coop_kernel            persistent cooperative kernel for rows longer
//       than a cluster: G CTAs per row, reductions through global memory.
#include <cooperative_groups.h>

#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace klnmf {
namespace {

constexpr int C = 4;          // coordinates per chunk (16 B of fp32 per entry)
constexpr int NV = 2 * C;     // reduced values per pass: g partials then h partials
// cp.async ring depth of the warp/block kernels: 3 stages; 2 when a thread
// holds many entries (the ring is the shared-memory budget that sets how many
// subproblems are resident per SM)
constexpr int ring_stages(int npl) { return npl >= 10 ? 2 : 3; }
constexpr int KMAX_RP = 256;  // largest padded rank of the fp32 kernels (row sums staged in smem)

struct Counters {
    unsigned n_inner = 0, n_cap = 0, n_deg = 0;
};

// Scalar parameters of the Newton loop, hoisted out of the argument struct.
struct Params {
    double alpha, beta, eps_grad, eps_x, eps_div;
    int inner_cap;
    __device__ explicit Params(const klnmf_solve_args_t &a)
        : alpha(a.alpha), beta(a.beta), eps_grad(a.eps_grad), eps_x(a.eps_x), eps_div(a.eps_div),
          inner_cap((int)a.inner_cap) {}
};

__device__ __forceinline__ bool enters(double g, double x, double eg) {
    return (g < -eg) || (fabs(g) > eg && x > eg);  // _kernels.py:78
}

// fp32 -> fp64 of a stored factor value (non-negative and finite, DenseFactor
// validation sparse.py:184; subnormals are flushed to zero at every store).
__device__ __forceinline__ double widen(float f) { return (double)f; }

// Rounds a non-negative coordinate to its fp32 storage value (subnormals to 0).
__device__ __forceinline__ double round_store(double x) {
    const float f = __double2float_rn(x);
    return f < 1.17549435e-38f ? 0.0 : (double)f;
}

// 1/x: MUFU approximation refined twice (full fp64 accuracy up to the last
// bit or so); x > 0 (eps_div > 0 keeps every t + eps positive).
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// One Newton step of the inner loop (_kernels.py:78-115), x rounded to fp32.
// Returns the applied delta; clears `active` when the loop ends, sets `again`
// when the loop needs a fresh gradient.
__device__ __forceinline__ double newton_step(double g, double h, double &x, int &inner, bool &active,
                                              bool &again, const Params &pm, Counters &cnt) {
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
    double target = x - g / h;  // IEEE division: once per step, and it keeps x's rounding exact
    if (target < 0.0) target = 0.0;
    const double xn = round_store(target);
    delta = xn - x;
    const double xo = x;
    x = xn;
    ++inner;
    ++cnt.n_inner;
    if (fabs(delta) < pm.eps_x * xo) {
        active = false;
    } else if (inner >= pm.inner_cap) {
        ++cnt.n_cap;
        active = false;
    } else {
        again = true;
    }
    return delta;
}

// Per-entry state (see the header): u = v/(t+eps), vi = 1/v.  Absent
// (padding) entries hold u = vi = 0 and contribute exactly 0.
__device__ __forceinline__ void entry_init(double t, float v, double eps, double &u, double &vi) {
    const double vd = (double)v;
    u = vd * fast_rcp(t + eps);
    vi = v > 0.f ? fast_rcp(vd) : 0.0;
}
// z = u/(t+eps), the curvature weight of the entry
__device__ __forceinline__ double entry_z(double u, double vi) { return (u * u) * vi; }
// the maintained product written back at the end of the half-step
__device__ __forceinline__ double entry_t(double u, double vi, double eps) {
    return fmax(1.0 / (u * vi) - eps, 0.0);
}
// Move of the visited coordinate by delta: t' + eps = (t + eps) * q with
// q = 1 + delta*a/(t+eps), so u' = u / q; the reference clamps t' at 0
// (_kernels.py:105-106): t' < 0 <=> q < eps/(t+eps), and then u' = v/eps.
// CLAMP = false when delta >= 0 (q >= 1: the clamp cannot fire).  Applied
// branch-free to every entry: a == 0 gives q = 1 and leaves u unchanged.
template <bool CLAMP>
__device__ __forceinline__ void entry_update(double delta, double a, double eps, double &u, double vi) {
    const double p = u * vi;                  // 1/(t+eps)
    const double q = fma(p, delta * a, 1.0);  // (t'+eps)/(t+eps)
    double un = u * fast_rcp(q);
    if (CLAMP && q < eps * p) un = fast_rcp(vi * eps);
#ifdef KLNMF_EXP_MOVEDP  // experiment: +4 DP ops per entry update, results unchanged
    un = (un + 0.0 * q) + 0.0 * p;
#endif
    u = un;
}

// Calls f(CLAMP) as a compile-time constant for a group-uniform move.
template <typename F>
__device__ __forceinline__ void with_clamp(bool any_negative, F &&f) {
    if (any_negative) f(std::true_type{});
    else f(std::false_type{});
}

// Adds one entry's contribution to a coordinate's (g, h) partial sums.  The
// reference skips a == 0 (_kernels.py:32); u and z are finite (eps_div > 0),
// so an a == 0 term adds exactly +0.0 and needs no test.
__device__ __forceinline__ void accum(double &g, double &h, double u, double z, double av) {
    g = fma(u, av, g);
    h = fma(z * av, av, h);
#ifdef KLNMF_EXP_PASSDP  // experiment: +2 DP ops per term, results unchanged (g finite)
    h = h + 0.0 * g;
#endif
}

// Partials of the chunk's coordinates CC..C-1 from one entry's 16-byte chunk
// (compile-time first coordinate: no predication, no conversions of the
// components already consumed).
template <int CC>
__device__ __forceinline__ void accum_from(double (&red)[NV], const float4 &a4, double u, double z) {
    if (CC <= 0) accum(red[0], red[C + 0], u, z, widen(a4.x));
    if (CC <= 1) accum(red[1], red[C + 1], u, z, widen(a4.y));
    if (CC <= 2) accum(red[2], red[C + 2], u, z, widen(a4.z));
    accum(red[3], red[C + 3], u, z, widen(a4.w));
}
// runtime first coordinate (the rare spilled entries of the long-row kernels)
__device__ __forceinline__ void accum_chunk(double (&red)[NV], const float4 &a4, double u, double z, int cc) {
    if (cc <= 0) accum(red[0], red[C + 0], u, z, widen(a4.x));
    if (cc <= 1) accum(red[1], red[C + 1], u, z, widen(a4.y));
    if (cc <= 2) accum(red[2], red[C + 2], u, z, widen(a4.z));
    accum(red[3], red[C + 3], u, z, widen(a4.w));
}

// Calls f(std::integral_constant<int, cc>) for a runtime cc in [0, C).
template <typename F>
__device__ __forceinline__ void with_cc(int cc, F &&f) {
    switch (cc) {
        case 0: f(std::integral_constant<int, 0>{}); break;
        case 1: f(std::integral_constant<int, 1>{}); break;
        case 2: f(std::integral_constant<int, 2>{}); break;
        default: f(std::integral_constant<int, 3>{}); break;
    }
}

__device__ __forceinline__ void cp_async16(unsigned smem_addr, const void *gmem, bool pred) {
    const int n = pred ? 16 : 0;  // zero-fill when the entry does not exist
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ float comp(const float4 *p, int c) { return reinterpret_cast<const float *>(p)[c]; }

// xs[k] = moving row j at visit position k, for k = first, first + step, ...
// (pin: the visit-order map staged in shared memory).  Four loads are issued
// before their stores, so a subproblem's start costs one load latency, not
// one per position.
__device__ __forceinline__ void load_row(float *xs, const float *row, const int *pin, int r, int first, int step,
                                         bool valid, float *xo = nullptr) {
    for (int k0 = first; k0 < r; k0 += 4 * step) {
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = k0 + i * step;
            v[i] = (valid && k < r) ? row[pin[k]] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (k0 + i * step < r) {
                xs[k0 + i * step] = v[i];
                if (xo) xo[k0 + i * step] = v[i];
            }
    }
}

// Transposed reduction of NV values across the L lanes of a group: after it
// each lane holds KEEP totals; lanes whose low (NL-HL) bits are zero hold
// distinct totals, indices (gl >> (NL-HL)) * KEEP + s.
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
    // write this group's totals to tot[NV]
    __device__ __forceinline__ static void store(const double (&v)[NV], int gl, double *tot) {
        constexpr int LOW = (1 << (NL - HL)) - 1;
        if ((gl & LOW) == 0) {
#pragma unroll
            for (int s = 0; s < KEEP; ++s) tot[(gl >> (NL - HL)) * KEEP + s] = v[s];
        }
    }
};

// Checked build (build.py variant "checked", tools/checked_run.py): device-side
// bounds checks and inter-CTA protocol assertions.  A violation is counted
// (and its first code recorded) instead of trapping, so the run continues
// and the host reads the counters after the workload (klnmf_debug_checks).
// Codes: 1 gather offset, 2 item id, 3 maintained-product index, 4 moving
// store, 5 product store, 6 cooperative slot overwritten before it was read
// (parity reuse violated), 7 arrival counter two rounds ahead, 8 spill
// record out of range, 9 non-finite / negative entry state, 10 cluster inbox
// round mismatch, 11 a chunk skipped by its mask holds a nonzero.
#ifdef KLNMF_CHECKED
__device__ unsigned long long g_check[2];
__device__ __forceinline__ void kcheck(bool ok, unsigned code) {
    if (!ok) {
        atomicAdd(&g_check[0], 1ull);
        atomicCAS(&g_check[1], 0ull, (unsigned long long)code);
    }
}
#else
__device__ __forceinline__ void kcheck(bool, unsigned) {}
#endif

// index of an entry's maintained product in t_in: the entry itself when the
// previous half-step scattered its products into this side's entry order
// (t_scatter), else through the entry map
__device__ __forceinline__ int64_t t_index(const klnmf_solve_args_t &a, int64_t q) {
    const int64_t i = (a.tmap && !a.t_scatter) ? (int64_t)a.tmap[q] : q;
    kcheck(i >= 0 && i < a.side.nnz, 3);
    return i;
}
// gather offset (row * rp) of an entry's fixed-factor row
__device__ __forceinline__ int gather_off(const klnmf_solve_args_t &a, int64_t q) {
    const int32_t row = a.side.idx[q];
    kcheck(row >= 0 && row < a.side.n_fix, 1);
    return row * a.rp;
}
__device__ __forceinline__ int64_t item_at(const klnmf_solve_args_t &a, int64_t slot) {
    const int64_t j = a.items[slot];
    kcheck(j >= 0 && j < a.side.n_mov, 2);
    return j;
}

// A result of this rank's subproblems (a moving-factor value, a maintained
// product): stored locally and, in a fused sharded exchange, into every
// peer's copy through its CUDA-IPC mapping (NVLink stores issued as the
// results are produced) -- no all-gather follows the half-step.
__device__ __forceinline__ void put_moving(const klnmf_solve_args_t &a, float *moving, int64_t i, float v) {
    kcheck(i >= 0 && i < a.side.n_mov * a.rp, 4);
    moving[i] = v;
    for (int p = 0; p < a.n_peers; ++p) static_cast<float *>(a.peer_moving[p])[i] = v;
}
// (t_scatter: the product of entry i lands at its position in the other
// side's entry order, where the next half-step reads it coalesced; the
// stores are fire-and-forget, the subproblem start no longer waits on a
// dependent gather through the map)
__device__ __forceinline__ void put_t(const klnmf_solve_args_t &a, int64_t i, double v) {
    kcheck(i >= 0 && i < a.side.nnz, 5);
    kcheck(v >= 0.0 && v < INFINITY, 9);
    const int64_t o = (a.tmap && a.t_scatter) ? (int64_t)a.tmap[i] : i;
    kcheck(o >= 0 && o < a.side.nnz, 5);
    a.t_out[o] = v;
    for (int p = 0; p < a.n_peers; ++p) a.peer_t[p][o] = v;
}

// After a thread's last peer store of the half-step: order its NVLink stores
// before anything the host sequences after the kernel (the barrier that ends
// the half-step is a stream-ordered collective on another device's queue).
__device__ __forceinline__ void peer_fence(const klnmf_solve_args_t &a) {
    if (a.n_peers > 0) __threadfence_system();
}

__device__ __forceinline__ void flush_stats(const Counters &cnt, bool lead, unsigned long long *stats, bool warp_sum) {
    if (!stats) return;
    unsigned ci = lead ? cnt.n_inner : 0u, cc = lead ? cnt.n_cap : 0u, cd = lead ? cnt.n_deg : 0u;
    unsigned cp = lead ? 1u : 0u;
    if (warp_sum) {
        ci = __reduce_add_sync(FULL_MASK, ci);
        cc = __reduce_add_sync(FULL_MASK, cc);
        cd = __reduce_add_sync(FULL_MASK, cd);
        cp = __reduce_add_sync(FULL_MASK, cp);
        if ((threadIdx.x & 31) != 0) return;
    } else if (!lead) {
        return;
    }
    if (ci) atomicAdd(stats + KLNMF_STAT_INNER_ITERS, (unsigned long long)ci);
    if (cc) atomicAdd(stats + KLNMF_STAT_CAP_HITS, (unsigned long long)cc);
    if (cd) atomicAdd(stats + KLNMF_STAT_DEGENERATE, (unsigned long long)cd);
    if (cp) atomicAdd(stats + KLNMF_STAT_PASSES, (unsigned long long)cp);
}

// Diagnostic build only (build.py variant "phase", tools/phase_timing.py):
// clock cycles per phase of the long-row kernels, thread 0 of every CTA,
// [kind][slot], kind 0 = cluster, 1 = cooperative, 2 = warp kernels (lane 0
// of every warp), 3 = block kernels (thread 0).  Slots 0-7 are cycles
// (init, gather, pass, chunk reduction, scalar Newton, update/re-evaluation,
// re-evaluation reduction, final writes), 8-11 counts (chunk reductions,
// re-evaluation reductions, moves, chunks), 12 the cycles of each subproblem's
// first reduction (which also waits for the slowest CTA of the group to arrive).
#ifdef KLNMF_PHASE_TIMING
__device__ unsigned long long g_phase[4][16];
__device__ __forceinline__ long long phase_now() {
    long long n;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(n));
    return n;
}
struct PhaseClock {
    long long t, acc[16];
    __device__ PhaseClock() : t(phase_now()) {
        for (int i = 0; i < 16; ++i) acc[i] = 0;
    }
    __device__ __forceinline__ void mark(int i) {
        const long long n = phase_now();
        acc[i] += n - t;
        t = n;
    }
    __device__ __forceinline__ void count(int i) { ++acc[i]; }
    __device__ void flush(int kind, bool lead) {
        if (lead)
            for (int i = 0; i < 16; ++i) atomicAdd(&g_phase[kind][i], (unsigned long long)acc[i]);
    }
};
#else
struct PhaseClock {
    __device__ __forceinline__ void mark(int) {}
    __device__ __forceinline__ void count(int) {}
    __device__ __forceinline__ void flush(int, bool) {}
};
#endif

// ---------------------------------------------------------------------------
// Warp kernel: groups of L <= 32 lanes, 32/L subproblems per warp in lock-step.
// CTR: counter coordinate order (a compile-time switch, so the shared order's
// code is not slowed by the per-subproblem order's indirections).
// Register caps (occupancy): the warp kernels with NPL <= 12 are compiled for
// 4 resident blocks per SM (128 registers; the uncapped code used 164-165
// and fit 3), the block kernels for <= 128 registers at NPL <= 12 (16 warps
// per SM; BK(256, *) had 8) and <= 168 above (the compiler's 230-246
// allowed 8 warps per SM).  Measured on C4: the warp and
// NPL > 12 block caps -9.2% per outer iteration against no caps, the
// NPL <= 12 block cap a further -1.5%; NPL = 14/16 warp kernels keep their
// registers (the shared-memory ring limits them to 3 blocks anyway).
#ifndef KLNMF_WARP_MINB
#define KLNMF_WARP_MINB 4
#endif
#ifndef KLNMF_WARP_MINB_NPL
#define KLNMF_WARP_MINB_NPL 12
#endif
#ifndef KLNMF_WARP_MINB_SMALL  // the same for NPL <= 7
#define KLNMF_WARP_MINB_SMALL KLNMF_WARP_MINB
#endif
#ifndef KLNMF_BATCH_TESTS  // batched entry tests after each chunk pass (warp kernels, L >= 4)
#define KLNMF_BATCH_TESTS 1
#endif
#ifndef KLNMF_WARP_MINB_LARGE  // the same for NPL > KLNMF_WARP_MINB_NPL
#define KLNMF_WARP_MINB_LARGE 1
#endif
constexpr int warp_minb(int npl) {
    return npl <= 7 ? KLNMF_WARP_MINB_SMALL : (npl <= KLNMF_WARP_MINB_NPL ? KLNMF_WARP_MINB : KLNMF_WARP_MINB_LARGE);
}
// Gather offsets of the entries in shared memory instead of registers
// (KLNMF_ROFF_SMEM) for the warp kernels whose blocks per SM it does not cut
// at rp <= 128 (the NPL = 8, 12, 16 rings leave no room): registers freed
// under the cap, C4 -1.0% (A/B, two repetitions).
#ifndef KLNMF_ROFF_SMEM
#define KLNMF_ROFF_SMEM 1
#endif
constexpr bool warp_roff_smem(int npl) { return KLNMF_ROFF_SMEM && (npl <= 7 || npl == 10 || npl == 14); }
// Threads per warp-kernel block.  One warp per block (32): a warp that
// finishes its subproblems releases its slot at once instead of idling until
// the slowest warp of its block is done; the row sums and the visit map are
// then read through L1 instead of being staged per block.
#ifndef KLNMF_WARP_NT
#define KLNMF_WARP_NT 32
#endif
constexpr int WARP_NT = KLNMF_WARP_NT;
constexpr bool WARP_STAGE_SUMS = WARP_NT >= 128;  // row sums / visit map staged in shared memory
template <int L, int NPL, bool CTR>
__global__ void __launch_bounds__(WARP_NT, warp_minb(NPL) * (128 / WARP_NT)) solve_warp_kernel(const klnmf_solve_args_t a) {
    constexpr int NT = WARP_NT;
    constexpr int GPB = NT / L;  // groups per block
    constexpr int STAGES = ring_stages(NPL);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool RS = warp_roff_smem(NPL);
    float4 *ring = reinterpret_cast<float4 *>(smem_raw);                 // [STAGES][NPL][NT]
    int *sroff = reinterpret_cast<int *>(ring + STAGES * NPL * NT);        // [NPL][NT] if RS
    float *xs_all = reinterpret_cast<float *>(sroff + (RS ? NPL * NT : 0));  // [GPB][2][rps]
    // counter order only: [GPB][MAX_CHUNKS] visit order of each group's chunks
    uint8_t *cord_all = reinterpret_cast<uint8_t *>(xs_all + GPB * 2 * (a.rp | 1));
    __shared__ double ssum_s[WARP_STAGE_SUMS ? KMAX_RP : 1];  // fixed-factor row sums by position
    __shared__ int pin_s[WARP_STAGE_SUMS ? KMAX_RP : 1];      // visit position -> stored position (perm_in)
    __shared__ double tots[GPB][NV];  // reduced partial sums of each group
    const double *ssum = WARP_STAGE_SUMS ? ssum_s : a.sum_pos;
    const int *pin = WARP_STAGE_SUMS ? pin_s : a.perm_in;

    const int tid = threadIdx.x;
    const int grp = tid / L;
    const int gl = tid & (L - 1);
    const int rp = a.rp, r = a.r;
    const int rps = rp | 1;
    // xs: the row as read (never written during the sweep), xo: the result.
    float *xs = xs_all + grp * 2 * rps;
    float *xo = xs + rps;
    double *tot = tots[grp];
    const int64_t slot = (int64_t)blockIdx.x * GPB + grp;
    const bool valid = slot < a.n_items;
    if (WARP_STAGE_SUMS) {
        for (int k = tid; k < r; k += NT) {
            ssum_s[k] = a.sum_pos[k];
            pin_s[k] = a.perm_in[k];
        }
        __syncthreads();
    }
    if (!__any_sync(FULL_MASK, valid)) return;

    PhaseClock ph;
    const Params pm(a);
    const float *fixed = static_cast<const float *>(a.fixed);
    float *moving = static_cast<float *>(a.moving);
    const float *val = static_cast<const float *>(a.side.val);
    const int64_t j = valid ? item_at(a, slot) : 0;
    const int64_t lo = valid ? a.side.ptr[j] : 0;
    const int s = valid ? (int)(a.side.ptr[j + 1] - lo) : 0;

    // batched entry tests (L >= 4): the result row starts as the input row and
    // only coordinates that enter the Newton loop write it
    constexpr bool BATCH = KLNMF_BATCH_TESTS && L >= 4;
    load_row(xs, moving + j * rp, pin, r, gl, L, valid, BATCH ? xo : nullptr);
    const int nchunks = (r + C - 1) / C;
    constexpr bool counter = CTR;
    uint8_t *cord = cord_all + grp * MAX_CHUNKS;
    if (counter && gl == 0) chunk_order(a.order_seed, *a.order_iter, (uint32_t)j, a.order_side, nchunks, cord);
    __syncwarp();

    double u[NPL], vi[NPL];
    int roff_r[RS ? 1 : NPL];  // gather source of each entry (row 0 for absent entries)
    auto roff = [&](int e) -> int & {
        if constexpr (RS) return sroff[e * NT + tid];
        else return roff_r[e];
    };
#pragma unroll
    for (int e = 0; e < NPL; ++e) {
        const int p = gl + e * L;
        if (p < s) {
            const int64_t q = lo + p;
            roff(e) = gather_off(a, q);
            entry_init(a.t_in[t_index(a, q)], val[q], pm.eps_div, u[e], vi[e]);
        } else {
            roff(e) = 0;
            u[e] = vi[e] = 0.0;  // contributes exactly 0 to every sum
        }
    }
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring) + 16u * tid;
    auto phys = [&](int chunk) -> int { return counter ? (int)cord[chunk] : chunk; };
    auto issue = [&](int chunk) {
        if (chunk < nchunks) {
            const unsigned base = ring_s + 16u * NT * NPL * (chunk % STAGES);
            const int pc = phys(chunk);
#pragma unroll
            for (int e = 0; e < NPL; ++e)
                cp_async16(base + 16u * NT * e, fixed + roff(e) + pc * C, gl + e * L < s);
        }
        cp_commit();
    };
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) issue(st);
    __syncwarp();
    ph.mark(0);

    Counters cnt;
    for (int ch = 0; ch < nchunks; ++ch) {
        ph.count(11);
        issue(ch + STAGES - 1);
        cp_wait<STAGES - 1>();
        ph.mark(1);
        const float4 *Ach = ring + (ch % STAGES) * NPL * NT + tid;  // own slots of this stage
        const int pc = phys(ch);  // per group in counter order
        const int nc = counter ? C : min(C, r - ch * C);
        // counter order: this group's own order of the chunk's 4 coordinates
        const uint32_t perm = counter ? chunk_perm4(a.order_seed, *a.order_iter, (uint32_t)j, a.order_side, ch)
                                      : PERM4_IDENTITY;
        bool fresh = false;  // tot valid for the current t
        unsigned emask = 0;  // BATCH: slots of this chunk whose coordinate enters (valid while fresh)
#pragma unroll 1
        for (int cc = 0; cc < nc; ++cc) {
            const int q = (int)((perm >> (2 * cc)) & 3u);  // chunk coordinate visited in slot cc
            const int tt = pc * C + q;
            const bool live = tt < r;
            const bool need_pass = __any_sync(FULL_MASK, !fresh);
            if (need_pass) {
                double red[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
                // shared order: the chunk's remaining coordinates cc..C-1;
                // counter order: all four (the remaining ones are any subset)
                with_cc(counter ? 0 : cc, [&](auto ccv) {
#pragma unroll
                    for (int e = 0; e < NPL; ++e)
                        accum_from<decltype(ccv)::value>(red, Ach[e * NT], u[e], entry_z(u[e], vi[e]));
                });
                ph.mark(2);
                TReduce<L>::run(red, gl);
                TReduce<L>::store(red, gl, tot);
                __syncwarp();
                ph.mark(3);
                ph.count(8);
                fresh = true;
            }
            if (BATCH) {
                if (need_pass) {
                    // entry tests of the slots cc..nc-1 at once, lane gl testing slot
                    // cc + gl, with the same expressions as the visit below (so the
                    // same bits): the visits no group enters are skipped
                    const int sl = cc + gl;
                    bool ent = false;
                    if (valid && sl < nc) {
                        const int qs = (int)((perm >> (2 * sl)) & 3u);
                        const int ts = pc * C + qs;
                        if (!counter || ts < r) {
                            const double xv = (double)xs[ts];
                            const double bv = ssum[ts] + pm.beta;
                            ent = enters((bv + pm.alpha * xv) - tot[qs], xv, pm.eps_grad);
                        }
                    }
                    const unsigned b = __ballot_sync(FULL_MASK, ent);
                    const unsigned gb = L == 32 ? b : (b >> ((threadIdx.x & 31) & ~(L - 1))) & ((1u << (L & 31)) - 1u);
                    emask = (gb & 0xFu) << cc;
                }
                if (!__any_sync(FULL_MASK, (emask >> cc) & 1u)) continue;  // x unchanged, xo = xs already
            }
            double x = (!counter || live) ? (double)xs[tt] : 0.0;
            const double base = ((!counter || live) ? ssum[tt] : 0.0) + pm.beta;
            double g = (base + pm.alpha * x) - tot[q];
            double h = pm.alpha + tot[C + q];
            int inner = 0;
            bool active = valid && live && enters(g, x, pm.eps_grad);
            bool moved = false;
            while (__any_sync(FULL_MASK, active)) {
                bool again = false;
                double delta = 0.0;
                if (active) delta = newton_step(g, h, x, inner, active, again, pm, cnt);
                ph.mark(4);
                if (__any_sync(FULL_MASK, delta != 0.0)) {
                    if (delta != 0.0) moved = true;
                    // delta == 0 (groups not moving) leaves every entry unchanged (q = 1)
                    with_clamp(__any_sync(FULL_MASK, delta < 0.0), [&](auto cl) {
#pragma unroll
                        for (int e = 0; e < NPL; ++e)
                            entry_update<decltype(cl)::value>(delta, widen(comp(Ach + e * NT, q)), pm.eps_div, u[e],
                                                              vi[e]);
                    });
                    ph.mark(5);
                    ph.count(10);
                }
                if (__any_sync(FULL_MASK, again)) {
                    double g2 = 0.0, h2 = 0.0;
#pragma unroll
                    for (int e = 0; e < NPL; ++e)
                        accum(g2, h2, u[e], entry_z(u[e], vi[e]), widen(comp(Ach + e * NT, q)));
#pragma unroll
                    for (int o = L / 2; o > 0; o >>= 1) {
                        g2 += __shfl_xor_sync(FULL_MASK, g2, o);
                        h2 += __shfl_xor_sync(FULL_MASK, h2, o);
                    }
                    if (again) {
                        g = (base + pm.alpha * x) - g2;
                        h = pm.alpha + h2;
                        active = enters(g, x, pm.eps_grad);
                    }
                    ph.mark(6);
                    ph.count(9);
                }
            }
            if (moved) fresh = false;
            if (gl == 0 && valid && live) xo[tt] = (float)x;
            ph.mark(4);
        }
    }
    cp_wait<0>();
    __syncwarp();
    if (valid) {
        for (int k = gl; k < r; k += L) put_moving(a, moving, j * rp + a.perm_out[k], xo[k]);
#pragma unroll
        for (int e = 0; e < NPL; ++e)
            if (gl + e * L < s) put_t(a, lo + gl + e * L, entry_t(u[e], vi[e], pm.eps_div));
    }
    peer_fence(a);
    flush_stats(cnt, gl == 0 && valid, a.stats, true);
    ph.mark(7);
    ph.flush(2, (threadIdx.x & 31) == 0);
}

// ---------------------------------------------------------------------------
// Block-wide reduction of NV values: warp transposed reduce, per-warp totals
// to shared memory (double-buffered, one barrier per reduction).  The block
// total of value i is then the fixed-order sum over warps, read on demand.
template <int NT>
struct BlockSums {
    static constexpr int NW = NT / 32;
    double w[2][NW][NV];
    __device__ __forceinline__ void reduce(double (&v)[NV], int buf) {
        const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
        TReduce<32>::run(v, lane);
        if ((lane & 3) == 0) w[buf][wi][lane >> 2] = v[0];
        __syncthreads();
    }
    // (g, h) of one coordinate into slots 0, 1: one halving level, then a
    // butterfly on the kept value (lanes < 16 end with g, the others with h)
    __device__ __forceinline__ void reduce2(double g, double h, int buf) {
        const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
        const bool up = (lane & 16) != 0;
        double keep = (up ? h : g) + __shfl_xor_sync(FULL_MASK, up ? g : h, 16);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) keep += __shfl_xor_sync(FULL_MASK, keep, o);
        if ((lane & 15) == 0) w[buf][wi][lane >> 4] = keep;
        __syncthreads();
    }
    __device__ __forceinline__ double get(int buf, int i) const {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) s += w[buf][q][i];
        return s;
    }
};

// One subproblem per block, NPL register entries per thread.
#ifndef KLNMF_BLOCK_MAXREG  // register cap of the block kernels (0 = none)
#define KLNMF_BLOCK_MAXREG 168
#endif
#ifndef KLNMF_BLOCK_MAXREG_SMALL  // the same for NPL <= KLNMF_BLOCK_SMALL_NPL
#define KLNMF_BLOCK_MAXREG_SMALL 128
#endif
#ifndef KLNMF_BLOCK_SMALL_NPL
#define KLNMF_BLOCK_SMALL_NPL 12
#endif
constexpr int block_minb(int nt, int npl) {
    const int cap = npl <= KLNMF_BLOCK_SMALL_NPL ? KLNMF_BLOCK_MAXREG_SMALL : KLNMF_BLOCK_MAXREG;
    return cap > 0 ? (65536 / (nt * cap) > 0 ? 65536 / (nt * cap) : 1) : 1;
}
#ifndef KLNMF_BROFF_SMEM  // the same for the block kernels that keep their blocks per SM (C4 -0.9%)
#define KLNMF_BROFF_SMEM 1
#endif
constexpr bool block_roff_smem(int nt, int npl) {
    return KLNMF_BROFF_SMEM && (npl == 10 || npl == 14 || (nt == 256 && npl == 16));
}
template <int NT, int NPL, bool CTR>
__global__ void __launch_bounds__(NT, block_minb(NT, NPL)) solve_block_kernel(const klnmf_solve_args_t a) {
    constexpr int STAGES = ring_stages(NPL);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4 *ring = reinterpret_cast<float4 *>(smem_raw);             // [STAGES][NPL][NT]
    constexpr bool RS = block_roff_smem(NT, NPL);
    int *sroff = reinterpret_cast<int *>(ring + STAGES * NPL * NT);      // [NPL][NT] if RS
    float *xs = reinterpret_cast<float *>(sroff + (RS ? NPL * NT : 0));  // [2][rps]: input row, result
    float *xo = xs + (a.rp | 1);
    uint8_t *cord = reinterpret_cast<uint8_t *>(xo + (a.rp | 1));  // counter order only
    __shared__ double ssum[KMAX_RP];
    __shared__ BlockSums<NT> bs;

    const int tid = threadIdx.x;
    const int64_t slot = blockIdx.x;
    if (slot >= a.n_items) return;
    PhaseClock ph;
    const Params pm(a);
    const int rp = a.rp, r = a.r;
    const float *fixed = static_cast<const float *>(a.fixed);
    float *moving = static_cast<float *>(a.moving);
    const float *val = static_cast<const float *>(a.side.val);
    const int64_t j = item_at(a, slot);
    const int64_t lo = a.side.ptr[j];
    const int s = (int)(a.side.ptr[j + 1] - lo);

    for (int k = tid; k < r; k += NT) ssum[k] = a.sum_pos[k];
    // the result row starts as the input row (batched entry tests: only
    // coordinates that enter the Newton loop write it)
    for (int k = tid; k < r; k += NT) xs[k] = xo[k] = moving[j * rp + a.perm_in[k]];

    double u[NPL], vi[NPL];
    int roff_r[RS ? 1 : NPL];
    auto roff = [&](int e) -> int & {
        if constexpr (RS) return sroff[e * NT + tid];
        else return roff_r[e];
    };
#pragma unroll
    for (int e = 0; e < NPL; ++e) {
        const int p = tid + e * NT;
        if (p < s) {
            const int64_t q = lo + p;
            roff(e) = gather_off(a, q);
            entry_init(a.t_in[t_index(a, q)], val[q], pm.eps_div, u[e], vi[e]);
        } else {
            roff(e) = 0;
            u[e] = vi[e] = 0.0;
        }
    }
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring) + 16u * tid;
    const int nchunks = (r + C - 1) / C;
    constexpr bool counter = CTR;
    if (counter) {
        if (tid == 0) chunk_order(a.order_seed, *a.order_iter, (uint32_t)j, a.order_side, nchunks, cord);
        __syncthreads();
    }
    auto phys = [&](int chunk) -> int { return counter ? (int)cord[chunk] : chunk; };
    auto issue = [&](int chunk) {
        if (chunk < nchunks) {
            const unsigned base = ring_s + 16u * NT * NPL * (chunk % STAGES);
            const int pc = phys(chunk);
#pragma unroll
            for (int e = 0; e < NPL; ++e)
                cp_async16(base + 16u * NT * e, fixed + roff(e) + pc * C, tid + e * NT < s);
        }
        cp_commit();
    };
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) issue(st);
    __syncthreads();
    ph.mark(0);

    Counters cnt;
    int buf = 0, cur = 0;  // cur: buffer holding the last pass's sums
    for (int ch = 0; ch < nchunks; ++ch) {
        ph.count(11);
        issue(ch + STAGES - 1);
        cp_wait<STAGES - 1>();
        ph.mark(1);
        const float4 *Ach = ring + (ch % STAGES) * NPL * NT + tid;
        const int pc = phys(ch);
        const int nc = counter ? C : min(C, r - pc * C);
        const uint32_t perm = counter ? chunk_perm4(a.order_seed, *a.order_iter, (uint32_t)j, a.order_side, ch)
                                      : PERM4_IDENTITY;
        bool fresh = false;
        unsigned emask = 0;  // slots of this chunk whose coordinate enters (valid while fresh)
#pragma unroll 1
        for (int cc = 0; cc < nc; ++cc) {
            const int q = (int)((perm >> (2 * cc)) & 3u);  // chunk coordinate visited in slot cc
            const int tt = pc * C + q;
            if (counter && tt >= r) continue;  // counter order: padding slot of the last chunk
            if (!fresh) {  // block-uniform
                double red[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
                with_cc(counter ? 0 : cc, [&](auto ccv) {
#pragma unroll
                    for (int e = 0; e < NPL; ++e)
                        accum_from<decltype(ccv)::value>(red, Ach[e * NT], u[e], entry_z(u[e], vi[e]));
                });
                ph.mark(2);
                bs.reduce(red, buf);
                ph.mark(3);
                ph.count(8);
                cur = buf;
                buf ^= 1;
                fresh = true;
                // entry tests of the slots cc..nc-1 at once (lane l of every warp
                // tests slot cc + l, same expressions as the visit below); the
                // mask is identical in every warp, so the skip is block-uniform
                const int sl = cc + (tid & 31);
                bool ent = false;
                if (sl < nc) {
                    const int qs = (int)((perm >> (2 * sl)) & 3u);
                    const int ts = pc * C + qs;
                    if (!counter || ts < r) {
                        const double xv = (double)xs[ts];
                        const double bv = ssum[ts] + pm.beta;
                        ent = enters((bv + pm.alpha * xv) - bs.get(cur, qs), xv, pm.eps_grad);
                    }
                }
                emask = (__ballot_sync(FULL_MASK, ent) & 0xFu) << cc;
            }
            if (!((emask >> cc) & 1u)) continue;  // x unchanged, xo = xs already
            double x = (double)xs[tt];
            const double base = ssum[tt] + pm.beta;
            double g = (base + pm.alpha * x) - bs.get(cur, q);
            double h = pm.alpha + bs.get(cur, C + q);
            int inner = 0;
            bool active = enters(g, x, pm.eps_grad);
            bool moved = false;
            while (active) {  // block-uniform
                bool again = false;
                const double delta = newton_step(g, h, x, inner, active, again, pm, cnt);
                ph.mark(4);
                if (delta != 0.0) {
                    ph.count(10);
                    moved = true;
                    with_clamp(delta < 0.0, [&](auto cl) {
#pragma unroll
                        for (int e = 0; e < NPL; ++e)
                            entry_update<decltype(cl)::value>(delta, widen(comp(Ach + e * NT, q)), pm.eps_div, u[e],
                                                              vi[e]);
                    });
                }
                ph.mark(5);
                if (again) {
                    double g2 = 0.0, h2 = 0.0;
#pragma unroll
                    for (int e = 0; e < NPL; ++e)
                        accum(g2, h2, u[e], entry_z(u[e], vi[e]), widen(comp(Ach + e * NT, q)));
                    bs.reduce2(g2, h2, buf);
                    ph.mark(6);
                    ph.count(9);
                    g = (base + pm.alpha * x) - bs.get(buf, 0);
                    h = pm.alpha + bs.get(buf, 1);
                    buf ^= 1;
                    active = enters(g, x, pm.eps_grad);
                    moved = true;  // the chunk sums' buffer may be recycled: re-pass next
                }
            }
            if (moved) fresh = false;
            if (tid == 0) xo[tt] = (float)x;
            ph.mark(4);
        }
    }
    cp_wait<0>();
    __syncthreads();
    for (int k = tid; k < r; k += NT) put_moving(a, moving, j * rp + a.perm_out[k], xo[k]);
#pragma unroll
    for (int e = 0; e < NPL; ++e)
        if (tid + e * NT < s) put_t(a, lo + tid + e * NT, entry_t(u[e], vi[e], pm.eps_div));
    peer_fence(a);
    flush_stats(cnt, tid == 0, a.stats, false);
    ph.mark(7);
    ph.flush(3, tid == 0);
}

// ---------------------------------------------------------------------------
// Long subproblems (the W side's popular rows): one subproblem per CTA
// cluster of k <= 16 CTAs, or (solve_coop_kernel) per group of G CTAs of a
// persistent cooperative launch.  Each CTA owns a contiguous slice of the
// entries and keeps their state ON CHIP -- NR entries per thread in
// registers, NS in shared memory; only entries beyond that spill to global
// memory (t_out / scratch).  At the start of every chunk each thread gathers
// the chunk of its resident entries into shared memory once; all passes and
// moves of the chunk read it from there.
namespace cg = cooperative_groups;

// 256 threads and ~101 KB of shared memory per CTA: two slices (of different
// rows, or of one row) share an SM, so one CTA's reduction and gather latency
// overlaps the other's arithmetic.  16 resident entries per thread: 8 in
// registers (u, 1/v, row offset), 8 in shared memory.
#ifndef KLNMF_CL_NT  // slice-CTA shape (overridable for experiments)
#define KLNMF_CL_NT 256
#define KLNMF_CL_PER_SM 2
#endif
#ifndef KLNMF_CL_OFF_SMEM  // long-row kernels: the shared-memory entries' gather offsets in shared memory (C4 -1.4%)
#define KLNMF_CL_OFF_SMEM 1
#endif
constexpr int CL_NT = KLNMF_CL_NT, CL_NR = 8, CL_NS = 8, CL_PER_SM = KLNMF_CL_PER_SM;
constexpr int CL_NE = CL_NR + CL_NS;  // resident entries per thread
constexpr int CL_MAXG = CL_PER_SM > 2 ? 1024 : 512;  // most CTAs in one cooperative row group
constexpr size_t COOP_GROUP_BYTES = 2 * CL_MAXG * NV * 2 * sizeof(unsigned long long) + 128;

// Record of a spilled entry of the long-row kernels (scratch): u, 1/v and
// the current chunk's four fixed-factor values -- one 32-byte sector, so a
// warp's consecutive entries stream whole sectors (a structure-of-arrays
// layout, reading only the components a pass or move uses, measured 3.7%
// slower on C5's spilled rows: more requests for the same sectors).  Next
// to the records (after 4*nnz doubles), one byte per entry holds the chunk's
// nonzero mask (bit c: a_c != 0), written by the stage: a pass over
// coordinates c0..3 reads only the records with a nonzero among them, a move
// or re-evaluation of coordinate q only those with a_q != 0 (78-85% of the
// fixed factors are zeros; a zero term adds exactly 0 and leaves u exactly
// unchanged), and a move writes back only what it changed.  The loops are
// kept out of line: they run only for rows longer than the on-chip capacity
// of their CTAs, and inlined they raised the register pressure (spills) of
// every long-row slice (out of line: C4 -1.0%).
struct __align__(32) SpillRec {
    double2 uv;  // u = v/(t+eps), vi = 1/v
    float4 a;    // the current chunk of the entry's fixed-factor row
};
static_assert(sizeof(SpillRec) == 32, "one 32-byte sector per spilled entry");
struct P8 {
    double v[NV];
};
struct P2 {
    double g, h;
};
// the chunk's fixed-factor slice of every spilled entry i0, i0 + step, ... < cn
__device__ __noinline__ void spill_stage(SpillRec *rec, uint8_t *mask, int64_t i0, int64_t cn, int64_t step,
                                        const float *fixed, const int32_t *idx, int64_t n_fix, int rp, int pc) {
#pragma unroll 4
    for (int64_t i = i0; i < cn; i += step) {
        const int32_t row = idx[i];
        kcheck(row >= 0 && row < n_fix, 1);
        const float4 a4 = ldg_f4(fixed + (int64_t)row * rp + pc * C);
        const unsigned m = (a4.x != 0.f ? 1u : 0u) | (a4.y != 0.f ? 2u : 0u) | (a4.z != 0.f ? 4u : 0u) |
                           (a4.w != 0.f ? 8u : 0u);
        mask[i] = (uint8_t)m;
        if (m) __stcg(&rec[i].a, a4);
    }
}
// partials of the chunk's coordinates c0..3 over the spilled entries, added to acc
__device__ __noinline__ P8 spill_pass(const SpillRec *rec, const uint8_t *mask, int64_t i0, int64_t cn,
                                     int64_t step, int c0, P8 acc) {
#pragma unroll 4
    for (int64_t i = i0; i < cn; i += step) {
        if ((__ldcg(mask + i) >> c0) == 0) continue;  // a_c0..a_3 all zero: adds exactly 0
        const double2 uv = __ldcg(&rec[i].uv);
        accum_chunk(acc.v, __ldcg(&rec[i].a), uv.x, entry_z(uv.x, uv.y), c0);
    }
    return acc;
}
// a move of coordinate q by delta (upd) and/or its re-evaluation partials
// (again, added to acc) over the spilled entries
__device__ __noinline__ P2 spill_move(SpillRec *rec, const uint8_t *mask, int64_t i0, int64_t cn, int64_t step,
                                     int q, double delta, bool upd, bool again, bool clamp, double eps, P2 acc) {
#pragma unroll 4
    for (int64_t i = i0; i < cn; i += step) {
        if (!((__ldcg(mask + i) >> q) & 1u)) continue;  // a_q == 0: u unchanged, contributes exactly 0
        const double av = (double)__ldcg(reinterpret_cast<const float *>(&rec[i].a) + q);
        double2 uv = __ldcg(&rec[i].uv);
        if (upd) {
            if (clamp) entry_update<true>(delta, av, eps, uv.x, uv.y);
            else entry_update<false>(delta, av, eps, uv.x, uv.y);
            __stcg(&rec[i].uv, uv);
        }
        if (again) accum(acc.g, acc.h, uv.x, entry_z(uv.x, uv.y), av);
    }
    return acc;
}

struct GroupRed {
    double wred[2][CL_NT / 32][NV];
    double cpart[2][NV];
    double tot[2][NV];
};

// CTA part of a group reduction: warp transposed reduce, fixed-order sum over
// warps.  Returns the CTA partial of value `lane` in warp 0, lanes < NV (and
// also stores it to cpart[buf]).
__device__ __forceinline__ double cta_partial(double (&v)[NV], GroupRed &R, int buf) {
    constexpr int NW = CL_NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    TReduce<32>::run(v, lane);
    if ((lane & 3) == 0) R.wred[buf][w][lane >> 2] = v[0];
    __syncthreads();
    double s = 0.0;
    if (w == 0 && lane < NV) {
#pragma unroll
        for (int q = 0; q < NW; ++q) s += R.wred[buf][q][lane];
        R.cpart[buf][lane] = s;
    }
    return s;
}

// Fixed-order warp sum (butterfly); every lane gets the total.
__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL_MASK, s, o);
    return s;
}

// --- DSMEM push primitives (sm_90+ cluster PTX) ---
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa_u32(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned a, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
// CTA-scope acquire: the awaited data are shared-memory bytes counted by the
// barrier's transaction count, written before the phase can complete.
__device__ __forceinline__ bool mbar_try(unsigned a, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}
// 16 bytes into a peer CTA's shared memory, completing bytes on its mbarrier.
__device__ __forceinline__ void st_async_v2(unsigned raddr, double x, double y, unsigned rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "d"(x), "d"(y), "r"(rmbar)
                 : "memory");
}

#ifndef KLNMF_CL_SUM_UNROLL
#define KLNMF_CL_SUM_UNROLL 4
#endif
constexpr int CL_SUM_UNROLL = KLNMF_CL_SUM_UNROLL;
constexpr int CL_MAXK = 16;  // largest cluster
// Per-CTA inbox of the cluster all-reduce: round parity x source CTA x value.
#ifdef KLNMF_CHECKED
constexpr unsigned INBOX_TAG_BYTES = 16;  // checked build: (round, sender) rides along
#else
constexpr unsigned INBOX_TAG_BYTES = 0;
#endif
struct ClusterInbox {
    __align__(16) double box[2][CL_MAXK][NV];
#ifdef KLNMF_CHECKED
    __align__(16) double tag[2][CL_MAXK][2];
#endif
    __align__(8) unsigned long long mbar[2];
};

// Sum over the k CTAs of a cluster: every CTA pushes its NV partials into
// every peer's inbox with st.async (one-way DSMEM traffic, completion counted
// in bytes on the receiver's mbarrier) and waits only for its own inbox -- no
// cluster-wide barrier per reduction.  The receiver sums the k partials in CTA
// order, so the total is identical in every CTA and deterministic.
// Reuse: round n+2 writes the parity buffer of round n; a peer can only send
// it after receiving this CTA's round n+1 partial, which is sent after this
// CTA has finished reading round n.
struct ClusterReducer {
    GroupRed &R;
    ClusterInbox &P;
    int k, rank;
    unsigned round;
    __device__ __forceinline__ void operator()(double (&v)[NV], int buf) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        const double s = cta_partial(v, R, buf);
        if (w == 0) {
            if (k > 1) {
                const int b = round & 1;
                const unsigned mb = smem_u32(&P.mbar[b]);
                const unsigned slot = smem_u32(&P.box[b][rank][0]);
                const int q = lane & (NV / 2 - 1);  // value pair of this lane
                const double x0 = __shfl_sync(FULL_MASK, s, 2 * q);
                const double x1 = __shfl_sync(FULL_MASK, s, 2 * q + 1);
                for (int i = lane; i < k * (NV / 2); i += 32) {
                    const unsigned peer = (unsigned)(i / (NV / 2));
                    st_async_v2(mapa_u32(slot + 16u * q, peer), x0, x1, mapa_u32(mb, peer));
                }
#ifdef KLNMF_CHECKED
                if (lane < k)
                    st_async_v2(mapa_u32(smem_u32(&P.tag[b][rank][0]), (unsigned)lane), (double)round, (double)rank,
                                mapa_u32(mb, (unsigned)lane));
#endif
                if (lane == 0) mbar_arrive_tx(mb, (unsigned)(k * (NV * sizeof(double) + INBOX_TAG_BYTES)));
                while (!mbar_try(mb, (round >> 1) & 1u)) {
                }
#ifdef KLNMF_CHECKED
                // every peer's partial of this round, none of an older or newer one
                if (lane < k) kcheck(P.tag[b][lane][0] == (double)round && P.tag[b][lane][1] == (double)lane, 10);
#endif
                if (lane < NV) {
                    double t = 0.0;
                    // the peers' partials are loaded in batches ahead of the ordered sum
                    _Pragma("unroll CL_SUM_UNROLL")
                    for (int c = 0; c < k; ++c) t += P.box[b][c][lane];
                    R.tot[buf][lane] = t;
                }
            } else if (lane < NV) {
                R.tot[buf][lane] = s;
            }
        }
        __syncthreads();
        ++round;
    }
};

// Sum over the G CTAs of a cooperative row group through global memory.
// Each partial travels as two 8-byte words {32 value bits, 32-bit round tag}
// (the LL idea of NCCL's low-latency protocol): 8-byte accesses are
// single-copy atomic, so a reader that sees the current tag in both words
// has the whole value and per-location coherence rules out stale words --
// no fence is needed anywhere.  Arrival is signalled by a relaxed atomic on
// the group counter that one lane per CTA polls (one word of polling
// traffic); should a counter increment overtake its data, the tag check
// simply waits for the data.  Tags are round + 1 (memset 0 = empty) and never
// repeat, so parity double-buffering is enough: a slot of round n is
// rewritten at round n + 2, after every reader of round n has published
// round n + 1.  Warp i then sums value i over the G CTAs (lane c reads CTA c)
// in a fixed order.
__device__ __forceinline__ ulonglong2 ld_relaxed_v2(const unsigned long long *p) {
    ulonglong2 v;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_v2(unsigned long long *p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

#ifndef KLNMF_COOP_SLEEP_NS
#define KLNMF_COOP_SLEEP_NS 32
#endif
__device__ __forceinline__ void coop_backoff() {
    if (KLNMF_COOP_SLEEP_NS > 0) __nanosleep(KLNMF_COOP_SLEEP_NS);
}

// Lane `lane`'s share of one value's sum over the G slots of a cooperative
// reduction round (slots c = lane, lane + 32, ... in ascending order).
// KLNMF_COOP_RD slots per lane are requested before the first tag is tested,
// so a wide group (G up to 512: 16 slots per lane) pays one L2 round trip per
// batch instead of one per slot.  Out of line (KLNMF_COOP_NOINLINE): the
// batch's registers do not add to the pressure of the slice loop.
#ifndef KLNMF_COOP_RD
#define KLNMF_COOP_RD 2
#endif
#ifndef KLNMF_COOP_NOINLINE
#define KLNMF_COOP_NOINLINE 1
#endif
#if KLNMF_COOP_NOINLINE
#define KLNMF_COOP_SUM_ATTR __noinline__
#else
#define KLNMF_COOP_SUM_ATTR __forceinline__
#endif
__device__ KLNMF_COOP_SUM_ATTR double coop_sum_column(const unsigned long long *col, int G, unsigned tag, int lane) {
    double acc = 0.0;
    for (int c0 = 0; c0 < G; c0 += 32 * KLNMF_COOP_RD) {
        ulonglong2 q[KLNMF_COOP_RD];
#pragma unroll
        for (int b2 = 0; b2 < KLNMF_COOP_RD; ++b2) {
            const int c = c0 + 32 * b2 + lane;
            if (c < G) q[b2] = ld_relaxed_v2(col + 2 * c);
        }
#pragma unroll
        for (int b2 = 0; b2 < KLNMF_COOP_RD; ++b2) {
            const int c = c0 + 32 * b2 + lane;
            double x = 0.0;
            if (c < G) {
                while ((unsigned)q[b2].x != tag || (unsigned)q[b2].y != tag) {
                    // a newer tag means round n+2 overwrote this slot before it was read
                    kcheck((unsigned)q[b2].x <= tag && (unsigned)q[b2].y <= tag, 6);
                    coop_backoff();
                    q[b2] = ld_relaxed_v2(col + 2 * c);
                }
                x = __longlong_as_double((long long)((q[b2].x & 0xffffffff00000000ull) | (q[b2].y >> 32)));
            }
            acc += x;
        }
    }
    return acc;
}

struct CoopReducer {
    GroupRed &R;
    unsigned long long *slots;  // [2][NV][CL_MAXG][2] tagged words
    unsigned *counter;          // arrivals, G per round
    int G, rank;
    unsigned round;
    __device__ __forceinline__ void operator()(double (&v)[NV], int buf) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        const double s = cta_partial(v, R, buf);
        if (G == 1) {
            if (w == 0 && lane < NV) R.tot[buf][lane] = s;
            __syncthreads();
            return;
        }
        const unsigned b = round & 1u;
        const unsigned long long tag = round + 1u;
        if (w == 0 && lane < NV) {
            const unsigned long long bits = (unsigned long long)__double_as_longlong(s);
            st_relaxed_v2(slots + (((size_t)b * NV + lane) * CL_MAXG + rank) * 2, (bits & 0xffffffff00000000ull) | tag,
                          (bits << 32) | tag);
        }
        if (w == 0) {
            __syncwarp();
            if (lane == 0) {
                atomicAdd(counter, 1u);
                const unsigned target = (unsigned)G * (round + 1u);
                unsigned seen;
                while ((seen = *(volatile unsigned *)counter) < target) coop_backoff();
                // no partner can arrive twice before this CTA arrives again
                kcheck(seen <= (unsigned)G * (round + 2u), 7);
            }
        }
        __syncthreads();
        for (int vw = w; vw < NV; vw += CL_NT / 32) {  // warp vw sums value vw (any CTA width)
            const unsigned long long *col = slots + ((size_t)b * NV + vw) * CL_MAXG * 2;
            double acc = coop_sum_column(col, G, (unsigned)tag, lane);
            acc = warp_sum(acc);
            if (lane == 0) R.tot[buf][vw] = acc;
        }
        __syncthreads();
        ++round;
    }
};

// Per-thread chunk masks of a slice (klnmf_solve_args_t.fixed_mask): word
// [chunk][tid] holds bit e = "resident entry e of this thread has a nonzero
// in that chunk of its fixed-factor row".  Built once per slice from the
// per-row masks into klnmf_solve_args_t.slice_words (8 bytes of word space
// per entry: the slice's own range), read back one word per thread and chunk.
// Out of line: the 16 row masks are live only here.
constexpr int SLICE_MASK_CHUNKS = 32;  // one bit per chunk in the per-row words: r <= 128
__device__ __noinline__ void slice_masks_build(uint16_t *words, const uint32_t *fixed_mask, const int32_t *idx,
                                               int64_t cn, int nchunks) {
    const int tid = threadIdx.x;
    uint32_t m[CL_NE];
#pragma unroll
    for (int e = 0; e < CL_NE; ++e) {
        const int64_t i = tid + (int64_t)e * CL_NT;
        m[e] = i < cn ? __ldg(fixed_mask + idx[i]) : 0u;
    }
    for (int c = 0; c < nchunks; ++c) {
        unsigned w = 0;
#pragma unroll
        for (int e = 0; e < CL_NE; ++e) w |= ((m[e] >> c) & 1u) << e;
        words[c * CL_NT + tid] = (uint16_t)w;
    }
}

// One subproblem's slice on one CTA (rank cq of the k CTAs sharing it).
template <bool CTR, typename Reducer>
__device__ __forceinline__ void solve_slice(const klnmf_solve_args_t &a, int64_t slot, int cq, int k, Reducer &reduce,
                                            GroupRed &R, unsigned char *smem_raw, const double *ssum) {
    constexpr int NT = CL_NT, NR = CL_NR, NS = CL_NS;
    float4 *cache = reinterpret_cast<float4 *>(smem_raw);             // [NR+NS][NT]: current chunk
    double *Us = reinterpret_cast<double *>(cache + (NR + NS) * NT);  // [NS][NT]
    double *VIs = Us + NS * NT;                                       // [NS][NT]
    // gather offsets of the shared-memory entries: in shared memory too
    // (KLNMF_CL_OFF_SMEM), or in registers
    int *Offs = reinterpret_cast<int *>(VIs + NS * NT);                          // [NS][NT] if in smem
    float *xs = reinterpret_cast<float *>(Offs + (KLNMF_CL_OFF_SMEM ? NS * NT : 0));  // [2][rps]: input row, result
    float *xo = xs + (a.rp | 1);
    uint8_t *cord = reinterpret_cast<uint8_t *>(xo + (a.rp | 1));  // counter order

    PhaseClock ph;
    const Params pm(a);
    const int tid = threadIdx.x;
    const int rp = a.rp, r = a.r;
    const float *fixed = static_cast<const float *>(a.fixed);
    float *moving = static_cast<float *>(a.moving);
    const float *val = static_cast<const float *>(a.side.val);
    const int64_t j = item_at(a, slot);
    const int64_t lo = a.side.ptr[j];
    const int64_t s = a.side.ptr[j + 1] - lo;
    const int64_t per = (s + k - 1) / k;
    const int64_t c0 = min(s, (int64_t)cq * per);
    const int64_t cn = min(s, c0 + per) - c0;  // entries of this CTA
    const int64_t base = lo + c0;              // global entry index of local entry 0
    // resident entry slots in use (CTA-uniform): slots e >= ne hold no entry
    // in any thread and are skipped, so a slice filled to 70% of its 16
    // slots per thread costs ~70% of a full one
    // (cooperative rows fill their slices by construction: no test there)
    const int ne = std::is_same<Reducer, CoopReducer>::value ? NR + NS
                                                             : (int)min((cn + NT - 1) / NT, (int64_t)(NR + NS));
    const double eps = pm.eps_div;
    // spilled entries (rows longer than the on-chip capacity of their CTAs):
    // a 32-byte record per entry in scratch -- (u, vi) and the current
    // chunk's 4 fixed-factor values, staged once per chunk -- so every pass
    // and move streams whole sectors instead of re-gathering the fixed factor
    SpillRec *UVg = reinterpret_cast<SpillRec *>(a.scratch) + base;
    uint8_t *UVm = reinterpret_cast<uint8_t *>(a.scratch + 4 * a.side.nnz) + base;  // chunk nonzero masks

    for (int kk = tid; kk < r; kk += NT) xs[kk] = moving[j * rp + a.perm_in[kk]];

    // chunk masks of this thread's resident entries (each thread writes and
    // reads only its own words): all-zero slices of the fixed factor are not
    // gathered
    const int nchunks = (r + C - 1) / C;
    uint16_t *mwords = a.slice_words + 4 * base;  // 8 bytes of word space per entry of the slice
    const bool masked = a.fixed_mask != nullptr && a.slice_words != nullptr && 4 * cn >= (int64_t)nchunks * NT &&
                        nchunks <= SLICE_MASK_CHUNKS && NR + NS <= 16;
    if (masked) slice_masks_build(mwords, a.fixed_mask, a.side.idx + base, cn, nchunks);

    double u[NR], vi[NR];
    int off[NR];
#pragma unroll
    for (int e = 0; e < NR; ++e) {
        const int64_t i = tid + (int64_t)e * NT;
        if (i < cn) {
            const int64_t g = base + i;
            off[e] = gather_off(a, g);
            entry_init(a.t_in[t_index(a, g)], val[g], eps, u[e], vi[e]);
        } else {
            off[e] = -1;
            u[e] = vi[e] = 0.0;
        }
    }
    [[maybe_unused]] int offs_r[KLNMF_CL_OFF_SMEM ? 1 : NS];
    auto offs = [&](int e) -> int & {
        if constexpr (KLNMF_CL_OFF_SMEM) return Offs[e * NT + tid];
        else return offs_r[e];
    };
#pragma unroll
    for (int e = 0; e < NS; ++e) {
        const int64_t i = tid + (int64_t)(NR + e) * NT;
        const int si = e * NT + tid;
        if (i < cn) {
            const int64_t g = base + i;
            offs(e) = gather_off(a, g);
            entry_init(a.t_in[t_index(a, g)], val[g], eps, Us[si], VIs[si]);
        } else {
            offs(e) = -1;
            Us[si] = VIs[si] = 0.0;
        }
    }
    const int64_t spill0 = (int64_t)(NR + NS) * NT;  // first spilled local entry
    for (int64_t i = spill0 + tid; i < cn; i += NT) {
        const int64_t g = base + i;
        double uu, vv;
        entry_init(a.t_in[t_index(a, g)], val[g], eps, uu, vv);
        kcheck(base + i < a.side.nnz, 8);
        UVg[i].uv = make_double2(uu, vv);
    }
    const unsigned cache_s = (unsigned)__cvta_generic_to_shared(cache) + 16u * tid;
    constexpr bool counter = CTR;
    if (counter && tid == 0) chunk_order(a.order_seed, *a.order_iter, (uint32_t)j, a.order_side, nchunks, cord);
    __syncthreads();
    ph.mark(0);

    Counters cnt;
    int buf = 0, cur = 0;
    // this chunk's mask word, loaded one chunk ahead
    unsigned mnext = masked ? (unsigned)mwords[(counter ? (int)cord[0] : 0) * NT + tid] : 0xffffu;
    for (int ch = 0; ch < nchunks; ++ch) {
        ph.count(11);
        const int pc = counter ? (int)cord[ch] : ch;  // physical chunk
        const unsigned mw = mnext;
        if (masked && ch + 1 < nchunks) mnext = (unsigned)mwords[(counter ? (int)cord[ch + 1] : ch + 1) * NT + tid];
        // gather this chunk of every resident entry once (own slots only);
        // entries whose row is all zero in this chunk are zero-filled without a request
#pragma unroll
        for (int e = 0; e < NR; ++e)
            if (e < ne)
                cp_async16(cache_s + 16u * NT * e, fixed + max(off[e], 0) + pc * C, off[e] >= 0 && ((mw >> e) & 1u));
#pragma unroll
        for (int e = 0; e < NS; ++e)
            if (NR + e < ne)
                cp_async16(cache_s + 16u * NT * (NR + e), fixed + max(offs(e), 0) + pc * C,
                           offs(e) >= 0 && ((mw >> (NR + e)) & 1u));
        cp_commit();
#ifdef KLNMF_CHECKED  // a skipped chunk really is all zero (code 11)
        if (masked) {
            for (int e = 0; e < NR + NS; ++e) {
                const int64_t i = tid + (int64_t)e * NT;
                if (e < ne && i < cn && !((mw >> e) & 1u)) {
                    const float4 z = ldg_f4(fixed + (int64_t)a.side.idx[base + i] * rp + pc * C);
                    kcheck(z.x == 0.f && z.y == 0.f && z.z == 0.f && z.w == 0.f, 11);
                }
            }
        }
#endif
        // spilled entries: stage the chunk's slice next to their state
        // (each thread stages and later reads only its own records)
        if (cn > spill0)
            spill_stage(UVg, UVm, spill0 + tid, cn, NT, fixed, a.side.idx + base, a.side.n_fix, rp, pc);
        cp_wait<0>();
        ph.mark(1);
        const float4 *A = cache + tid;
        const int nc = counter ? C : min(C, r - pc * C);
        const uint32_t perm = counter ? chunk_perm4(a.order_seed, *a.order_iter, (uint32_t)j, a.order_side, ch)
                                      : PERM4_IDENTITY;
        bool fresh = false;
#pragma unroll 1
        for (int cc = 0; cc < nc; ++cc) {
            const int q = (int)((perm >> (2 * cc)) & 3u);  // chunk coordinate visited in slot cc
            const int tt = pc * C + q;
            if (counter && tt >= r) continue;  // counter order: padding slot of the last chunk
            if (!fresh) {  // uniform over the group
                double red[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i) red[i] = 0.0;
                with_cc(counter ? 0 : cc, [&](auto ccv) {
                    constexpr int CC = decltype(ccv)::value;
#pragma unroll
                    for (int e = 0; e < NR; ++e)
                        if (e < ne) accum_from<CC>(red, A[e * NT], u[e], entry_z(u[e], vi[e]));
#pragma unroll
                    for (int e = 0; e < NS; ++e) {
                        if (NR + e >= ne) break;
                        const double uu = Us[e * NT + tid];
                        accum_from<CC>(red, A[(NR + e) * NT], uu, entry_z(uu, VIs[e * NT + tid]));
                    }
                });
                if (cn > spill0) {  // CTA-uniform
                    P8 acc;
#pragma unroll
                    for (int i = 0; i < NV; ++i) acc.v[i] = red[i];
                    acc = spill_pass(UVg, UVm, spill0 + tid, cn, NT, counter ? 0 : cc, acc);
#pragma unroll
                    for (int i = 0; i < NV; ++i) red[i] = acc.v[i];
                }
                ph.mark(2);
                reduce(red, buf);
                ph.mark(ch == 0 && cc == 0 ? 12 : 3);  // a job's first reduction also waits for its partners
                ph.count(8);
                cur = buf;
                buf ^= 1;
                fresh = true;
            }
            double x = (double)xs[tt];
            const double sb = ssum[tt] + pm.beta;
            double g = (sb + pm.alpha * x) - R.tot[cur][q];
            double h = pm.alpha + R.tot[cur][C + q];
            int inner = 0;
            bool active = enters(g, x, pm.eps_grad);
            bool moved = false;
            while (active) {  // uniform over the group
                bool again = false;
                const double delta = newton_step(g, h, x, inner, active, again, pm, cnt);
                ph.mark(4);
                const bool upd = delta != 0.0;  // uniform over the group
                if (upd) moved = true;
                double g2 = 0.0, h2 = 0.0;
                // apply the move and, if the loop continues, re-evaluate this coordinate
                if (upd || again) {
                    with_clamp(delta < 0.0, [&](auto cl) {
                        constexpr bool CL = decltype(cl)::value;
#pragma unroll
                        for (int e = 0; e < NR; ++e) {  // register entries: branch-free
                            if (e >= ne) break;
                            const double av = widen(comp(A + e * NT, q));
                            if (upd) entry_update<CL>(delta, av, eps, u[e], vi[e]);
                            if (again) accum(g2, h2, u[e], entry_z(u[e], vi[e]), av);
                        }
#pragma unroll
                        for (int e = 0; e < NS; ++e) {
                            if (NR + e >= ne) break;
                            const int si = e * NT + tid;
                            const double av = widen(comp(A + (NR + e) * NT, q));
                            double uu = Us[si];
                            const double vv = VIs[si];
                            if (upd) {
                                entry_update<CL>(delta, av, eps, uu, vv);
                                Us[si] = uu;
                            }
                            if (again) accum(g2, h2, uu, entry_z(uu, vv), av);
                        }
                        if (cn > spill0) {  // CTA-uniform
                            const P2 acc = spill_move(UVg, UVm, spill0 + tid, cn, NT, q, delta, upd, again, CL, eps,
                                                      P2{g2, h2});
                            g2 = acc.g;
                            h2 = acc.h;
                        }
                    });
                    ph.mark(5);
                    if (upd) ph.count(10);
                }
                if (again) {
                    double ev[NV] = {g2, h2};
                    reduce(ev, buf);
                    ph.mark(6);
                    ph.count(9);
                    g = (sb + pm.alpha * x) - R.tot[buf][0];
                    h = pm.alpha + R.tot[buf][1];
                    buf ^= 1;
                    active = enters(g, x, pm.eps_grad);
                    moved = true;  // the chunk sums' buffer may be recycled: re-pass next
                }
            }
            if (moved) fresh = false;
            if (tid == 0) xo[tt] = (float)x;
            ph.mark(4);
        }
    }
    __syncthreads();
    if (cq == 0)
        for (int kk = tid; kk < r; kk += NT) put_moving(a, moving, j * rp + a.perm_out[kk], xo[kk]);
#pragma unroll
    for (int e = 0; e < NR; ++e)
        if (off[e] >= 0) put_t(a, base + tid + (int64_t)e * NT, entry_t(u[e], vi[e], eps));
#pragma unroll
    for (int e = 0; e < NS; ++e)
        if (offs(e) >= 0)
            put_t(a, base + tid + (int64_t)(NR + e) * NT, entry_t(Us[e * NT + tid], VIs[e * NT + tid], eps));
    for (int64_t i = spill0 + tid; i < cn; i += NT) {
        const double2 uv = UVg[i].uv;
        put_t(a, base + i, entry_t(uv.x, uv.y, eps));
    }
    peer_fence(a);
    flush_stats(cnt, cq == 0 && tid == 0, a.stats, false);
    ph.mark(7);
    ph.flush(std::is_same<Reducer, CoopReducer>::value ? 1 : 0, threadIdx.x == 0);
}

template <bool CTR>
__global__ void __launch_bounds__(CL_NT, CL_PER_SM) solve_cluster_kernel(const klnmf_solve_args_t a) {
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.num_blocks();
    const int cq = (int)cl.block_rank();
    const int64_t slot = blockIdx.x / k;
    if (slot >= a.n_items) return;  // uniform over the cluster
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ GroupRed R;
    __shared__ ClusterInbox P;
    __shared__ double ssum[KMAX_RP];
    for (int kk = threadIdx.x; kk < a.r; kk += CL_NT) ssum[kk] = a.sum_pos[kk];
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&P.mbar[0]), 1);
        mbar_init(smem_u32(&P.mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (k > 1) cl.sync();  // every inbox is initialised before the first push
    else __syncthreads();
    ClusterReducer red{R, P, k, cq, 0u};
    solve_slice<CTR>(a, slot, cq, k, red, R, smem_raw, ssum);
    if (k > 1) cl.sync();  // no CTA exits while a peer may still address it
}

// schedule: [n_waves][gridDim.x] int4 (item slot or -1, rank, G, group id);
// sync: per group, [2][NV][CL_MAXG] tagged 16-byte reduction slots, then a
// 128-byte line holding the arrival counter (CoopReducer).
// A row group's waits only point to rows of the same or an earlier wave and
// every CTA is resident (cooperative launch), so the schedule cannot deadlock.

template <bool CTR>
__global__ void __launch_bounds__(CL_NT, CL_PER_SM) solve_coop_kernel(const klnmf_solve_args_t a, const int4 *schedule,
                                                              int n_waves, unsigned char *sync) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ GroupRed R;
    __shared__ double ssum[KMAX_RP];
    for (int kk = threadIdx.x; kk < a.r; kk += CL_NT) ssum[kk] = a.sum_pos[kk];
    for (int wv = 0; wv < n_waves; ++wv) {
        const int4 job = schedule[(size_t)wv * gridDim.x + blockIdx.x];
        if (job.x < 0) continue;
        unsigned char *gb = sync + (size_t)job.w * COOP_GROUP_BYTES;
        CoopReducer red{R, reinterpret_cast<unsigned long long *>(gb),
                        reinterpret_cast<unsigned *>(gb + COOP_GROUP_BYTES - 128), job.z, job.y, 0u};
        __syncthreads();  // shared buffers of the previous row are no longer read
        solve_slice<CTR>(a, job.x, job.y, job.z, red, R, smem_raw, ssum);
    }
}

struct FastKernel {
    int lanes, npl, nt;
    int64_t capacity;  // -1 = unbounded
    void (*fn)(const klnmf_solve_args_t);      // shared coordinate order
    void (*fn_ctr)(const klnmf_solve_args_t);  // counter coordinate order
    int gpb;           // subproblems per block
    int ring_entries;  // float4 ring slots per thread and stage (NPL)
    int cluster;       // CTAs per subproblem (cluster kernel), 0 = plain launch, -1 = cooperative
    bool roff_smem;    // gather offsets in shared memory (warp_roff_smem)
};

#define WK(L, NPL) \
    {L, NPL, WARP_NT, (int64_t)(L) * (NPL), solve_warp_kernel<L, NPL, false>, solve_warp_kernel<L, NPL, true>, WARP_NT / (L), NPL, 0, \
     warp_roff_smem(NPL)}
#define BK(NT, NPL) \
    {NT, NPL, NT, (int64_t)(NT) * (NPL), solve_block_kernel<NT, NPL, false>, solve_block_kernel<NT, NPL, true>, 1, NPL, 0, \
     block_roff_smem(NT, NPL)}
#define CK(K) \
    {CL_NT * (K), CL_NE, CL_NT, (int64_t)(K) * CL_NT * CL_NE, solve_cluster_kernel<false>, solve_cluster_kernel<true>, 1, 0, (K), false}
// Ascending capacity.  Every padding slot of a subproblem costs as much as a
// real entry, so the ladder is dense (<= 25% steps) where the F side's and the
// W side's subproblem sizes concentrate (SURVEY.md §8(d) size profiles).
const FastKernel kFast[] = {
    WK(1, 4),   WK(2, 4),   WK(4, 4),   WK(8, 4),   WK(8, 6),   WK(8, 8),   WK(16, 6),  WK(16, 8),
    WK(32, 5),  WK(32, 6),  WK(32, 7),  WK(32, 8),  WK(32, 10), WK(32, 12), WK(32, 14), WK(32, 16),
    BK(64, 10), BK(64, 12), BK(64, 14), BK(64, 16), BK(128, 10), BK(128, 12), BK(128, 14), BK(128, 16),
    BK(256, 10), BK(256, 12), BK(256, 14), BK(256, 16),
    // clusters of every width up to 8, then steps of 2: the W side's long
    // rows spread evenly over (4096, 65536], and a cluster bucket spanning a
    // factor of 2 left 30% of its slots empty
    CK(2),      CK(3),      CK(4),      CK(5),      CK(6),      CK(7),      CK(8),      CK(10),
    CK(12),     CK(14),     CK(16),
    // unbounded: the cooperative long-row kernel (klnmf_solve_coop, schedule built by the caller)
    {CL_NT, CL_NE, CL_NT, -1, nullptr, nullptr, 1, 0, -1, false},
};
#undef WK
#undef BK
#undef CK
constexpr int kNumFast = sizeof(kFast) / sizeof(kFast[0]);

inline size_t slice_smem(int rp) {
    return (size_t)CL_NE * CL_NT * sizeof(float4) + (size_t)CL_NS * CL_NT * 2 * sizeof(double) +
           (KLNMF_CL_OFF_SMEM ? (size_t)CL_NS * CL_NT * sizeof(int) : 0) + 2 * sizeof(float) * (size_t)(rp | 1) +
           MAX_CHUNKS + 16;
}

}  // namespace
}  // namespace klnmf

#ifdef KLNMF_CHECKED
// checked build only: (violations, first violation code); optionally cleared
extern "C" int klnmf_debug_checks(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, klnmf::g_check, sizeof(klnmf::g_check)) != cudaSuccess) return 1;
    if (reset) {
        static const unsigned long long zero[2] = {0, 0};
        if (cudaMemcpyToSymbol(klnmf::g_check, zero, sizeof(zero)) != cudaSuccess) return 1;
    }
    return 0;
}
#endif

#ifdef KLNMF_PHASE_TIMING
// diagnostic build only: copies out (and optionally clears) the phase counters
extern "C" int klnmf_debug_phase(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, klnmf::g_phase, sizeof(klnmf::g_phase)) != cudaSuccess) return 1;
    if (reset) {
        static const unsigned long long zero[4][16] = {};
        if (cudaMemcpyToSymbol(klnmf::g_phase, zero, sizeof(zero)) != cudaSuccess) return 1;
    }
    return 0;
}
#endif

using namespace klnmf;

extern "C" int klnmf_fast_kernel_count(void) { return kNumFast; }

// Dynamic shared memory of a bucket kernel at padded rank rp (counter order:
// the larger layout); the plan drops kernels that exceed the device limit.
// Dynamic shared memory above which a launch opts in to the large carve-out:
// static + dynamic must stay within 48 KB without it, and the kernels' static
// shared memory (row sums, visit map, per-group sums) reaches ~11 KB.
constexpr size_t SMEM_OPTIN = 32 * 1024;

// cudaFuncAttributeNonPortableClusterSizeAllowed once per kernel function.
static cudaError_t ensure_nonportable(const void *fn) {
    static const void *done[8] = {};
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    for (const void *d : done)
        if (d == fn) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess)
        for (auto &d : done)
            if (!d) {
                d = fn;
                break;
            }
    return e;
}

static size_t fast_kernel_smem(const FastKernel &k, int32_t rp) {
    if (k.cluster != 0) return slice_smem(rp);
    return sizeof(float4) * (size_t)ring_stages(k.ring_entries) * (size_t)k.ring_entries * (size_t)k.nt +
           (k.roff_smem ? sizeof(int) * (size_t)k.ring_entries * (size_t)k.nt : 0) +
           2 * sizeof(float) * (size_t)k.gpb * (size_t)(rp | 1) + (size_t)k.gpb * MAX_CHUNKS + 16;
}

extern "C" int klnmf_fast_kernel_fits(int kernel_id, int32_t rp, int32_t *fits) {
    if (kernel_id < 0 || kernel_id >= kNumFast) return set_error_msg(1, "klnmf_fast_kernel_fits: bad kernel id");
    int dev = 0, lim = 0;
    KLNMF_CHECK(cudaGetDevice(&dev));
    KLNMF_CHECK(cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    *fits = (rp % 4 == 0 && rp <= KMAX_RP && fast_kernel_smem(kFast[kernel_id], rp) + 8 * 1024 <= (size_t)lim) ? 1 : 0;
    return 0;
}

extern "C" int klnmf_fast_kernel_info(int kernel_id, int64_t *capacity, int32_t *lanes, int32_t *npl) {
    if (kernel_id < 0 || kernel_id >= kNumFast) return set_error_msg(1, "klnmf_fast_kernel_info: bad kernel id");
    *capacity = kFast[kernel_id].capacity;
    *lanes = kFast[kernel_id].lanes;
    *npl = kFast[kernel_id].npl;
    return 0;
}

// Sets every fp32 kernel's launch attributes (dynamic shared memory for the
// larger, counter-order layout; non-portable cluster sizes), both coordinate
// orders, for padded rank rp, so that later launches -- in particular inside
// CUDA-graph capture -- issue no attribute calls.
extern "C" int klnmf_prepare_fast(int32_t rp) {
    if (rp % 4 != 0 || rp > KMAX_RP) return set_error_msg(1, "klnmf_prepare_fast: bad padded rank");
    cudaFuncAttributes fa;
    KLNMF_CHECK(cudaFuncGetAttributes(&fa, (const void *)solve_coop_kernel<false>));  // loads the module now
    int dev = 0, lim = 0;
    KLNMF_CHECK(cudaGetDevice(&dev));
    KLNMF_CHECK(cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    for (int id = 0; id < kNumFast; ++id) {
        const FastKernel &k = kFast[id];
        if (fast_kernel_smem(k, rp) + 8 * 1024 > (size_t)lim) continue;  // not used at this rank
        if (k.cluster < 0) {
            KLNMF_CHECK(ensure_smem((const void *)solve_coop_kernel<false>, slice_smem(rp)));
            KLNMF_CHECK(ensure_smem((const void *)solve_coop_kernel<true>, slice_smem(rp)));
#if defined(KLNMF_CARVEOUT) && KLNMF_CARVEOUT >= 0
            KLNMF_CHECK(cudaFuncSetAttribute((const void *)solve_coop_kernel<false>,
                                             cudaFuncAttributePreferredSharedMemoryCarveout, KLNMF_CARVEOUT));
            KLNMF_CHECK(cudaFuncSetAttribute((const void *)solve_coop_kernel<true>,
                                             cudaFuncAttributePreferredSharedMemoryCarveout, KLNMF_CARVEOUT));
#endif
            continue;
        }
        for (auto fn : {k.fn, k.fn_ctr}) {
            KLNMF_CHECK(cudaFuncGetAttributes(&fa, (const void *)fn));
#if defined(KLNMF_CARVEOUT) && KLNMF_CARVEOUT >= 0
            KLNMF_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, KLNMF_CARVEOUT));
#endif
            if (k.cluster > 0) {
                KLNMF_CHECK(ensure_smem((const void *)fn, slice_smem(rp)));
                if (k.cluster > 8)
                    KLNMF_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            } else {
                const size_t smem = fast_kernel_smem(k, rp);
                if (smem > SMEM_OPTIN) KLNMF_CHECK(ensure_smem((const void *)fn, smem));
            }
        }
    }
    return 0;
}

extern "C" int klnmf_solve_fast(const klnmf_solve_args_t *args, int kernel_id, void *stream) {
    if (kernel_id < 0 || kernel_id >= kNumFast) return set_error_msg(1, "klnmf_solve_fast: bad kernel id");
    if (args->n_items <= 0) return 0;
    if (args->rp % 4 != 0) return set_error_msg(1, "klnmf_solve_fast: rp must be a multiple of 4");
    if (args->rp > KMAX_RP) return set_error_msg(1, "klnmf_solve_fast: rank above 256 is not supported in fp32 mode");
    if (args->order_mode != KLNMF_ORDER_SHARED && (args->order_mode != KLNMF_ORDER_COUNTER || !args->order_iter))
        return set_error_msg(1, "klnmf_solve_fast: bad coordinate order mode");
    if (!(args->eps_div > 0.0)) return set_error_msg(1, "klnmf_solve_fast: the fp32 mode needs eps_div > 0");
    // the gather offsets of the fixed factor are 32-bit (register budget)
    if (args->side.n_fix * (int64_t)args->rp >= (int64_t)INT32_MAX)
        return set_error_msg(1, "klnmf_solve_fast: fixed-factor items x padded rank must be < 2^31 in the fp32 mode");
    if (args->n_peers < 0 || (args->n_peers > 0 && (!args->peer_moving || !args->peer_t)))
        return set_error_msg(1, "klnmf_solve_fast: n_peers > 0 needs both peer pointer arrays");
    const FastKernel &k = kFast[kernel_id];
    if (k.cluster < 0) return set_error_msg(1, "klnmf_solve_fast: the long-row bucket runs through klnmf_solve_coop");
    void (*fn)(const klnmf_solve_args_t) = args->order_mode == KLNMF_ORDER_SHARED ? k.fn : k.fn_ctr;
    if (k.cluster > 0) {
        if (args->scratch == nullptr)
            return set_error_msg(1, "klnmf_solve_fast: the cluster kernel needs a scratch buffer");
        const size_t smem = slice_smem(args->rp);
        KLNMF_CHECK(ensure_smem((const void *)fn, smem));
        if (k.cluster > 8) KLNMF_CHECK(ensure_nonportable((const void *)fn));
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
        KLNMF_CHECK(cudaLaunchKernelEx(&cfg, fn, *args));
        return 0;
    }
    const int64_t blocks = (args->n_items + k.gpb - 1) / k.gpb;
    const size_t ring = sizeof(float4) * (size_t)ring_stages(k.ring_entries) * (size_t)k.ring_entries * (size_t)k.nt +
                        (k.roff_smem ? sizeof(int) * (size_t)k.ring_entries * (size_t)k.nt : 0);
    const size_t smem = ring + 2 * sizeof(float) * (size_t)k.gpb * (size_t)(args->rp | 1) +
                        (args->order_mode != KLNMF_ORDER_SHARED ? (size_t)k.gpb * MAX_CHUNKS : 0) + 16;
    if (smem > SMEM_OPTIN) KLNMF_CHECK(ensure_smem((const void *)fn, smem));
    fn<<<(unsigned)blocks, k.nt, smem, as_stream(stream)>>>(*args);
    KLNMF_CHECK_LAUNCH("klnmf_solve_fast");
    return 0;
}

extern "C" int klnmf_coop_info(int32_t rp, int64_t *entries_per_cta, int32_t *n_ctas, int64_t *sync_bytes_per_group) {
    const size_t smem = slice_smem(rp);
    KLNMF_CHECK(ensure_smem((const void *)solve_coop_kernel<false>, smem));
    KLNMF_CHECK(ensure_smem((const void *)solve_coop_kernel<true>, smem));
    int dev = 0, sms = 0, per_sm = 0;
    KLNMF_CHECK(cudaGetDevice(&dev));
    KLNMF_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    KLNMF_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_coop_kernel<false>, CL_NT, smem));
    *entries_per_cta = (int64_t)CL_NT * CL_NE;
    *n_ctas = sms * per_sm < CL_MAXG ? sms * per_sm : CL_MAXG;
    *sync_bytes_per_group = (int64_t)COOP_GROUP_BYTES;
    return 0;
}

extern "C" int klnmf_solve_coop(const klnmf_solve_args_t *args, const void *schedule, int32_t n_waves,
                                int32_t n_ctas, void *sync, int64_t n_groups, void *stream) {
    if (n_waves <= 0 || args->n_items <= 0) return 0;
    if (args->rp > KMAX_RP) return set_error_msg(1, "klnmf_solve_coop: rank above 256 is not supported");
    if (args->scratch == nullptr) return set_error_msg(1, "klnmf_solve_coop: needs a scratch buffer");
    if (args->order_mode != KLNMF_ORDER_SHARED && (args->order_mode != KLNMF_ORDER_COUNTER || !args->order_iter))
        return set_error_msg(1, "klnmf_solve_coop: bad coordinate order mode");
    if (!(args->eps_div > 0.0)) return set_error_msg(1, "klnmf_solve_coop: the fp32 mode needs eps_div > 0");
    // the gather offsets of the fixed factor are 32-bit (register budget)
    if (args->side.n_fix * (int64_t)args->rp >= (int64_t)INT32_MAX)
        return set_error_msg(1, "klnmf_solve_coop: fixed-factor items x padded rank must be < 2^31 in the fp32 mode");
    if (args->n_peers < 0 || (args->n_peers > 0 && (!args->peer_moving || !args->peer_t)))
        return set_error_msg(1, "klnmf_solve_coop: n_peers > 0 needs both peer pointer arrays");
    cudaStream_t st = as_stream(stream);
    const size_t smem = slice_smem(args->rp);
    const void *fn = args->order_mode == KLNMF_ORDER_SHARED ? (const void *)solve_coop_kernel<false>
                                                            : (const void *)solve_coop_kernel<true>;
    KLNMF_CHECK(ensure_smem(fn, smem));
    KLNMF_CHECK(cudaMemsetAsync(sync, 0, (size_t)n_groups * COOP_GROUP_BYTES, st));  // tag 0: empty
    klnmf_solve_args_t a = *args;
    const int4 *sched = static_cast<const int4 *>(schedule);
    unsigned char *sy = static_cast<unsigned char *>(sync);
    int nw = n_waves;
    void *kargs[] = {&a, &sched, &nw, &sy};
    KLNMF_CHECK(cudaLaunchCooperativeKernel(fn, dim3((unsigned)n_ctas), dim3(CL_NT),
                                            kargs, smem, st));
    return 0;
}
