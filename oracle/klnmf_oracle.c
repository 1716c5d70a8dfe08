/*
 * klnmf_oracle.c -- CPU restatement of the reference SRCD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product (paper_1604_04026_b200)
 * never links, imports or calls it; there is no CPU fallback.
 *
 * Every function restates one numba kernel of the reference package
 * (klnmf, /root/reference/pkg/src/klnmf) with the same operation order:
 * numba emits no FMA and no fast-math (SURVEY.md finding 3), so this file is
 * compiled with -ffp-contract=off and without -ffast-math, and the results
 * are bit-identical to the reference (pinned by tests/test_oracle_golden.py
 * against fixtures generated from the reference itself).
 *
 *   oracle_sweep_range_dense    _kernels.py:123-144 (+ solve_column :53-120,
 *                               _grad_hess :24-36, compute_ax :39-50), with the
 *                               reference's dense length-n_fix maintained product
 *   oracle_sweep_range_support  the same algorithm with the maintained product
 *                               kept only on the column's support S (bitwise
 *                               identical: every ax[i] evolves independently and
 *                               is only read at S -- SURVEY.md finding 2)
 *   oracle_sweep                the reference's sweep() thread pool
 *                               (solver.py:165-216), columns handed out in blocks
 *   oracle_sweep_cols_timed     sweep_range on a column sample with per-column
 *                               thread CPU times (bench.py's CPU baseline)
 *   oracle_kl_data_term         _kernels.py:147-160
 *   oracle_row_sums             DenseFactor.row_sums (sparse.py:194-196) =
 *                               numpy's pairwise summation (SURVEY.md finding 8)
 *   oracle_sweep_fp32           the fp32-storage / fp64-arithmetic mode of the
 *                               CUDA path, restated on
 *                               the device layout so sampled subproblems can be
 *                               compared one by one at full problem sizes
 */
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define STAT_CAP_HITS 0   /* _kernels.py:17 */
#define STAT_DEGENERATE 1 /* _kernels.py:18 */
#define STAT_INNER_ITERS 2/* _kernels.py:19 */
#define STAT_PASSES 3     /* _kernels.py:20 */

/* ------------------------------------------------------------------ */
/* _grad_hess, _kernels.py:24-36.  ax is indexed by row (dense) or by the
 * position p inside the column (support variant, ax_is_local != 0).      */
static inline void grad_hess(int64_t k, const int64_t *v_idx, const double *v_val, int64_t s,
                             const double *at, int64_t n_fix, const double *ax, int ax_is_local,
                             const double *sum_a, double x_k, double alpha, double beta,
                             double eps_div, double *g_out, double *h_out) {
    double g = sum_a[k] + alpha * x_k + beta;
    double h = alpha;
    const double *row = at + k * n_fix;
    for (int64_t p = 0; p < s; ++p) {
        double a = row[v_idx[p]];
        if (a != 0.0) {
            double q = a / (ax[ax_is_local ? p : v_idx[p]] + eps_div);
            g -= v_val[p] * q;
            h += v_val[p] * q * q;
        }
    }
    *g_out = g;
    *h_out = h;
}

/* compute_ax, _kernels.py:39-50: natural k order, exact zeros of x skipped. */
static void compute_ax_dense(const double *at, int64_t r, int64_t n_fix, const double *x, double *ax) {
    for (int64_t i = 0; i < n_fix; ++i) ax[i] = 0.0;
    for (int64_t k = 0; k < r; ++k) {
        double xk = x[k];
        if (xk != 0.0) {
            const double *row = at + k * n_fix;
            for (int64_t i = 0; i < n_fix; ++i) ax[i] += xk * row[i];
        }
    }
}

static void compute_ax_support(const double *at, int64_t r, int64_t n_fix, const double *x,
                               const int64_t *v_idx, int64_t s, double *t) {
    for (int64_t p = 0; p < s; ++p) t[p] = 0.0;
    for (int64_t k = 0; k < r; ++k) {
        double xk = x[k];
        if (xk != 0.0) {
            const double *row = at + k * n_fix;
            for (int64_t p = 0; p < s; ++p) t[p] += xk * row[v_idx[p]];
        }
    }
}

/* ax += delta * at[k], clamped at 0: _kernels.py:86-90 and :103-106. */
static inline void update_ax(const double *at, int64_t k, int64_t n_fix, double delta, double *ax,
                             int local, const int64_t *v_idx, int64_t s) {
    const double *row = at + k * n_fix;
    if (!local) {
        for (int64_t i = 0; i < n_fix; ++i) {
            ax[i] += delta * row[i];
            if (ax[i] < 0.0) ax[i] = 0.0;
        }
    } else {
        for (int64_t p = 0; p < s; ++p) {
            ax[p] += delta * row[v_idx[p]];
            if (ax[p] < 0.0) ax[p] = 0.0;
        }
    }
}

/* solve_column, _kernels.py:53-120 (max_passes as in the reference). */
void oracle_solve_column(const int64_t *v_idx, const double *v_val, int64_t s, const double *at,
                         int64_t r, int64_t n_fix, const double *sum_a, double *x, double *ax,
                         int local, const int64_t *ids, double alpha, double beta, double eps_grad,
                         double eps_x, double eps_div, int64_t inner_cap, int64_t max_passes,
                         int64_t *stats) {
    if (local)
        compute_ax_support(at, r, n_fix, x, v_idx, s, ax);
    else
        compute_ax_dense(at, r, n_fix, x, ax);
    for (int64_t pass = 0; pass < max_passes; ++pass) {
        stats[STAT_PASSES] += 1;
        int moved = 0;
        for (int64_t tt = 0; tt < r; ++tt) {
            int64_t k = ids[tt];
            double x_enter = x[k];
            double g, h;
            grad_hess(k, v_idx, v_val, s, at, n_fix, ax, local, sum_a, x[k], alpha, beta, eps_div, &g, &h);
            int64_t inner = 0;
            while ((g < -eps_grad) || (fabs(g) > eps_grad && x[k] > eps_grad)) {
                if (h <= 0.0) {
                    if (g > 0.0) {
                        double delta = -x[k];
                        if (delta != 0.0) {
                            update_ax(at, k, n_fix, delta, ax, local, v_idx, s);
                            x[k] = 0.0;
                        }
                    } else {
                        stats[STAT_DEGENERATE] += 1;
                    }
                    break;
                }
                double target = x[k] - g / h;
                if (target < 0.0) target = 0.0;
                double delta = target - x[k];
                update_ax(at, k, n_fix, delta, ax, local, v_idx, s);
                double xs = x[k];
                x[k] = xs + delta;
                inner += 1;
                stats[STAT_INNER_ITERS] += 1;
                if (fabs(delta) < eps_x * xs) break;
                if (inner >= inner_cap) {
                    stats[STAT_CAP_HITS] += 1;
                    break;
                }
                grad_hess(k, v_idx, v_val, s, at, n_fix, ax, local, sum_a, x[k], alpha, beta, eps_div, &g, &h);
            }
            if (x[k] != x_enter) moved = 1;
        }
        if (!moved) break;
    }
}

/* sweep_range, _kernels.py:123-144 (one pass per column).  at is (r, n_fix)
 * C-order, moving is (r, n_mov) C-order, both fp64 -- the reference layout.
 * ax_buf has n_fix entries (dense) or max column nnz entries (support).   */
static void sweep_range_impl(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                             const double *at, int64_t r, int64_t n_fix, const double *sum_a,
                             double *moving, int64_t n_mov, int64_t j_lo, int64_t j_hi,
                             const int64_t *ids, double alpha, double beta, double eps_grad,
                             double eps_x, double eps_div, int64_t inner_cap, double *ax_buf,
                             double *x_buf, int64_t *stats, int local) {
    for (int64_t j = j_lo; j < j_hi; ++j) {
        for (int64_t k = 0; k < r; ++k) x_buf[k] = moving[k * n_mov + j];
        int64_t lo = col_ptr[j], hi = col_ptr[j + 1];
        oracle_solve_column(row_idx + lo, values + lo, hi - lo, at, r, n_fix, sum_a, x_buf, ax_buf,
                            local, ids, alpha, beta, eps_grad, eps_x, eps_div, inner_cap, 1, stats);
        for (int64_t k = 0; k < r; ++k) moving[k * n_mov + j] = x_buf[k];
    }
}

void oracle_sweep_range_dense(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                              const double *at, int64_t r, int64_t n_fix, const double *sum_a,
                              double *moving, int64_t n_mov, int64_t j_lo, int64_t j_hi,
                              const int64_t *ids, double alpha, double beta, double eps_grad,
                              double eps_x, double eps_div, int64_t inner_cap, double *ax_buf,
                              double *x_buf, int64_t *stats) {
    sweep_range_impl(col_ptr, row_idx, values, at, r, n_fix, sum_a, moving, n_mov, j_lo, j_hi, ids,
                     alpha, beta, eps_grad, eps_x, eps_div, inner_cap, ax_buf, x_buf, stats, 0);
}

void oracle_sweep_range_support(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                                const double *at, int64_t r, int64_t n_fix, const double *sum_a,
                                double *moving, int64_t n_mov, int64_t j_lo, int64_t j_hi,
                                const int64_t *ids, double alpha, double beta, double eps_grad,
                                double eps_x, double eps_div, int64_t inner_cap, double *ax_buf,
                                double *x_buf, int64_t *stats) {
    sweep_range_impl(col_ptr, row_idx, values, at, r, n_fix, sum_a, moving, n_mov, j_lo, j_hi, ids,
                     alpha, beta, eps_grad, eps_x, eps_div, inner_cap, ax_buf, x_buf, stats, 1);
}

/* ------------------------------------------------------------------ */
/* sweep(), solver.py:165-216: the reference splits the columns into
 * equal-count chunks (_chunk_bounds, solver.py:160-162 = np.linspace(0, n,
 * workers+1).astype(int64)), one worker each, stats summed.  Results are
 * invariant to how columns are assigned; with several workers the oracle
 * hands out small column blocks dynamically (load balance on skewed sides). */
/* Columns are independent and each is written by exactly one worker, so
 * the result is identical for any assignment of columns to workers.  The
 * reference's equal-count chunks leave one worker with all of a Zipf head's
 * long rows (the W side of C3-C5 is essentially serial then), so workers
 * here claim blocks of columns from a shared counter instead; `next` is
 * NULL for the static equal-count chunk [j_lo, j_hi). */
#define DYN_BLOCK 8
typedef struct {
    const int64_t *col_ptr, *row_idx;
    const double *values, *at, *sum_a;
    double *moving;
    const int64_t *ids;
    int64_t r, n_fix, n_mov, j_lo, j_hi, inner_cap, scratch;
    double alpha, beta, eps_grad, eps_x, eps_div;
    int local;
    int64_t *next;
    int64_t stats[4];
} sweep_task_t;

static void *sweep_worker(void *arg) {
    sweep_task_t *t = (sweep_task_t *)arg;
    double *ax = (double *)malloc(sizeof(double) * (size_t)(t->scratch > 0 ? t->scratch : 1));
    double *x = (double *)malloc(sizeof(double) * (size_t)t->r);
    if (!t->next) {
        sweep_range_impl(t->col_ptr, t->row_idx, t->values, t->at, t->r, t->n_fix, t->sum_a, t->moving,
                         t->n_mov, t->j_lo, t->j_hi, t->ids, t->alpha, t->beta, t->eps_grad, t->eps_x,
                         t->eps_div, t->inner_cap, ax, x, t->stats, t->local);
    } else {
        for (;;) {
            const int64_t a = __atomic_fetch_add(t->next, DYN_BLOCK, __ATOMIC_RELAXED);
            if (a >= t->n_mov) break;
            const int64_t b = a + DYN_BLOCK < t->n_mov ? a + DYN_BLOCK : t->n_mov;
            sweep_range_impl(t->col_ptr, t->row_idx, t->values, t->at, t->r, t->n_fix, t->sum_a, t->moving,
                             t->n_mov, a, b, t->ids, t->alpha, t->beta, t->eps_grad, t->eps_x, t->eps_div,
                             t->inner_cap, ax, x, t->stats, t->local);
        }
    }
    free(ax);
    free(x);
    return NULL;
}

int oracle_sweep(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                 const double *at, int64_t r, int64_t n_fix, const double *sum_a, double *moving,
                 int64_t n_mov, const int64_t *ids, double alpha, double beta, double eps_grad,
                 double eps_x, double eps_div, int64_t inner_cap, int n_workers, int local,
                 int64_t *stats_out) {
    if (n_workers < 1) n_workers = 1;
    int64_t max_s = 0;
    for (int64_t j = 0; j < n_mov; ++j) {
        int64_t s = col_ptr[j + 1] - col_ptr[j];
        if (s > max_s) max_s = s;
    }
    sweep_task_t *tasks = (sweep_task_t *)calloc((size_t)n_workers, sizeof(sweep_task_t));
    pthread_t *th = (pthread_t *)calloc((size_t)n_workers, sizeof(pthread_t));
    int n_tasks = 0;
    int64_t next = 0; /* dynamic column blocks (see sweep_task_t) */
    for (int w = 0; w < n_workers; ++w) {
        /* np.linspace(0, n, W+1).astype(int64): floor of w*n/W in fp64 */
        int64_t a = (int64_t)((double)n_mov * (double)w / (double)n_workers);
        int64_t b = (w + 1 == n_workers) ? n_mov : (int64_t)((double)n_mov * (double)(w + 1) / (double)n_workers);
        if (b <= a) continue;
        sweep_task_t *t = &tasks[n_tasks++];
        t->col_ptr = col_ptr; t->row_idx = row_idx; t->values = values; t->at = at; t->sum_a = sum_a;
        t->moving = moving; t->ids = ids; t->r = r; t->n_fix = n_fix; t->n_mov = n_mov;
        t->j_lo = a; t->j_hi = b; t->inner_cap = inner_cap; t->scratch = local ? max_s : n_fix;
        t->alpha = alpha; t->beta = beta; t->eps_grad = eps_grad; t->eps_x = eps_x; t->eps_div = eps_div;
        t->local = local;
        t->next = n_workers > 1 ? &next : NULL;
    }
    if (n_tasks == 1) {
        sweep_worker(&tasks[0]);
    } else {
        for (int i = 0; i < n_tasks; ++i) pthread_create(&th[i], NULL, sweep_worker, &tasks[i]);
        for (int i = 0; i < n_tasks; ++i) pthread_join(th[i], NULL);
    }
    for (int i = 0; i < n_tasks; ++i)
        for (int q = 0; q < 4; ++q) stats_out[q] += tasks[i].stats[q];
    free(tasks);
    free(th);
    return 0;
}

/* ------------------------------------------------------------------ */
/* CPU-baseline sampler (bench.py): sweep_range on an explicit list of
 * columns -- each solved exactly as sweep_range solves it, in place in
 * `moving` -- with the thread CPU time of every column recorded, so a
 * stratified sample extrapolates to a full half-step without depending on
 * how well a small sample fills the worker threads.  Workers claim columns
 * from a shared counter.                                                  */
#include <time.h>

typedef struct {
    const int64_t *col_ptr, *row_idx, *cols;
    const double *values, *at, *sum_a;
    double *moving, *col_seconds;
    const int64_t *ids;
    int64_t r, n_fix, n_mov, n_cols, inner_cap, scratch;
    double alpha, beta, eps_grad, eps_x, eps_div;
    int local;
    int64_t *next;
    int64_t stats[4];
} timed_task_t;

static double thread_seconds(void) {
    struct timespec ts;
    clock_gettime(CLOCK_THREAD_CPUTIME_ID, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void *timed_worker(void *arg) {
    timed_task_t *t = (timed_task_t *)arg;
    double *ax = (double *)malloc(sizeof(double) * (size_t)(t->scratch > 0 ? t->scratch : 1));
    double *x = (double *)malloc(sizeof(double) * (size_t)t->r);
    for (;;) {
        const int64_t q = __atomic_fetch_add(t->next, 1, __ATOMIC_RELAXED);
        if (q >= t->n_cols) break;
        const int64_t j = t->cols[q];
        const double t0 = thread_seconds();
        sweep_range_impl(t->col_ptr, t->row_idx, t->values, t->at, t->r, t->n_fix, t->sum_a, t->moving,
                         t->n_mov, j, j + 1, t->ids, t->alpha, t->beta, t->eps_grad, t->eps_x, t->eps_div,
                         t->inner_cap, ax, x, t->stats, t->local);
        t->col_seconds[q] = thread_seconds() - t0;
    }
    free(ax);
    free(x);
    return NULL;
}

int oracle_sweep_cols_timed(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                            const double *at, int64_t r, int64_t n_fix, const double *sum_a, double *moving,
                            int64_t n_mov, const int64_t *cols, int64_t n_cols, const int64_t *ids, double alpha,
                            double beta, double eps_grad, double eps_x, double eps_div, int64_t inner_cap,
                            int n_workers, int local, int64_t *stats_out, double *col_seconds) {
    if (n_workers < 1) n_workers = 1;
    int64_t max_s = 0;
    for (int64_t q = 0; q < n_cols; ++q) {
        const int64_t s = col_ptr[cols[q] + 1] - col_ptr[cols[q]];
        if (s > max_s) max_s = s;
    }
    timed_task_t *tasks = (timed_task_t *)calloc((size_t)n_workers, sizeof(timed_task_t));
    pthread_t *th = (pthread_t *)calloc((size_t)n_workers, sizeof(pthread_t));
    int64_t next = 0;
    for (int w = 0; w < n_workers; ++w) {
        timed_task_t *t = &tasks[w];
        t->col_ptr = col_ptr; t->row_idx = row_idx; t->cols = cols; t->values = values; t->at = at;
        t->sum_a = sum_a; t->moving = moving; t->col_seconds = col_seconds; t->ids = ids; t->r = r;
        t->n_fix = n_fix; t->n_mov = n_mov; t->n_cols = n_cols; t->inner_cap = inner_cap;
        t->scratch = local ? max_s : n_fix; t->alpha = alpha; t->beta = beta; t->eps_grad = eps_grad;
        t->eps_x = eps_x; t->eps_div = eps_div; t->local = local; t->next = &next;
    }
    for (int i = 0; i < n_workers; ++i) pthread_create(&th[i], NULL, timed_worker, &tasks[i]);
    for (int i = 0; i < n_workers; ++i) pthread_join(th[i], NULL);
    for (int i = 0; i < n_workers; ++i)
        for (int q = 0; q < 4; ++q) stats_out[q] += tasks[i].stats[q];
    free(tasks);
    free(th);
    return 0;
}

/* ------------------------------------------------------------------ */
/* kl_data_term, _kernels.py:147-160: serial over columns then nonzeros. */
double oracle_kl_data_term(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                           int64_t n_cols, const double *w, int64_t n_rows, const double *f,
                           int64_t r, double eps_div) {
    double total = 0.0;
    for (int64_t j = 0; j < n_cols; ++j) {
        for (int64_t p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
            int64_t i = row_idx[p];
            double d = 0.0;
            for (int64_t k = 0; k < r; ++k) d += w[k * n_rows + i] * f[k * n_cols + j];
            double v = values[p];
            total += v * log(v / (d + eps_div)) - v;
        }
    }
    return total;
}

/* numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), the algorithm
 * behind DenseFactor.row_sums (sparse.py:194-196); PW_BLOCKSIZE 128, 8-way
 * unrolled leaves.  Matches numpy 2.3 bit for bit (tests/test_oracle_golden). */
static double pairwise_sum(const double *a, int64_t n, int64_t stride) {
    if (n < 8) {
        double res = 0.;
        for (int64_t i = 0; i < n; ++i) res += a[i * stride];
        return res;
    } else if (n <= 128) {
        double r[8], res;
        int64_t i;
        for (int q = 0; q < 8; ++q) r[q] = a[q * stride];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int q = 0; q < 8; ++q) r[q] += a[(i + q) * stride];
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * stride];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2, stride) + pairwise_sum(a + n2 * stride, n - n2, stride);
    }
}

void oracle_row_sums(const double *factor, int64_t r, int64_t n, double *out) {
    for (int64_t k = 0; k < r; ++k) out[k] = pairwise_sum(factor + k * n, n, 1);
}

/* ------------------------------------------------------------------ */
/* fp32-storage mode: factors are fp32 values stored item-major
 * in visit order (row i of `fixed` is the r-vector of item i, column tt is the
 * coordinate visited tt-th), arithmetic is fp64, the maintained product t of
 * every stored entry is carried between half-steps, and each Newton step
 * rounds the coordinate to fp32 so t stays consistent with the stored factor.
 * Per entry the state is u = v/(t+eps) and vi = 1/v: the reference's
 * _grad_hess (_kernels.py:24-36) becomes g = sum_a + alpha*x + beta -
 * sum(u*a), h = alpha + sum(z*a*a) with z = u*u*vi, a move t' = t + delta*a
 * becomes u' = u/q with q = 1 + delta*a*u*vi (clamp t' < 0 -> 0 as
 * _kernels.py:105-106: q < eps*u*vi -> u' = v/eps), and t = 1/(u*vi) - eps
 * is written back at the end.  eps_div > 0.  The control flow is
 * solve_column's (_kernels.py:73-118) verbatim.                             */
/* fp32 storage value of a non-negative coordinate; subnormals are flushed to
 * zero (the device kernels widen stored values with integer arithmetic that
 * is exact for zero and normal floats only). */
/* kkt_violation, _kernels.py:176-190, for every column of x (r, n_mov):
 * out (r, n_mov).  compute_ax on the support (bitwise equal to the dense
 * product there, SURVEY.md finding 2). */
void oracle_kkt_violation(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                          const double *at, int64_t r, int64_t n_fix, const double *sum_a,
                          const double *x, int64_t n_mov, double alpha, double beta, double eps_grad,
                          double eps_x, double eps_div, double *out) {
    int64_t cap = 1;
    for (int64_t j = 0; j < n_mov; ++j)
        if (col_ptr[j + 1] - col_ptr[j] > cap) cap = col_ptr[j + 1] - col_ptr[j];
    double *t = (double *)malloc(sizeof(double) * (size_t)cap);
    double *xj = (double *)malloc(sizeof(double) * (size_t)r);
    for (int64_t j = 0; j < n_mov; ++j) {
        const int64_t lo = col_ptr[j], s = col_ptr[j + 1] - lo;
        for (int64_t k = 0; k < r; ++k) xj[k] = x[k * n_mov + j];
        compute_ax_support(at, r, n_fix, xj, row_idx + lo, s, t);
        for (int64_t k = 0; k < r; ++k) {
            double g, h;
            grad_hess(k, row_idx + lo, values + lo, s, at, n_fix, t, 1, sum_a, xj[k], alpha, beta, eps_div, &g,
                      &h);
            double v;
            if (xj[k] <= eps_grad) {
                v = -g - eps_grad;
            } else {
                double scale = eps_x * xj[k] * h;
                if (!(scale > eps_grad)) scale = eps_grad; /* max(eps_grad, scale) */
                v = fabs(g) - scale;
            }
            out[k * n_mov + j] = v > 0.0 ? v : 0.0; /* max(0.0, v) */
        }
    }
    free(t);
    free(xj);
}

/* mu_update_range, _kernels.py:193-214 (moving rescaled in place). */
void oracle_mu_update_range(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                            const double *fixed, double *moving, const double *sum_fixed, double eps_mu,
                            int64_t j_lo, int64_t j_hi, int64_t r, int64_t n_fix, int64_t n_mov) {
    double *num = (double *)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
    for (int64_t j = j_lo; j < j_hi; ++j) {
        for (int64_t k = 0; k < r; ++k) num[k] = 0.0;
        for (int64_t p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
            const int64_t i = row_idx[p];
            double d = 0.0;
            for (int64_t k = 0; k < r; ++k) d += fixed[k * n_fix + i] * moving[k * n_mov + j];
            const double ratio = values[p] / (d + eps_mu);
            for (int64_t k = 0; k < r; ++k) num[k] += fixed[k * n_fix + i] * ratio;
        }
        for (int64_t k = 0; k < r; ++k)
            moving[k * n_mov + j] = moving[k * n_mov + j] * (num[k] + eps_mu) / (sum_fixed[k] + eps_mu);
    }
    free(num);
}

/* ------------------------------------------------------------------ */
/* Counter-based coordinate order (north-star (c)).  Not part
 * of the reference: it replaces the reference's single ids permutation per
 * iteration (solver.py:276,287) by an order per (seed, iteration, subproblem,
 * side) that needs no host stream.  Generator: Philox4x32-10 (Salmon et al.,
 * SC'11, "Parallel random numbers: as easy as 1, 2, 3"), restated from the
 * published round function:
 *   (hi0, lo0) = mulhilo(0xD2511F53, c0); (hi1, lo1) = mulhilo(0xCD9E8D57, c2)
 *   c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);  k += (0x9E3779B9, 0xBB67AE85)
 * with the key bumped between the 10 rounds.                                  */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int rnd = 0; rnd < 10; ++rnd) {
        if (rnd > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* Visit order of the nchunks 4-coordinate chunks of subproblem `item`:
 * Fisher-Yates from the top, step k = n-1-i drawing word k of the Philox
 * stream with counter (k / 4, item, iter, side) and key (seed lo, seed hi);
 * the index is the multiply-shift (word * (i+1)) >> 32. */
void oracle_chunk_order(uint64_t seed, uint32_t iter, uint32_t item, uint32_t side, int32_t nchunks,
                        uint8_t *order) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t words[4] = {0, 0, 0, 0};
    for (int32_t i = 0; i < nchunks; ++i) order[i] = (uint8_t)i;
    for (int32_t i = nchunks - 1, k = 0; i >= 1; --i, ++k) {
        if ((k & 3) == 0) {
            const uint32_t ctr[4] = {(uint32_t)(k >> 2), item, iter, side};
            oracle_philox4x32_10(ctr, key, words);
        }
        const uint32_t j = (uint32_t)(((uint64_t)words[k & 3] * (uint32_t)(i + 1)) >> 32);
        const uint8_t tmp = order[i];
        order[i] = order[j];
        order[j] = tmp;
    }
}

/* Visit order of the 4 coordinates inside the chunk at visit position pos:
 * Fisher-Yates over (0,1,2,3) from the top with word pos % 4 of the Philox
 * block (0x100 + pos / 4, item, iter, side); step i takes the high word of
 * word * (i+1) and continues with its low word.  perm[c] = coordinate of
 * slot c. */
void oracle_chunk_perm4(uint64_t seed, uint32_t iter, uint32_t item, uint32_t side, int32_t pos, uint8_t perm[4]) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const uint32_t ctr[4] = {0x100u + (uint32_t)(pos >> 2), item, iter, side};
    uint32_t words[4];
    oracle_philox4x32_10(ctr, key, words);
    uint32_t word = words[pos & 3];
    for (int i = 0; i < 4; ++i) perm[i] = (uint8_t)i;
    for (int i = 3; i >= 1; --i) {
        const uint64_t m = (uint64_t)word * (uint32_t)(i + 1);
        const uint32_t j = (uint32_t)(m >> 32);
        word = (uint32_t)m;
        const uint8_t tmp = perm[i];
        perm[i] = perm[j];
        perm[j] = tmp;
    }
}

static inline double round_f32(double x) {
    float f = (float)x;
    return f < FLT_MIN ? 0.0 : (double)f;
}

void oracle_sweep_fp32(const int64_t *ptr, const int32_t *idx, const float *val, int64_t n_mov,
                       const float *fixed, int64_t rp, int64_t r, const double *sum_fixed,
                       float *moving, double *t, const int64_t *items, int64_t n_items,
                       double alpha, double beta, double eps_grad, double eps_x, double eps_div,
                       int64_t inner_cap, int64_t *stats, int order_mode, uint64_t order_seed,
                       uint32_t order_iter, uint32_t order_side) {
    (void)n_mov;
    const int32_t nchunks = (int32_t)((r + 3) / 4);
    uint8_t corder[64];
    int64_t cap_s = 0;
    for (int64_t q = 0; q < n_items; ++q) {
        int64_t j = items ? items[q] : q;
        int64_t s = ptr[j + 1] - ptr[j];
        if (s > cap_s) cap_s = s;
    }
    double *u = (double *)malloc(sizeof(double) * (size_t)(cap_s + 1));
    double *vi = (double *)malloc(sizeof(double) * (size_t)(cap_s + 1));
    for (int64_t q = 0; q < n_items; ++q) {
        int64_t j = items ? items[q] : q;
        int64_t lo = ptr[j], s = ptr[j + 1] - lo;
        double *tj = t + lo;
        for (int64_t p = 0; p < s; ++p) {
            const double v = (double)val[lo + p];
            u[p] = v * (1.0 / (tj[p] + eps_div));
            vi[p] = 1.0 / v;
        }
        stats[STAT_PASSES] += 1;
        /* shared order: storage order; counter order: chunks in the
         * subproblem's own order, and inside each chunk its own order of
         * the 4 coordinates */
        if (order_mode) oracle_chunk_order(order_seed, order_iter, (uint32_t)j, order_side, nchunks, corder);
        uint8_t perm4[4] = {0, 1, 2, 3};
        for (int64_t vis = 0; vis < (order_mode ? 4 * (int64_t)nchunks : r); ++vis) {
            if (order_mode && vis % 4 == 0)
                oracle_chunk_perm4(order_seed, order_iter, (uint32_t)j, order_side, (int32_t)(vis / 4), perm4);
            const int64_t tt = order_mode ? 4 * (int64_t)corder[vis / 4] + perm4[vis % 4] : vis;
            if (tt >= r) continue;
            double x = (double)moving[j * rp + tt];
            double g, h;
#define EVAL()                                                            \
    do {                                                                  \
        double gp = 0.0, hp = 0.0;                                        \
        for (int64_t p = 0; p < s; ++p) {                                 \
            double a = (double)fixed[(int64_t)idx[lo + p] * rp + tt];     \
            if (a != 0.0) {                                               \
                double z = (u[p] * u[p]) * vi[p];                         \
                gp = fma(u[p], a, gp);                                    \
                hp = fma(z * a, a, hp);                                   \
            }                                                             \
        }                                                                 \
        g = sum_fixed[tt] + alpha * x + beta - gp;                        \
        h = alpha + hp;                                                   \
    } while (0)
            EVAL();
            int64_t inner = 0;
            while ((g < -eps_grad) || (fabs(g) > eps_grad && x > eps_grad)) {
                double delta;
                int stop = 0;
                if (h <= 0.0) {
                    if (g > 0.0 && x != 0.0) {
                        delta = -x;
                        x = 0.0;
                    } else {
                        if (!(g > 0.0)) stats[STAT_DEGENERATE] += 1;
                        delta = 0.0;
                    }
                    stop = 1;
                } else {
                    double target = x - g / h;
                    if (target < 0.0) target = 0.0;
                    double xn = round_f32(target);
                    delta = xn - x;
                    double xs = x;
                    x = xn;
                    inner += 1;
                    stats[STAT_INNER_ITERS] += 1;
                    if (fabs(delta) < eps_x * xs) stop = 1;
                    else if (inner >= inner_cap) { stats[STAT_CAP_HITS] += 1; stop = 1; }
                }
                if (delta != 0.0) {
                    for (int64_t p = 0; p < s; ++p) {
                        double a = (double)fixed[(int64_t)idx[lo + p] * rp + tt];
                        if (a != 0.0) {
                            /* the device's operation sequence (fused q, u times 1/q) */
                            double pp = u[p] * vi[p]; /* 1/(t+eps) */
                            double q = fma(pp, delta * a, 1.0);
                            if (q < eps_div * pp) u[p] = 1.0 / (vi[p] * eps_div); /* t' clamped to 0 */
                            else u[p] = u[p] * (1.0 / q);
                        }
                    }
                }
                if (stop) break;
                EVAL();
            }
#undef EVAL
            moving[j * rp + tt] = (float)x;
        }
        for (int64_t p = 0; p < s; ++p) {
            double tn = 1.0 / (u[p] * vi[p]) - eps_div;
            tj[p] = tn < 0.0 ? 0.0 : tn;
        }
    }
    free(u);
    free(vi);
}
