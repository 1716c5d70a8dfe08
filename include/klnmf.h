/*
 * klnmf.h -- C ABI of the B200-native SRCD hot path (libklnmf.so).
 *
 * Two layers:
 *
 *  1. Drop-in entry points with HOST pointers in the reference's own layout
 *     (factors (r, n_items) C-order fp64, CSC with int64 indices).  They are
 *     exactly the native functions the reference Python package calls, so a
 *     maintainer binds them with ctypes in place of the numba kernels
 *     (INTEGRATION.md shows the stub):
 *       klnmf_sweep_range   replaces _kernels.sweep_range  (pkg/src/klnmf/_kernels.py:123-144)
 *       klnmf_kl_data_term  replaces _kernels.kl_data_term (pkg/src/klnmf/_kernels.py:147-160)
 *       klnmf_row_sums      replaces DenseFactor.row_sums  (pkg/src/klnmf/sparse.py:194-196)
 *     Results are bit-identical to the reference (fp64 oracle mode).
 *
 *  2. Device-resident entry points (DEVICE pointers + a cudaStream_t passed as
 *     void*) used by the Python host layer's plan (paper_1604_04026_b200/plan.py),
 *     which replaces the reference's sweep()/factorize() loop
 *     (pkg/src/klnmf/solver.py:165-216, :237-326): device CSC->CSR build and nnz
 *     bucketing, row sums, the subproblem solver kernels (fp64 exact mode and
 *     fp32-storage throughput mode), the KL objective and factor statistics.
 *
 * Device layout: a factor with n items and rank r is stored item-major as
 * (n, rp) with rp = r rounded up to a multiple of 4 (zero padding), so the
 * gather of one stored entry's fixed-factor vector is one contiguous run.
 * Columns are kept in VISIT ORDER of the current outer iteration: position tt
 * holds the coordinate ids[tt] (solver.py:287 shares one permutation across
 * both sweeps and all subproblems), so the solver streams each row front to
 * back.  perm_in/perm_out maps re-order a moving row on the fly.
 *
 * Every function returns 0 on success or a CUDA error code; the message is
 * available from klnmf_last_error().  Kernels never raise on numerical
 * trouble: like the reference (numba error_model="numpy") they produce IEEE
 * inf/nan.  Nothing here has a CPU fallback.
 */
#ifndef KLNMF_H
#define KLNMF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KLNMF_ABI_VERSION 1

/* stats slots, _kernels.py:16-21 */
#define KLNMF_STAT_CAP_HITS 0
#define KLNMF_STAT_DEGENERATE 1
#define KLNMF_STAT_INNER_ITERS 2
#define KLNMF_STAT_PASSES 3
#define KLNMF_STATS_LEN 4

int klnmf_abi_version(void);
/* sizeof(klnmf_solve_args_t) / sizeof(klnmf_side_t) as compiled (binding checks) */
int klnmf_sizeof_solve_args(void);
int klnmf_sizeof_side(void);
const char *klnmf_last_error(void);
/* Counter-mode chunk order of one subproblem, computed on the host with the
 * device's generator (uint8 order[nchunks], nchunks <= 64). */
int klnmf_chunk_order(uint64_t seed, uint32_t iter, uint32_t item, uint32_t side, int32_t nchunks, uint8_t *order);
/* Counter-mode order of the 4 coordinates inside the chunk visited at
 * position pos (uint8 perm[4]: slot c visits coordinate perm[c] of the
 * chunk), computed on the host with the device's generator. */
int klnmf_chunk_perm4(uint64_t seed, uint32_t iter, uint32_t item, uint32_t side, int32_t pos, uint8_t *perm);
/* Record a CUDA event on a stream; external != 0 makes a recording inside a
 * CUDA-graph capture a real (timing-capable) event node, re-recorded by every
 * replay (used for per-kernel timing of captured half-steps). */
int klnmf_event_record(void *event, void *stream, int external);
/* fork/join plumbing for launching independent buckets on several streams
 * (captured into one graph): a timing-free event, and stream waits on it */
int klnmf_event_create(void **event);
int klnmf_event_destroy(void *event);
int klnmf_stream_wait(void *stream, void *event);
/* CUDA IPC for the fused sharded exchange (klnmf_solve_args_t.peer_*):
 * export the device allocation holding ptr as a 64-byte handle plus ptr's
 * byte offset inside it; open a peer process's handle (returns the mapped
 * base of its allocation, peer access enabled lazily over NVLink); close a
 * mapped base. */
int klnmf_ipc_export(const void *ptr, void *handle, int64_t *offset);
int klnmf_ipc_open(const void *handle, void **base);
int klnmf_ipc_close(void *base);

/* ------------------------------------------------------------------ */
/* 1. Drop-in host entry points (reference layout, fp64, bit-exact).   */

/* _kernels.sweep_range(col_ptr, row_idx, values, at, sum_a, moving, j_lo, j_hi,
 *   ids, alpha, beta, eps_grad, eps_x, eps_div, inner_cap, ax_buf, x_buf, stats)
 * (_kernels.py:124-127).  The numba signature takes shapes from the arrays;
 * here they are explicit (n_fix = at.shape[1], n_mov = moving.shape[1],
 * r = at.shape[0]).  ax_buf/x_buf are not needed (device scratch).  Columns
 * j_lo..j_hi-1 of moving (r, n_mov) are updated in place; stats (int64[4])
 * are ACCUMULATED like the reference does. */
int klnmf_sweep_range(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                      const double *at, const double *sum_a, double *moving, int64_t j_lo,
                      int64_t j_hi, const int64_t *ids, double alpha, double beta,
                      double eps_grad, double eps_x, double eps_div, int64_t inner_cap,
                      int64_t r, int64_t n_fix, int64_t n_mov, int64_t *stats);

/* _kernels.kl_data_term(col_ptr, row_idx, values, w, f, eps_div) (_kernels.py:148):
 * sum over stored entries of v*log(v/((W^T F)_ij + eps)) - v.  w is (r, n_rows),
 * f is (r, n_cols).  Result in *out. */
/* sweep_range with solve_column's max_passes (_kernels.py:53-120): the
 * passes over a column repeat until one moves nothing (the stationarity
 * certificate of subproblem.solve_column) or max_passes is reached. */
int klnmf_sweep_range_passes(const int64_t *col_ptr, const int64_t *row_idx, const double *values, const double *at,
                             const double *sum_a, double *moving, int64_t j_lo, int64_t j_hi, const int64_t *ids,
                             double alpha, double beta, double eps_grad, double eps_x, double eps_div,
                             int64_t inner_cap, int64_t max_passes, int64_t r, int64_t n_fix, int64_t n_mov,
                             int64_t *stats);

/* replaces _kernels.kkt_violation (_kernels.py:176-190) for every column of
 * x (r, n_mov): out (r, n_mov) in the reference layout, bit-identical. */
int klnmf_kkt_violation(const int64_t *col_ptr, const int64_t *row_idx, const double *values, const double *at,
                        const double *sum_a, const double *x, double alpha, double beta, double eps_grad,
                        double eps_x, double eps_div, int64_t r, int64_t n_fix, int64_t n_mov, double *out);

/* replaces _kernels.mu_update_range (_kernels.py:193-214): moving[:, j] for
 * j in [j_lo, j_hi) rescaled in place, bit-identical (num_buf is device
 * scratch). */
int klnmf_mu_update_range(const int64_t *col_ptr, const int64_t *row_idx, const double *values, const double *fixed,
                          double *moving, const double *sum_fixed, double eps_mu, int64_t j_lo, int64_t j_hi,
                          int64_t r, int64_t n_fix, int64_t n_mov);

int klnmf_kl_data_term(const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                       const double *w, const double *f, double eps_div, int64_t r,
                       int64_t n_rows, int64_t n_cols, double *out);

/* DenseFactor.row_sums (sparse.py:194-196): out[k] = sum_i factor[k, i] with
 * numpy's pairwise summation order (bit-identical). factor is (r, n). */
int klnmf_row_sums(const double *factor, int64_t r, int64_t n, double *out);

/* ------------------------------------------------------------------ */
/* 2. Device-resident entry points.                                    */

/* One oriented view of V: CSC of V (F-side) or CSC of V^T (= CSR of V, W-side). */
typedef struct {
    const int64_t *ptr;   /* n_mov + 1 */
    const int32_t *idx;   /* nnz, index into the fixed factor */
    const void *val;      /* nnz, float (fp32 mode) or double (exact mode) */
    int64_t n_fix;
    int64_t n_mov;
    int64_t nnz;
} klnmf_side_t;

/* Solver arguments shared by both precisions.  Pointers are device pointers. */
typedef struct {
    klnmf_side_t side;
    const void *fixed;        /* (n_fix, rp) visit order, float or double */
    void *moving;             /* (n_mov, rp), float or double, in/out */
    const double *sum_pos;    /* rp: fixed-factor row sums by position */
    const int32_t *perm_in;   /* rp: moving row position holding visit position tt */
    const int32_t *perm_out;  /* rp: moving row position to write visit position tt */
    const int32_t *nat_pos;   /* r: visit position of natural coordinate k (exact mode) */
    const int32_t *items;     /* subproblem (moving item) ids to solve */
    int64_t n_items;
    /* fp32 mode: maintained products carried between half-steps */
    const int32_t *tmap;      /* nnz: position of each entry in the other side's entry order */
    const double *t_in;       /* nnz (see t_scatter) */
    double *t_out;            /* nnz (see t_scatter) */
    double *scratch;          /* exact mode: nnz doubles; fp32 long-row kernels: 4*nnz + ceil(nnz/8)
                                 (a 32-byte record and a one-byte chunk mask per entry, used only by
                                 entries beyond the on-chip capacity) */
    int32_t r;
    int32_t rp;
    double alpha, beta, eps_grad, eps_x, eps_div;
    int64_t inner_cap;
    unsigned long long *stats; /* device, KLNMF_STATS_LEN, accumulated */
    /* Coordinate order inside a subproblem (fp32 mode; exact mode requires
     * KLNMF_ORDER_SHARED).  KLNMF_ORDER_SHARED visits the storage order, i.e.
     * the iteration's shared permutation -- the reference's ids stream
     * (solver.py:276,287).  KLNMF_ORDER_COUNTER visits the subproblem's
     * 4-coordinate chunks in a per-(seed, iteration, subproblem, side) order:
     * Fisher-Yates driven by Philox4x32-10 with key (order_seed lo, hi) and
     * counter (block, subproblem id, *order_iter, order_side); storage order
     * inside a chunk.  order_iter is a device pointer so a captured launch
     * sequence can be replayed for every iteration. */
    int32_t order_mode;
    uint32_t order_side;
    uint64_t order_seed;
    const uint32_t *order_iter;
    /* exact mode: passes over the coordinates per subproblem, repeated until
     * one moves nothing (solve_column's max_passes, _kernels.py:70-120);
     * 0 or 1 = the single pass of sweep_range */
    int32_t max_passes;
    /* fp32 mode, fused exchange of a sharded run: the kernels also store every
     * result they write -- moving rows and maintained products of this rank's
     * subproblems -- into the n_peers other ranks' copies (device arrays of
     * peer base pointers, same layout as moving / t_out, mapped through CUDA
     * IPC over NVLink), so no all-gather follows the half-step.  0 = local
     * writes only. */
    int32_t n_peers;
    void *const *peer_moving;
    double *const *peer_t;
    /* fp32 mode, layout of the maintained products: 0 = t_in is read through
     * tmap (other side's entry order) and t_out / peer_t written in this
     * side's entry order; 1 = t_in is read in this side's entry order and
     * t_out / peer_t written through tmap into the other side's entry order
     * (coalesced reads at every subproblem start; scattered stores). */
    int32_t t_scatter;
    /* fp32 mode, long-row kernels: n_fix words, bit c set iff the fixed
     * factor's row has a nonzero among its stored positions 4c .. 4c+3
     * (klnmf_chunk_masks, computed at the start of the half-step).  A slice
     * gathers a row's 16-byte chunk only when its bit is set -- an all-zero
     * chunk is zero-filled without a memory request, which is bit-identical.
     * NULL = gather everything.  slice_words: 4 * nnz 16-bit words of work
     * space for the slices' per-thread transposed masks (a slice uses the
     * range of its own entries; slices shorter than 64 entries per chunk
     * gather everything). */
    const uint32_t *fixed_mask;
    uint16_t *slice_words;
} klnmf_solve_args_t;

#define KLNMF_ORDER_SHARED 0
#define KLNMF_ORDER_COUNTER 1

/* exact fp64 solver (bit-identical to _kernels.sweep_range, one warp per subproblem) */
int klnmf_solve_exact(const klnmf_solve_args_t *args, void *stream);
/* exact KKT violations (_kernels.kkt_violation) of every listed subproblem at
 * its current x; out (n_mov, rp) by position, device */
int klnmf_kkt_exact(const klnmf_solve_args_t *args, double *out, void *stream);
/* exact multiplicative update (_kernels.mu_update_range) of the listed
 * subproblems; factors (n, rp) item-major in natural order, ratio_scratch nnz */
int klnmf_mu_update_dev(const klnmf_side_t *side, const double *fixed, double *moving, const double *sum_fixed,
                        int32_t r, int32_t rp, double eps_mu, const int32_t *items, int64_t n_items,
                        double *ratio_scratch, void *stream);

/* fp32-storage / fp64-arithmetic solver.  kernel_id selects the bucket kernel:
 * lanes-per-subproblem L and entries-per-lane NPL (klnmf_fast_kernel_info). */
int klnmf_solve_fast(const klnmf_solve_args_t *args, int kernel_id, void *stream);
/* out[i] bit c = the (n_fix, rp) fp32 factor's row i has a nonzero among
 * positions 4c .. 4c+3 (c < ceil(r/4) <= 32, i.e. r <= 128; larger ranks: all
 * bits set).  For klnmf_solve_args_t.fixed_mask. */
int klnmf_chunk_masks(const float *fixed, int64_t n_fix, int32_t rp, int32_t r, uint32_t *out, void *stream);
/* Sets the launch attributes of every fp32 kernel for padded rank rp once
 * (call before capturing launches into a CUDA graph). */
int klnmf_prepare_fast(int32_t rp);
int klnmf_fast_kernel_count(void);
/* capacity (max nnz per subproblem) and lanes of kernel_id; capacity < 0 = unbounded */
int klnmf_fast_kernel_info(int kernel_id, int64_t *capacity, int32_t *lanes, int32_t *npl);
/* whether kernel_id's shared-memory layout fits the device at padded rank rp */
int klnmf_fast_kernel_fits(int kernel_id, int32_t rp, int32_t *fits);

/* Long-row bucket (capacity -1 in klnmf_fast_kernel_info): a persistent
 * cooperative kernel, one CTA per SM, each row spread over G CTAs so its
 * per-entry state stays on chip; reductions of a row group go through `sync`
 * (global memory).  klnmf_coop_info reports the CTA count, entries per CTA and
 * sync bytes per row group for padded rank rp; the caller packs the bucket's
 * rows into waves: schedule is int32[n_waves][n_ctas][4] = (index into
 * args->items or -1, rank in group, group size G, group id). */
int klnmf_coop_info(int32_t rp, int64_t *entries_per_cta, int32_t *n_ctas, int64_t *sync_bytes_per_group);
int klnmf_solve_coop(const klnmf_solve_args_t *args, const void *schedule, int32_t n_waves, int32_t n_ctas,
                     void *sync, int64_t n_groups, void *stream);

/* row sums of a device factor by position (n_items, rp): exact = numpy pairwise over
 * fp64 items in order; fast = deterministic fp64 two-level sum of fp32 items. */
int klnmf_row_sums_exact(const double *fac, int64_t n_items, int32_t rp, int32_t r,
                         double *out, void *stream);
int klnmf_row_sums_fast(const float *fac, int64_t n_items, int32_t rp, int32_t r,
                        double *out, void *stream);

/* reference layout (r, n) fp64 <-> device layout (n, rp) in visit order.
 * order[tt] = natural coordinate stored at position tt (tt < r). */
int klnmf_layout_to_device(const double *src, int64_t r, int64_t n, const int32_t *order,
                           int32_t rp, void *dst, int fp32, void *stream);
/* the same from an fp32 (r, n) source (fp32 storage only) */
int klnmf_layout_to_device_f32src(const float *src, int64_t r, int64_t n, const int32_t *order, int32_t rp,
                                  float *dst, void *stream);
int klnmf_layout_from_device(const void *src, int64_t r, int64_t n, const int32_t *order,
                             int32_t rp, int fp32, double *dst, void *stream);
/* fp32 factor (item-major, visit order) -> (r, n) natural-order fp32: the
 * values an fp32-mode download widens exactly on the host
 * (klnmf_download_f32_as_f64), half the bytes of the fp64 layout. */
int klnmf_layout_from_device_f32(const float *src, int64_t r, int64_t n, const int32_t *order, int32_t rp,
                                 float *dst, void *stream);

/* CSC (ptr/idx/val) -> CSC of the transpose, plus both entry maps:
 * map_t2o[q'] = position in the input of output entry q', map_o2t = inverse.
 * Stable (rows ascending, then columns ascending), as sparse.py:146-154. */
int klnmf_transpose(const int64_t *ptr, const int32_t *idx, const void *val, int val_bytes,
                    int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t *ptr_t,
                    int32_t *idx_t, void *val_t, int32_t *map_t2o, int32_t *map_o2t,
                    void *stream);

/* COO -> CSC (sorted by column then row, as sparse.py:92-124); values must be
 * > 0 (zeros dropped by the caller).  *dup_flag != 0 reports a duplicate. */
int klnmf_coo_to_csc(const int32_t *rows, const int32_t *cols, const void *vals, int val_bytes,
                     int64_t nnz, int64_t n_rows, int64_t n_cols, int64_t *ptr, int32_t *idx,
                     void *val, int32_t *dup_flag, void *stream);

/* nnz bucketing of subproblems j in [j_lo, j_hi): items sorted by nnz descending;
 * bucket_start[b] = first slot of bucket b where bucket b holds nnz <= bounds[b]
 * (bounds ascending, last bound may be INT64_MAX).  n_bounds <= 64. */
int klnmf_bucketize(const int64_t *ptr, int64_t j_lo, int64_t j_hi, const int64_t *bounds,
                    int n_bounds, int32_t *items, int64_t *bucket_count_host, void *stream);

/* fp32 mode: t[q] = <W_i, F_j> (fp64, natural order) for every entry of side. */
int klnmf_init_t(const klnmf_side_t *side, const float *fixed, const float *moving, int32_t rp,
                 const int32_t *fixed_pos, const int32_t *moving_pos, int32_t r, double *t,
                 void *stream);

/* KL data term over the CSC of V: sum v*log(v/(d+eps)) - v with d = <W_i,F_j>
 * accumulated in natural coordinate order (wpos/fpos map coordinate -> position).
 * fp32 selects float factors.  Deterministic.  Result (fp64) in *out_host. */
int klnmf_kl_data_term_dev(const klnmf_side_t *csc, const void *w, const void *f, int32_t rp,
                           const int32_t *wpos, const int32_t *fpos, int32_t r, int fp32,
                           double eps_div, double *out_host, void *stream);

/* fp32 mode: the KL data term from the maintained products t (fp64, one per
 * entry, in the order of val): sum v*log(v/(t+eps)) - v, a streaming pass
 * instead of nnz r-dots.  Deterministic.  Result (fp64) in *out_host. */
int klnmf_kl_data_term_t(const float *val, const double *t, int64_t nnz, double eps_div, double *out_host,
                         void *stream);
/* the same with the products of entry q at t[tmap[q]] (stored in the other
 * orientation; NULL = identity), summed in val's entry order -- so the value
 * does not depend on which orientation the products are carried in */
int klnmf_kl_data_term_t_mapped(const float *val, const double *t, const int32_t *tmap, int64_t nnz,
                                double eps_div, double *out_host, void *stream);

/* factor statistics over the r real columns: out_host[0] = sum x^2, [1] = sum x,
 * [2] = number of exact zeros (as double).  Deterministic. */
int klnmf_factor_stats(const void *fac, int64_t n_items, int32_t rp, int32_t r, int fp32,
                       double *out_host, void *stream);

/* Host <-> device bulk transfers through reusable pinned staging buffers,
 * converting on host threads (the API's int64 / fp64 arrays vs the device's
 * int32 / fp32).  Synchronous with respect to the host; n elements. */
int klnmf_upload_i64_as_i32(const int64_t *src_host, int64_t n, int32_t *dst_dev, void *stream);
int klnmf_upload_f64_as_f32(const double *src_host, int64_t n, float *dst_dev, void *stream);
int klnmf_upload_f64(const double *src_host, int64_t n, double *dst_dev, void *stream);
int klnmf_download_f32_as_f64(const float *src_dev, int64_t n, double *dst_host, void *stream);
int klnmf_download_f64(const double *src_dev, int64_t n, double *dst_host, void *stream);
/* min and max of a host array on the host threads (no device work): the
 * fp32 mode's range check of V, which the reference's SparseMatrix
 * validation (sparse.py:29-77) has no counterpart for */
int klnmf_host_minmax_f64(const double *src_host, int64_t n, double *lo_out, double *hi_out);

/* Device-side synthetic corpus (the planted-topic model of synth.py, drawn
 * with counter-based Philox streams).  Fills col_ptr
 * (device int64[m+1]), allocates the row indices and values on the device
 * (values float if fp32, else double) and returns them with nnz; hand them
 * to caller buffers with klnmf_synth_fetch (which frees them).
 * length_kind: 0 = Poisson(mean), 1 = lognormal(mean, sigma); zipf <= 0 =
 * uniform feature popularity. */
int klnmf_synth_build(uint64_t seed, int64_t n, int64_t m, int32_t topics, double zipf, int length_kind,
                      double length_mean, double length_sigma, int fp32, int64_t *nnz_out, int64_t *col_ptr,
                      int32_t **row_idx_out, void **values_out, void *stream);
int klnmf_synth_fetch(int32_t *rows, void *vals, int64_t nnz, int fp32, int32_t *rows_dst, void *vals_dst,
                      void *stream);

/* MatrixMarket coordinate files (native reader, the reference's rules and
 * messages, sparse.py:217-268).  klnmf_mm_header reports the size line;
 * klnmf_mm_read fills 0-based int64 rows/cols and fp64 values (nnz_cap >=
 * nnz).  Malformed files return KLNMF_MM_FORMAT_ERROR with the reference's
 * message in klnmf_last_error(). */
#define KLNMF_MM_FORMAT_ERROR 2
int klnmf_mm_header(const char *path, int64_t *n_rows, int64_t *n_cols, int64_t *nnz);
int klnmf_mm_read(const char *path, int64_t nnz_cap, int64_t *rows, int64_t *cols, double *vals);

#ifdef __cplusplus
}
#endif
#endif /* KLNMF_H */
