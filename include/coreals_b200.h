/*
 * coreals_b200.h -- C ABI of the B200 (sm_100a) core-elements ALS half-sweep.
 *
 * This is the drop-in boundary for the reference's hot path
 *   coreals.fit_core -> als._alternate -> core._CoreSweeper.row
 * (/root/reference/pkg/src/coreals/core.py:301-312, als.py:243-323,
 *  core.py:173-223).  The reference's per-row Python plugin seam
 * (`sweeper.begin/row`, als.py:281-285) is replaced at half-sweep
 * granularity: one call updates every row of one side.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller, unless the
 *    parameter name ends in `_host`.  Nothing here allocates device memory:
 *    scratch comes from a caller-provided workspace sized by
 *    cals_workspace_bytes().
 *  - Work is enqueued on `stream` (a cudaStream_t passed as void*); calls are
 *    asynchronous and capturable into CUDA graphs.  One host thread per
 *    device/stream.
 *  - Factor matrices are fp32, row-major, leading dimension `ld` >= n_f.  The
 *    SOURCE of a half-sweep must have ld a multiple of 4 (>= n_f rounded up),
 *    16-byte alignment and zeros in the padding columns: its rows are
 *    gathered as 16-byte chunks (cp.async).
 *  - Ratings are CSR (user side) or CSC (item side): int64 ptr, int32 idx
 *    ascending within each row, fp32 values (reference RatingMatrix,
 *    ratings.py:83-92, with values narrowed to fp32).
 *  - Return value: CALS_OK or a CALS_ERR_* code; cals_strerror() names it.
 *    Per-row numerical outcomes go to `row_status` (CALS_ROW_*), which the
 *    host maps to NumericalError exactly where the reference raises it
 *    (core.py:131, als.py:197).
 */
#ifndef COREALS_B200_H
#define COREALS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CALS_OK 0
#define CALS_ERR_ARG 1
#define CALS_ERR_CUDA 2
#define CALS_ERR_WORKSPACE 3
#define CALS_ERR_UNSUPPORTED 4

/* per-row status (core.py:120-131 / als.py:184-197 jitter semantics): a system the
 * fp32 solve cannot hold (breakdown, or a pivot-magnitude spread marking it
 * ill-conditioned) is re-solved in float64 inside the same call -- plain first
 * (CALS_ROW_OK), then with the reference's 1e-10 * tr(G) / n_f jitter
 * (CALS_ROW_JITTERED), else CALS_ROW_SINGULAR (row left untouched). */
#define CALS_ROW_OK 0
#define CALS_ROW_JITTERED 1
#define CALS_ROW_SINGULAR 2

#define CALS_MAX_NF 128

/* One side of the rating matrix (CSR over users or CSC over items). */
typedef struct cals_side {
    const int64_t* ptr; /* [n_rows + 1] */
    const int32_t* idx; /* [nnz]  source-row ids, ascending per row */
    const float* val;   /* [nnz]  ratings */
    int64_t n_rows;
    int64_t nnz;
} cals_side;

/*
 * Static per-side schedule, built once per (dataset, n_f, rate) on the host
 * by cals_plan_build(); the caller uploads the arrays and points the struct
 * at the device copies.  Rows with n_i = 0 are absent (skipped,
 * als.py:252-259).
 */
typedef struct cals_plan {
    const int32_t* budget;        /* [n_rows] s_i = sketch_budget(n_i, rate), core.py:48-54 */
    const int32_t* small_rows;    /* rows whose slice is staged whole in shared memory, n desc */
    int64_t n_small;
    int64_t small_seg[4];         /* small_rows[seg[g] .. seg[g+1]) have n_i <= small_seg_maxn[g] */
    int32_t small_seg_maxn[3];
    int32_t small_seg_maxs[3];    /* largest budget s_i < n_i in the segment (kept-row lists) */
    const int32_t* big_rows;      /* rows streamed in work items (slice > shared memory), n desc */
    int64_t n_big;
    const int64_t* big_tile_ptr;  /* [n_big + 1] prefix of work items per big row */
    int64_t n_big_tiles;
    const int64_t* big_cand_ptr;  /* [n_big + 1] candidate-key offsets per big row (n_f equal regions) */
    int64_t big_cand_total;
    int32_t item_rows;            /* slice rows per work item of a big row */
    int32_t n_f;                  /* rank the plan was built for */
    const int64_t* big_tile_ptr_host;  /* host copies (caller-owned) used to batch the tiled tier */
    const int64_t* big_cand_ptr_host;
    const int32_t* big_tile_row;  /* optional device [n_big_tiles]: big row of each work item (else searched) */
    int64_t n_rows;               /* rows of the side (sizes the per-row selection thresholds) */
} cals_plan;

/* Host: reference budget rule for every row (core.py:48-54), fp64, no FMA. */
int cals_budget_host(const int64_t* counts_host, int64_t n_rows, double rate, int32_t* budget_host);

/* Host: build the schedule.  counts_host[i] = n_i.  Output host arrays:
 * budget_host, small_rows_host, big_rows_host sized n_rows;
 * big_tile_ptr_host, big_cand_ptr_host sized n_rows + 1.  `meta` receives
 * the scalar fields (its pointer fields are set to NULL). */
int cals_plan_build(const int64_t* counts_host, int64_t n_rows, int n_f, double rate,
                    int32_t* budget_host, int32_t* small_rows_host, int32_t* big_rows_host,
                    int64_t* big_tile_ptr_host, int64_t* big_cand_ptr_host, cals_plan* meta);

/* Device workspace needed by cals_core_half_sweep for this plan. */
size_t cals_workspace_bytes(const cals_plan* plan);

/*
 * One core-estimator half-sweep (the GPU replacement for the per-row loop
 * als.py:282-288 driving core.py:199-223):
 *   for every row i with n_i > 0:
 *     per column c keep the s_i slice rows of largest |source[idx, c]| (ties to
 *     the smallest row), G = X*^T X + lam*n_i*I, b = X*^T y, solve G w = b by
 *     LU with partial pivoting (s_i == n_i: the exact SPD ridge row), target[i] = w.
 *   target may alias target_old only when rss_rows is NULL.
 *   rss_rows (nullable; needs target_old): fused residual of the PREVIOUS rows,
 *     sum_k (y_k - X_k . target_old[i])^2 per row, fp64 (_kernels.py:219-230).
 *     The reference fuses the residual of iteration t into its item half-sweep;
 *     here it rides on the first half-sweep of iteration t+1, whose slices
 *     hold exactly the needed rows, so it costs no extra memory traffic.
 *   pen_rows (nullable): n_i * |w_i|^2 of every new row, fp64 (als.py:162-167).
 *   thr_keys (nullable): [n_rows, n_f] selection threshold key per (row, column),
 *     key = (abs_bits(x) << 32) | (0xFFFFFFFF - slice_row); the kept set of column
 *     c is exactly {k : key(k, c) >= thr_keys[i, c]}.
 *   row_status: [n_rows] CALS_ROW_*; rows with n_i = 0 are left untouched.
 *   status_summary (nullable, 1 element, overwritten): max over rows of
 *     (status << 32) | (0xFFFFFFFF - row) -- 0 when every row is CALS_ROW_OK;
 *     otherwise the worst status and the first row having it, so the host can
 *     raise NumericalError with the reference's context after one tiny read.
 */
int cals_core_half_sweep(const cals_side* side, const cals_plan* plan, const float* source,
                         int64_t n_src, int ld_src, int n_f, double lam, float* target,
                         int ld_tgt, const float* target_old, int ld_old, double* rss_rows,
                         double* pen_rows, uint64_t* thr_keys, int32_t* row_status,
                         uint64_t* status_summary, void* workspace, size_t ws_bytes, void* stream);

/* Residual only: rss_rows[i] = sum over row i's ratings of (y - source[idx] . rows_w[i])^2,
 * fp64 (the fused residual of the final iteration, _kernels.py:219-230). */
int cals_residual(const cals_side* side, const float* source, int ld_src, int n_f, const float* rows_w, int ld_w,
                  double* rss_rows, void* stream);

/* Deterministic fp64 sum of an array (fixed reduction tree). out: 1 double. */
int cals_sum_f64(const double* x, int64_t n, double* out, void* workspace, size_t ws_bytes,
                 void* stream);

/* Weighted penalty term sum_i counts_i * ||F_i||^2 (als.py:162-167), fp64. */
int cals_weighted_sqnorm(const float* F, int64_t n_rows, int n_f, int ld, const int64_t* ptr,
                         double* out, void* workspace, size_t ws_bytes, void* stream);

/* Public subsample entry (core.py:95-115): per column of the dense slice X
 * (n x p, row-major fp32) keep s rows; rows_out (p*s) slice-local, strict-
 * then-tied ascending order as the reference emits them; vals_out = X[rows, c]. */
int cals_ces_sketch(const float* X, int64_t n, int p, int32_t s, int32_t* rows_out,
                    float* vals_out, void* workspace, size_t ws_bytes, void* stream);
size_t cals_ces_sketch_workspace_bytes(int64_t n, int p);

/* Same selection for a float64 slice (exact |x| ranks, any values): rows_out
 * as above.  workspace >= n * p bytes.  For the public API on float64 input. */
int cals_ces_sketch_f64(const double* X, int64_t n, int p, int32_t s, int32_t* rows_out, void* workspace,
                        size_t ws_bytes, void* stream);

/* Public single-row sketched update (core.py:134-157): X (n x p) float64,
 * sketch given as per-column slice-local rows (col_ptr int64[p+1], rows int32),
 * complete -> exact SPD path; float64 arithmetic.  w_out (p doubles), status_out (1 int32). */
int cals_update_core(const double* X, int64_t n, int p, const int64_t* col_ptr,
                     const int32_t* rows, const double* y, double lam_n, int complete,
                     double* w_out, int32_t* status_out, void* stream);

/* predict_entries (als.py:143-152): out[e] = U[users[e]] . M[items[e]]. */
int cals_predict_entries(const float* U, const float* M, int n_f, int ld_u, int ld_m,
                         const int64_t* users, const int64_t* items, int64_t n, double* out,
                         void* stream);
/* Same with float64 factors (FactorPair precision; the evaluation metrics rank by these scores,
 * metrics.py:64-160). */
int cals_predict_entries_f64(const double* U, const double* M, int n_f, int ld_u, int ld_m, const int64_t* users,
                             const int64_t* items, int64_t n, double* out, void* stream);
/* predict_full (als.py:155-157): out[u * ld_out + i] = U[u] . M[i] for every (u, i), float64
 * (a register-tiled 64 x 64 output tile per CTA). */
int cals_predict_full_f64(const double* U, const double* M, int64_t n_users, int64_t n_items, int n_f, int ld_u,
                          int ld_m, double* out, int64_t ld_out, void* stream);
/*
 * Ranking metrics per user (metrics.py:89-147: hit@k and score-gain NDCG@k), one warp per user
 * segment of the held-out entries.  seg_ptr int64[n_seg+1] groups the entries by user with items
 * ascending inside a segment (the device index of the held-out triplets); perm[e] is the
 * original position of grouped entry e, truths / scores are in original order.  An entry's
 * predicted rank counts the entries of its user with a larger score, or an equal score and a
 * smaller item (the reference's lexsort((item, -score))); its ideal rank orders by truth.
 * Per user (float64, 0/1 flags as 0.0/1.0; users without entries get zeros):
 *   qual[u]  any entry with truth >= threshold          (hit@k qualifies, metrics.py:113-116)
 *   hit[u]   qual and such an entry at predicted rank < k_hit
 *   used[u]  ideal DCG@k_ndcg > 0                        (metrics.py:142-143)
 *   ratio[u] DCG@k_ndcg / ideal DCG@k_ndcg if used, else 0
 * The caller reduces them (cals_sum_f64: fixed-order sums).
 */
int cals_rank_metrics(const int64_t* seg_ptr, int64_t n_seg, const int32_t* perm, const double* truths,
                      const double* scores, int k_hit, double threshold, int k_ndcg, double* qual, double* hit,
                      double* ratio, double* used, void* stream);

/*
 * Method 'fast_core' (core.py:255-298): ONE sketch of the whole source per
 * half-sweep instead of one per regression.
 *   cals_plan_build_fast: every active row becomes a work-item row (sorted by
 *     length); budget = n_i for a complete sketch (exact SPD rows), else 0
 *     (every row solved by LU, _solve_sketched).  rows_host [n_rows],
 *     tile_ptr_host / cand_ptr_host [n_rows + 1].
 *   cals_fast_sketch: thr[c] = key of the s-th largest |source[:, c]| (s =
 *     sketch_budget(n_src, rate), ties to the smaller row; key as thr_keys
 *     below with the source row as index), and the kept mask
 *     gmask[j * ceil(n_f/32) + c/32] bit c%32 = (key(j, c) >= thr[c])
 *     (ces_sketch of the whole matrix, core.py:95-115).
 *   cals_fast_half_sweep: per row G[c] sums the slice rows kept for column c
 *     by gmask; a column with none takes the slice's first largest-|x| row
 *     (gram_rhs_rowsketch, _kernels.py:172-216); G += lam*n_i*I; solve and
 *     write as cals_core_half_sweep (rss_rows / target_old: the fused residual
 *     of the previous rows, as there).
 */
int cals_plan_build_fast(const int64_t* counts_host, int64_t n_rows, int n_f, int complete, int32_t* budget_host,
                         int32_t* rows_host, int64_t* tile_ptr_host, int64_t* cand_ptr_host, cals_plan* meta);
size_t cals_fast_sketch_workspace_bytes(int n_f);
int cals_fast_sketch(const float* source, int64_t n_src, int ld_src, int n_f, int64_t s, uint64_t* thr,
                     uint32_t* gmask, void* ws, size_t ws_bytes, void* stream);
int cals_fast_half_sweep(const cals_side* side, const cals_plan* plan, const float* source, int64_t n_src, int ld_src,
                         int n_f, double lam, const uint32_t* gmask, float* target, int ld_tgt,
                         const float* target_old, int ld_old, double* rss_rows, double* pen_rows,
                         int32_t* row_status, uint64_t* status_summary, void* ws, size_t ws_bytes, void* stream);

/*
 * Device dual index (RatingMatrix, ratings.py:54-92): the reference's two host
 * lexsorts replaced by one device primitive, "group by key, order by
 * secondary" (paper_2509_18024_b200/csrc/index.cu).  Integer work, exact.
 *   cals_coo_to_csr: entries (keys[e], secs[e], vals[e]) -> ptr[n_keys + 1],
 *     out_idx[nnz] = secondaries ascending within each key, out_val[nnz];
 *     keys must lie in [0, n_keys) and secs in [0, n_sec) (validated by the
 *     caller, as ratings.py:62-68 does).  dup_out (1 device uint64): the first
 *     duplicated (key, sec) pair in (key, sec) order as (key << 32) | sec, or
 *     all ones -- the pair ratings.py:77-82 names in its DataError.
 *   cals_csr_to_csc: the dual (column-major) index of a CSR whose idx ascend
 *     within rows: col_ptr[n_cols + 1], col_idx = rows ascending within each
 *     column, col_val (ratings.py:86-92).
 *   Workspace: cals_index_workspace_bytes(n_keys, n_sec, nnz) with (n_keys,
 *   n_sec) = (n_rows, n_cols) for coo_to_csr and (n_cols, n_rows) for
 *   csr_to_csc.
 */
size_t cals_index_workspace_bytes(int64_t n_keys, int64_t n_sec, int64_t nnz);
int cals_coo_to_csr(const int32_t* keys, const int32_t* secs, const float* vals, int64_t nnz, int64_t n_keys,
                    int64_t n_sec, int64_t* ptr, int32_t* out_idx, float* out_val, uint64_t* dup_out, void* ws,
                    size_t ws_bytes, void* stream);
int cals_csr_to_csc(const int64_t* ptr, const int32_t* idx, const float* val, int64_t n_rows, int64_t n_cols,
                    int64_t nnz, int64_t* col_ptr, int32_t* col_idx, float* col_val, void* ws, size_t ws_bytes,
                    void* stream);

/* Optional per-kernel timing with CUDA events recorded on the launch stream
 * (for bench.py's roofline numbers).  collect() synchronises on the recorded
 * events, writes "name launches total_ms" lines into buf, and resets. */
void cals_profile_enable(int on);
/* 1 while per-kernel event timing is enabled (cals_profile_enable). */
int cals_profile_enabled(void);
/* Debug: point the sweep kernels at 16 device uint64 counters (NULL = off):
 * [0] table-resolved columns, [1] bracket fallbacks, [2] bracket candidates,
 * [3] candidates after pre-narrowing, [4] extra select rounds, [5] rows. */
void cals_debug_stats(void* device_counters);
/* Debug: override the tiled-tier batch budgets (candidate keys, work items per
 * batch; 0 = defaults of 2^27 keys and 1 GiB of partial normal equations).
 * Must stay in effect from sizing a workspace until its last half-sweep. */
void cals_debug_big_batch(int64_t cand_keys, int64_t tiles);
/*
 * Explicit tuning (process-wide; set it before building plans and sizing
 * workspaces, keep it until their last half-sweep).  NULL restores the
 * defaults.  Zero / negative fields select the built-in defaults.
 *   item_rows      slice rows per work item of a tiled row (default 16384)
 *   ill_ratio      pivot-magnitude spread that defers a system to the float64
 *                  solve (default rank-dependent; 0 = every system)
 *   rf_slice_max   deferred rows up to this length rebuild their Gram in float64
 *                  from the slice (default 4096)
 *   gram_path      tiled Gram at 32 < n_f <= 64: 0 the tensor-core integer Gram
 *                  (tcgen05 kind::i8, csrc/sweep_tc.cu), 1 the float64 SIMT
 *                  accumulate it replaced (comparison); both float64-quality
 *   calib_samples, calib_z   long-row bracket calibration (defaults 4096, 5.5)
 *   fold_chunks    fp32 tiled Gram (n_f <= 32, and method fast_core): staged chunks summed
 *                  before a float64 fold (4); above n_f = 32 the tiled Gram sums in float64
 *   serial_tiers   1: the staged tier runs on the caller's stream before the tiled
 *                  tier instead of beside it on a second stream (profiling)
 *   tc_debug       profiling only (results are then wrong): bit 0 skips the
 *                  tensor-core Gram's MMAs, bit 1 its digit pass, bit 2 its digit
 *                  stores; 8 traces CTA 0 into the cals_debug_stats buffer
 *   qtab_min_nnz   sides with fewer ratings skip the per-half-sweep quantile
 *                  table (the staged tier then selects by its exact column
 *                  search; default 2^20; 1 = always build it)
 *   staged_max_rows  rows up to this many ratings take the staged tier (whole slice in one
 *                  CTA's shared memory); longer rows the tiled tier.  0 = the longest row
 *                  whose staged layout fits the tier's shared-memory budget (384 at
 *                  n_f = 64, rate 0.1); values above that are clamped to it
 */
typedef struct cals_tuning {
    int32_t item_rows;
    float ill_ratio;
    int32_t rf_slice_max;
    int32_t gram_path;
    int32_t calib_samples;
    float calib_z;
    int32_t fold_chunks;
    int32_t serial_tiers;
    int32_t tc_debug;
    int64_t qtab_min_nnz;
    int32_t staged_max_rows;
} cals_tuning;
void cals_set_tuning(const cals_tuning* tuning);
void cals_get_tuning(cals_tuning* tuning);
int cals_profile_collect(char* buf, size_t len);

const char* cals_strerror(int status);
const char* cals_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* COREALS_B200_H */
