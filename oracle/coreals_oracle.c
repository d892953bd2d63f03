/*
 * coreals_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, float64 restatement of the reference's core-elements ALS
 * half-sweep (arXiv 2509.18024, reference package `coreals`).  It is the
 * checker for the CUDA path: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * (paper_2509_18024_b200) never calls into this file.
 *
 * Every function cites the reference code it restates
 * (paths relative to /root/reference/pkg/src/coreals/):
 *
 *   orc_budget            core.py:48-54      s = min(n, max(1, floor(n*rate + 1e-9)))
 *   orc_select_columns    _kernels.py:68-96  per-column top-s |x| (threshold, then
 *                                            strict-then-tied emission in row order)
 *                         _kernels.py:26-65  (threshold = s-th largest |x|)
 *   sketched Gram/RHS     _kernels.py:123-146, 149-169
 *   LU solve + jitter     core.py:120-131, _kernels.py:233-236 (LAPACK gesv)
 *   SPD solve + jitter    als.py:184-205 (scipy cho_factor / cho_solve)
 *   row dispatch          core.py:199-223 (s == n -> exact SPD row)
 *   fused residual        _kernels.py:219-230, als.py:287-288
 *
 * The threshold key used for exact selection parity with the GPU is
 *   key(k, c) = (abs_bits(float(x[k,c])) << 32) | (0xFFFFFFFF - k)
 * i.e. |x| descending, then slice-local row ascending -- the reference's
 * tie rule (ties go to the smallest row index, core.py:26-27 docstring,
 * _kernels.py:90-96).  For fp32-representable inputs this order is exactly
 * the float64 |x| order the reference uses.
 *
 * Build: see oracle/Makefile (-O2 -ffp-contract=off so no FMA contraction).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_JITTERED 1
#define ORC_SINGULAR 2

static const double JITTER_SCALE = 1e-10; /* als.py:37, core.py:126 */

/* core.py:48-54 */
int64_t orc_budget(int64_t n, double rate) {
    volatile double prod = (double)n * rate; /* multiply, then add: no FMA */
    double f = floor(prod + 1e-9);
    int64_t s = (int64_t)f;
    if (s < 1) s = 1;
    if (s > n) s = n;
    return s;
}

void orc_budget_array(const int64_t* counts, int64_t n_rows, double rate, int32_t* out) {
    for (int64_t i = 0; i < n_rows; ++i) out[i] = (int32_t)orc_budget(counts[i], rate);
}

static inline uint32_t abs_bits_f32(double x) {
    float f = (float)fabs(x);
    uint32_t u;
    memcpy(&u, &f, 4);
    return u & 0x7FFFFFFFu;
}

uint64_t orc_key(double x, int64_t k) {
    return ((uint64_t)abs_bits_f32(x) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)k);
}

/* s-th largest value (1-based) of buf[0..n), buf permuted.  Own quickselect
 * (Lomuto partition around a middle pivot); any correct selection yields
 * the same value as the reference's median-of-three variant. */
static double kth_largest(double* buf, int64_t n, int64_t s) {
    int64_t lo = 0, hi = n - 1, want = s - 1; /* index in descending order */
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        double piv = buf[mid];
        double t = buf[mid]; buf[mid] = buf[hi]; buf[hi] = t;
        int64_t store = lo;
        for (int64_t i = lo; i < hi; ++i) {
            if (buf[i] > piv) {
                t = buf[i]; buf[i] = buf[store]; buf[store] = t;
                ++store;
            }
        }
        t = buf[store]; buf[store] = buf[hi]; buf[hi] = t;
        /* buf[lo..store) > piv, buf[store] == piv */
        if (want == store) return buf[store];
        if (want < store) hi = store - 1; else lo = store + 1;
    }
    return buf[lo];
}

/* _kernels.py:68-96: Xt is NOT required; X is the (n, p) row-major slice.
 * rows_out[c*s .. c*s+s) gets slice-local rows: strictly-above-threshold
 * rows in row order, then tied rows in row order until s are emitted. */
void orc_select_columns(const double* X, int64_t n, int p, int64_t s, int32_t* rows_out,
                        double* scratch /* n */) {
    for (int c = 0; c < p; ++c) {
        for (int64_t i = 0; i < n; ++i) scratch[i] = fabs(X[i * p + c]);
        double thr = kth_largest(scratch, n, s);
        int64_t k = 0;
        int32_t* out = rows_out + (int64_t)c * s;
        for (int64_t i = 0; i < n && k < s; ++i)
            if (fabs(X[i * p + c]) > thr) out[k++] = (int32_t)i;
        for (int64_t i = 0; i < n && k < s; ++i)
            if (fabs(X[i * p + c]) == thr) out[k++] = (int32_t)i;
    }
}

/* Gaussian elimination with partial pivoting (first max |a| wins, like
 * LAPACK idamax).  A is (nf, nf) row-major, overwritten; b overwritten with
 * the solution.  Returns 0, or 1 when an exact zero pivot is met (the case
 * where LAPACK getrf reports info > 0 and numpy raises LinAlgError). */
static int lu_solve_inplace(double* A, double* b, int nf) {
    for (int k = 0; k < nf; ++k) {
        int piv = k;
        double best = fabs(A[k * nf + k]);
        for (int r = k + 1; r < nf; ++r) {
            double v = fabs(A[r * nf + k]);
            if (v > best) { best = v; piv = r; }
        }
        if (best == 0.0 || isnan(best)) return 1;
        if (piv != k) {
            for (int j = 0; j < nf; ++j) {
                double t = A[k * nf + j]; A[k * nf + j] = A[piv * nf + j]; A[piv * nf + j] = t;
            }
            double t = b[k]; b[k] = b[piv]; b[piv] = t;
        }
        double d = A[k * nf + k];
        for (int r = k + 1; r < nf; ++r) {
            double f = A[r * nf + k] / d;
            if (f == 0.0) continue;
            for (int j = k + 1; j < nf; ++j) A[r * nf + j] -= f * A[k * nf + j];
            b[r] -= f * b[k];
        }
    }
    for (int r = nf - 1; r >= 0; --r) {
        double acc = b[r];
        for (int j = r + 1; j < nf; ++j) acc -= A[r * nf + j] * b[j];
        b[r] = acc / A[r * nf + r];
    }
    return 0;
}

/* Cholesky (lower) solve; returns 1 when A is not numerically positive
 * definite (LAPACK potrf failure). */
static int chol_solve_inplace(double* A, double* b, int nf) {
    for (int j = 0; j < nf; ++j) {
        double d = A[j * nf + j];
        for (int k = 0; k < j; ++k) d -= A[j * nf + k] * A[j * nf + k];
        if (!(d > 0.0)) return 1;
        d = sqrt(d);
        A[j * nf + j] = d;
        for (int i = j + 1; i < nf; ++i) {
            double v = A[i * nf + j];
            for (int k = 0; k < j; ++k) v -= A[i * nf + k] * A[j * nf + k];
            A[i * nf + j] = v / d;
        }
    }
    for (int i = 0; i < nf; ++i) { /* L z = b */
        double v = b[i];
        for (int k = 0; k < i; ++k) v -= A[i * nf + k] * b[k];
        b[i] = v / A[i * nf + i];
    }
    for (int i = nf - 1; i >= 0; --i) { /* L^T x = z */
        double v = b[i];
        for (int k = i + 1; k < nf; ++k) v -= A[k * nf + i] * b[k];
        b[i] = v / A[i * nf + i];
    }
    return 0;
}

/* Solve with the reference's single jitter retry (core.py:120-131 for LU,
 * als.py:184-197 for SPD).  G is preserved; x receives the solution. */
static int solve_with_jitter(const double* G, const double* b, int nf, int spd,
                             double* work /* nf*nf */, double* x) {
    memcpy(work, G, sizeof(double) * nf * nf);
    memcpy(x, b, sizeof(double) * nf);
    int bad = spd ? chol_solve_inplace(work, x, nf) : lu_solve_inplace(work, x, nf);
    if (!bad) return ORC_OK;
    double tr = 0.0;
    for (int i = 0; i < nf; ++i) tr += G[i * nf + i];
    double jitter = JITTER_SCALE * tr / nf;
    memcpy(work, G, sizeof(double) * nf * nf);
    for (int i = 0; i < nf; ++i) work[i * nf + i] += jitter;
    memcpy(x, b, sizeof(double) * nf);
    bad = spd ? chol_solve_inplace(work, x, nf) : lu_solve_inplace(work, x, nf);
    return bad ? ORC_SINGULAR : ORC_JITTERED;
}

typedef struct {
    const int64_t* ptr;
    const int32_t* idx;
    const double* val;
    const double* source;
    int64_t n_src;
    int n_f;
    double lam;
    double rate;
    double* target;
    double* rss_rows;   /* nullable */
    int32_t* status;    /* nullable */
    uint64_t* thr_keys; /* nullable, [n_rows, n_f] */
    const int32_t* rows;
    int64_t n_list;
    int n_threads;
    int tid;
} sweep_args;

/* One regression (core.py:199-223 + als.py:286-288). */
static void do_row(const sweep_args* a, int64_t i, double* X, double* y, double* G, double* b,
                   double* work, double* w, int32_t* sel, double* scratch) {
    const int nf = a->n_f;
    int64_t lo = a->ptr[i], hi = a->ptr[i + 1];
    int64_t n = hi - lo;
    if (n <= 0) {
        if (a->rss_rows) a->rss_rows[i] = 0.0;
        if (a->status) a->status[i] = ORC_OK;
        return;
    }
    for (int64_t k = 0; k < n; ++k) {
        const double* src = a->source + (int64_t)a->idx[lo + k] * nf;
        for (int f = 0; f < nf; ++f) X[k * nf + f] = src[f];
        y[k] = a->val[lo + k];
    }
    int64_t s = orc_budget(n, a->rate);
    double lam_n = a->lam * (double)n;
    int spd = (s == n);
    if (spd) {
        /* als.py:200-205: A = X^T X + lam*n I, rhs X^T y */
        for (int c = 0; c < nf; ++c) {
            for (int f = 0; f < nf; ++f) {
                double acc = 0.0;
                for (int64_t k = 0; k < n; ++k) acc += X[k * nf + c] * X[k * nf + f];
                G[c * nf + f] = acc;
            }
            double acc = 0.0;
            for (int64_t k = 0; k < n; ++k) acc += X[k * nf + c] * y[k];
            b[c] = acc;
            G[c * nf + c] += lam_n;
        }
        if (a->thr_keys) {
            for (int c = 0; c < nf; ++c) {
                uint64_t mn = UINT64_MAX;
                for (int64_t k = 0; k < n; ++k) {
                    uint64_t key = orc_key(X[k * nf + c], k);
                    if (key < mn) mn = key;
                }
                a->thr_keys[i * nf + c] = mn;
            }
        }
    } else {
        orc_select_columns(X, n, nf, s, sel, scratch);
        /* _kernels.py:123-146: G[c,:] = sum_{k in S_c} X[k,c] X[k,:] */
        for (int c = 0; c < nf; ++c) {
            const int32_t* sc = sel + (int64_t)c * s;
            for (int f = 0; f < nf; ++f) G[c * nf + f] = 0.0;
            double acc = 0.0;
            uint64_t mn = UINT64_MAX;
            for (int64_t q = 0; q < s; ++q) {
                int64_t k = sc[q];
                double v = X[k * nf + c];
                for (int f = 0; f < nf; ++f) G[c * nf + f] += v * X[k * nf + f];
                acc += v * y[k];
                uint64_t key = orc_key(v, k);
                if (key < mn) mn = key;
            }
            b[c] = acc;
            G[c * nf + c] += lam_n;
            if (a->thr_keys) a->thr_keys[i * nf + c] = mn;
        }
    }
    int st = solve_with_jitter(G, b, nf, spd, work, w);
    if (a->status) a->status[i] = st;
    if (st == ORC_SINGULAR) return;
    double* t = a->target + i * nf;
    for (int f = 0; f < nf; ++f) t[f] = w[f];
    if (a->rss_rows) {
        /* _kernels.py:219-230 with the NEW row w */
        double acc = 0.0;
        for (int64_t k = 0; k < n; ++k) {
            double d = y[k];
            for (int f = 0; f < nf; ++f) d -= X[k * nf + f] * w[f];
            acc += d * d;
        }
        a->rss_rows[i] = acc;
    }
}

static void* sweep_worker(void* p) {
    const sweep_args* a = (const sweep_args*)p;
    const int nf = a->n_f;
    int64_t maxn = 0;
    for (int64_t q = a->tid; q < a->n_list; q += a->n_threads) {
        int64_t i = a->rows ? a->rows[q] : q;
        int64_t n = a->ptr[i + 1] - a->ptr[i];
        if (n > maxn) maxn = n;
    }
    if (maxn < 1) maxn = 1;
    double* X = (double*)malloc(sizeof(double) * maxn * nf);
    double* y = (double*)malloc(sizeof(double) * maxn);
    double* scratch = (double*)malloc(sizeof(double) * maxn);
    int32_t* sel = (int32_t*)malloc(sizeof(int32_t) * maxn * nf);
    double* G = (double*)malloc(sizeof(double) * nf * nf);
    double* work = (double*)malloc(sizeof(double) * nf * nf);
    double* b = (double*)malloc(sizeof(double) * nf);
    double* w = (double*)malloc(sizeof(double) * nf);
    for (int64_t q = a->tid; q < a->n_list; q += a->n_threads) {
        int64_t i = a->rows ? a->rows[q] : q;
        do_row(a, i, X, y, G, b, work, w, sel, scratch);
    }
    free(X); free(y); free(scratch); free(sel); free(G); free(work); free(b); free(w);
    return NULL;
}

/* One core-estimator half-sweep over the rows listed in `rows` (or all
 * n_list rows when rows == NULL).  source is (n_src, n_f) row-major f64;
 * target is (n_rows, n_f) and only listed rows with n_i > 0 are written
 * (als.py:252-259, 282-286). */
int orc_core_half_sweep(const int64_t* ptr, const int32_t* idx, const double* val,
                        const double* source, int64_t n_src, int n_f, double lam, double rate,
                        double* target, double* rss_rows, int32_t* status, uint64_t* thr_keys,
                        const int32_t* rows, int64_t n_list, int n_threads) {
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    pthread_t th[256];
    sweep_args args[256];
    for (int t = 0; t < n_threads; ++t) {
        sweep_args* a = &args[t];
        a->ptr = ptr; a->idx = idx; a->val = val; a->source = source; a->n_src = n_src;
        a->n_f = n_f; a->lam = lam; a->rate = rate; a->target = target; a->rss_rows = rss_rows;
        a->status = status; a->thr_keys = thr_keys; a->rows = rows; a->n_list = n_list;
        a->n_threads = n_threads; a->tid = t;
    }
    if (n_threads == 1) {
        sweep_worker(&args[0]);
        return 0;
    }
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, sweep_worker, &args[t]);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* Public single-row sketched update, core.py:134-157: X (n, p) dense slice,
 * sketch given as slice-local rows per column (col_ptr, rows), complete ->
 * SPD path.  Returns the solve status. */
int orc_update_core(const double* X, int64_t n, int p, const int64_t* col_ptr, const int32_t* rows,
                    const double* y, double lam, int64_t n_count, double* w_out) {
    double* G = (double*)calloc((size_t)p * p, sizeof(double));
    double* work = (double*)malloc(sizeof(double) * p * p);
    double* b = (double*)calloc((size_t)p, sizeof(double));
    double lam_n = lam * (double)n_count;
    int complete = (col_ptr[p] == n * p);
    if (complete) {
        for (int c = 0; c < p; ++c) {
            for (int f = 0; f < p; ++f) {
                double acc = 0.0;
                for (int64_t k = 0; k < n; ++k) acc += X[k * p + c] * X[k * p + f];
                G[c * p + f] = acc;
            }
            double acc = 0.0;
            for (int64_t k = 0; k < n; ++k) acc += X[k * p + c] * y[k];
            b[c] = acc;
            G[c * p + c] += lam_n;
        }
    } else {
        for (int c = 0; c < p; ++c) {
            double acc = 0.0;
            for (int64_t q = col_ptr[c]; q < col_ptr[c + 1]; ++q) {
                int64_t k = rows[q];
                double v = X[k * p + c];
                for (int f = 0; f < p; ++f) G[c * p + f] += v * X[k * p + f];
                acc += v * y[k];
            }
            b[c] = acc;
            G[c * p + c] += lam_n;
        }
    }
    int st = solve_with_jitter(G, b, p, complete, work, w_out);
    free(G); free(work); free(b);
    return st;
}
