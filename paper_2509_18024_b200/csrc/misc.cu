// misc.cu -- reductions, the public sketch / single-row update entry points,
// and prediction.  None of these is on the per-iteration critical path
// except the two deterministic reductions (objective terms).
#include "select.cuh"
#include "solve.cuh"
#include "sweep_common.cuh"

namespace cals {

constexpr int kRedBlocks = 296;  // 2 x 148 SMs, fixed so the reduction tree is fixed

// Stage 1 of a deterministic sum: per-block fp64 partials in a fixed tree.
template <class F>
__device__ void block_partial(F term, int64_t n, double* partials) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += term(i);
    acc = block_sum_d(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(256) sum_partial_kernel(const double* __restrict__ x, int64_t n, double* partials) {
    block_partial([x](int64_t i) { return x[i]; }, n, partials);
}

__global__ void __launch_bounds__(256) sqnorm_partial_kernel(const float* __restrict__ F, int64_t n_rows, int nf, int ld,
                                                             const int64_t* __restrict__ ptr, double* partials) {
    block_partial(
        [=](int64_t i) {
            const double cnt = (double)(ptr[i + 1] - ptr[i]);
            if (cnt == 0.0) return 0.0;
            double s = 0.0;
            for (int f = 0; f < nf; ++f) {
                const double v = (double)F[i * ld + f];
                s = fma(v, v, s);
            }
            return cnt * s;
        },
        n_rows, partials);
}

__global__ void __launch_bounds__(256) finish_sum_kernel(const double* __restrict__ partials, int nb, double* out) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += partials[i];
    acc = block_sum_d(acc, red);
    if (threadIdx.x == 0) out[0] = acc;
}

// ---- residual only (the fused residual of the last iteration) -------------
// rss_rows[i] = sum_k (y_k - source[idx_k] . w_i)^2 over row i's ratings,
// one warp per row, float64 accumulation (_kernels.py:219-230).
__global__ void __launch_bounds__(256) residual_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                                       const float* __restrict__ val, int64_t n_rows,
                                                       const float* __restrict__ src, int ld_src, int nf,
                                                       const float* __restrict__ w, int ld_w, double* rss_rows) {
    // the warp's row of w in shared memory (16-byte rows: ld_src is a multiple of 4 and the
    // padding of w is zero or never read), source rows gathered as 16-byte chunks
    __shared__ __align__(16) float ws[8][CALS_MAX_NF_DEV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nq = (nf + 3) >> 2;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float* wr = ws[warp];
    for (int64_t r = gw; r < n_rows; r += stride) {
        const int64_t lo = ptr[r], hi = ptr[r + 1];
        __syncwarp();
        for (int f = lane; f < 4 * nq; f += 32) wr[f] = f < nf ? w[r * ld_w + f] : 0.f;
        __syncwarp();
        double acc = 0.0;
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const float4* x = reinterpret_cast<const float4*>(src + (int64_t)__ldg(idx + e) * ld_src);
            double pred = 0.0;
            for (int q = 0; q < nq; ++q) {
                const float4 v = __ldg(x + q);
                const float4 u = *reinterpret_cast<const float4*>(wr + 4 * q);
                pred = fma((double)v.x, (double)u.x, pred);
                pred = fma((double)v.y, (double)u.y, pred);
                pred = fma((double)v.z, (double)u.z, pred);
                pred = fma((double)v.w, (double)u.w, pred);
            }
            const double d = (double)__ldg(val + e) - pred;
            acc = fma(d, d, acc);
        }
        acc = warp_sum_d(acc);
        if (lane == 0) rss_rows[r] = acc;
    }
}

// ---- public sketch (core.py:95-115) -------------------------------------
// One warp per column.  ws: p * n keys.
__global__ void __launch_bounds__(256) ces_sketch_kernel(const float* __restrict__ X, int n, int p, int s,
                                                         int32_t* __restrict__ rows_out, float* __restrict__ vals_out,
                                                         uint64_t* ws) {
    const int lane = threadIdx.x & 31;
    const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (c >= p) return;
    auto keyat = [X, p, c](int k) { return make_key(X[(int64_t)k * p + c], (uint32_t)k); };
    const int cap = n < 32 ? 32 : n;
    uint64_t* buf = ws + (int64_t)c * cap;
    const uint64_t T = warp_select_column(keyat, n, n, s, 0ull, ~0ull, buf, cap, lane);
    const uint32_t tabs = (uint32_t)(T >> 32);
    // emission: strictly-above rows in row order, then tied kept rows (_kernels.py:86-96)
    int w = 0;
    int32_t* ro = rows_out + (int64_t)c * s;
    float* vo = vals_out + (int64_t)c * s;
    for (int pass = 0; pass < 2; ++pass) {
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            bool take = false;
            float x = 0.f;
            if (k < n) {
                x = X[(int64_t)k * p + c];
                const uint64_t kk = make_key(x, (uint32_t)k);
                const uint32_t a = abs_bits(x);
                take = (kk >= T) && (pass == 0 ? (a > tabs) : (a == tabs));
            }
            const uint32_t bal = __ballot_sync(CALS_FULL_MASK, take);
            if (take) {
                const int pos = w + __popc(bal & lanemask_lt());
                ro[pos] = k;
                vo[pos] = x;
            }
            w += __popc(bal);
        }
    }
}

// ---- public sketch on float64 input (core.py:95-115), exact ranks ----------
// rank(i) = #{j : |x_j| > |x_i|  or  (|x_j| == |x_i| and j < i)} -- the
// reference's order (|x| descending, ties to the smaller row); kept = rank < s.
// O(n^2) per column with the column staged through shared memory in tiles;
// this serves the public single-slice API, not the fit.
__global__ void __launch_bounds__(256) ces_rank_f64_kernel(const double* __restrict__ X, int n, int p, int s,
                                                           uint8_t* __restrict__ kept) {
    __shared__ double tile[256];
    const int c = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const double xi = i < n ? fabs(X[(int64_t)i * p + c]) : 0.0;
    int rank = 0;
    for (int j0 = 0; j0 < n; j0 += 256) {
        const int j = j0 + threadIdx.x;
        tile[threadIdx.x] = j < n ? fabs(X[(int64_t)j * p + c]) : -1.0;
        __syncthreads();
        const int jn = min(256, n - j0);
        for (int t = 0; t < jn; ++t) {
            const double xj = tile[t];
            rank += (xj > xi) || (xj == xi && j0 + t < i);
        }
        __syncthreads();
    }
    if (i < n) kept[(int64_t)c * n + i] = rank < s;
}

// Emission in the reference order: kept rows with |x| > t in row order, then
// kept rows with |x| == t (t = smallest kept magnitude), one warp per column.
__global__ void __launch_bounds__(256) ces_emit_f64_kernel(const double* __restrict__ X, int n, int p, int s,
                                                           const uint8_t* __restrict__ kept,
                                                           int32_t* __restrict__ rows_out) {
    const int lane = threadIdx.x & 31;
    const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (c >= p) return;
    const uint8_t* kc = kept + (int64_t)c * n;
    double t = INFINITY;
    for (int k = lane; k < n; k += 32)
        if (kc[k]) t = fmin(t, fabs(X[(int64_t)k * p + c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmin(t, __shfl_xor_sync(CALS_FULL_MASK, t, o));
    int w = 0;
    int32_t* ro = rows_out + (int64_t)c * s;
    for (int pass = 0; pass < 2; ++pass) {
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            bool take = false;
            if (k < n && kc[k]) {
                const double a = fabs(X[(int64_t)k * p + c]);
                take = pass == 0 ? (a > t) : (a == t);
            }
            const uint32_t bal = __ballot_sync(CALS_FULL_MASK, take);
            if (take) ro[w + __popc(bal & lanemask_lt())] = k;
            w += __popc(bal);
        }
    }
}

// ---- public single-row update (core.py:134-157) ---------------------------
__global__ void __launch_bounds__(256) update_core_kernel(const double* __restrict__ X, int n, int p,
                                                          const int64_t* __restrict__ col_ptr,
                                                          const int32_t* __restrict__ rows, const double* __restrict__ y,
                                                          double lam_n, int complete, double* w_out, int32_t* status) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_piv[1];
    const int gs = p + 1, nout = p * gs, tid = threadIdx.x, nt = blockDim.x;
    double* G = reinterpret_cast<double*>(smem);
    double* W = G + nout;
    double* x = W + nout;
    for (int e = tid; e < nout; e += nt) {
        const int c = e / gs, f = e - c * gs;
        double acc = 0.0;
        if (complete) {
            for (int k = 0; k < n; ++k) {
                const double xc = X[(int64_t)k * p + c];
                const double xf = (f < p) ? X[(int64_t)k * p + f] : y[k];
                acc = fma(xc, xf, acc);
            }
        } else {
            for (int64_t q = col_ptr[c]; q < col_ptr[c + 1]; ++q) {
                const int k = rows[q];
                const double xc = X[(int64_t)k * p + c];
                const double xf = (f < p) ? X[(int64_t)k * p + f] : y[k];
                acc = fma(xc, xf, acc);
            }
        }
        G[e] = acc + ((c == f) ? lam_n : 0.0);
    }
    __syncthreads();
    for (int e = tid; e < nout; e += nt) W[e] = G[e];
    __syncthreads();
    int st = CALS_ROW_OK;
    int bad = block_lu_solve<double>(W, p, complete != 0, x, s_piv);
    if (bad) {
        double tr = 0.0;
        for (int c = 0; c < p; ++c) tr += G[c * gs + c];
        const double jit = 1e-10 * tr / (double)p;
        for (int e = tid; e < nout; e += nt) {
            const int c = e / gs, f = e - c * gs;
            W[e] = G[e] + ((c == f) ? jit : 0.0);
        }
        __syncthreads();
        bad = block_lu_solve<double>(W, p, complete != 0, x, s_piv);
        st = bad ? CALS_ROW_SINGULAR : CALS_ROW_JITTERED;
    }
    for (int f = tid; f < p; f += nt) w_out[f] = x[f];
    if (tid == 0) status[0] = st;
}

// ---- predict_entries (als.py:143-152) ---------------------------------------
__global__ void __launch_bounds__(256) predict_entries_kernel(const float* __restrict__ U, const float* __restrict__ M,
                                                              int nf, int ldu, int ldm, const int64_t* __restrict__ users,
                                                              const int64_t* __restrict__ items, int64_t n,
                                                              double* __restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const float* u = U + users[e] * ldu;
        const float* m = M + items[e] * ldm;
        double acc = 0.0;
        for (int f = 0; f < nf; ++f) acc = fma((double)u[f], (double)m[f], acc);
        out[e] = acc;
    }
}

// float64 factors (the reference's FactorPair precision, als.py:40-49): the
// evaluation metrics rank by these scores, so they are not narrowed to fp32.
__global__ void __launch_bounds__(256) predict_entries_f64_kernel(const double* __restrict__ U,
                                                                  const double* __restrict__ M, int nf, int ldu,
                                                                  int ldm, const int64_t* __restrict__ users,
                                                                  const int64_t* __restrict__ items, int64_t n,
                                                                  double* __restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const double* u = U + users[e] * ldu;
        const double* m = M + items[e] * ldm;
        double acc = 0.0;
        for (int f = 0; f < nf; ++f) acc = fma(u[f], m[f], acc);
        out[e] = acc;
    }
}

// ---- predict_full (als.py:155-157): out = U M^T, float64 -------------------
// 16 x 16 threads, a 64 x 64 output tile per CTA (4 x 4 per thread), K in steps of 16
// through shared memory (transposed tiles: conflict-free reads along the output rows).
__global__ void __launch_bounds__(256) predict_full_f64_kernel(const double* __restrict__ U, const double* __restrict__ M,
                                                               int64_t nu, int64_t ni, int nf, int ldu, int ldm,
                                                               double* __restrict__ out, int64_t ldo) {
    __shared__ double su[16][65], sm[16][65];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t u0 = (int64_t)blockIdx.y * 64, i0 = (int64_t)blockIdx.x * 64;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < nf; k0 += 16) {
        __syncthreads();
        for (int e = threadIdx.x; e < 64 * 16; e += 256) {
            const int r = e >> 4, k = e & 15;
            su[k][r] = (u0 + r < nu && k0 + k < nf) ? U[(u0 + r) * ldu + k0 + k] : 0.0;
            sm[k][r] = (i0 + r < ni && k0 + k < nf) ? M[(i0 + r) * ldm + k0 + k] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            double a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a[q] = su[k][ty + 16 * q];
                b[q] = sm[k][tx + 16 * q];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int w = 0; w < 4; ++w) acc[q][w] = fma(a[q], b[w], acc[q][w]);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int64_t u = u0 + ty + 16 * q, i = i0 + tx + 16 * w;
            if (u < nu && i < ni) out[u * ldo + i] = acc[q][w];
        }
}

// ---- ranking metrics per user (metrics.py:89-147) --------------------------
// One warp per user segment; entry i's predicted rank = entries of the segment with a larger
// score, or an equal score and an earlier position (items ascend inside a segment, so that
// is the reference's smaller-item tie rule); ideal rank likewise by truth.
__global__ void __launch_bounds__(256) rank_metrics_kernel(const int64_t* __restrict__ seg, int64_t n_seg,
                                                           const int32_t* __restrict__ perm,
                                                           const double* __restrict__ truths,
                                                           const double* __restrict__ scores, int k_hit, double thr,
                                                           int k_ndcg, double* __restrict__ qual,
                                                           double* __restrict__ hit, double* __restrict__ ratio,
                                                           double* __restrict__ used) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = w0; u < n_seg; u += nw) {
        const int64_t lo = seg[u], hi = seg[u + 1];
        double dcg = 0.0, idcg = 0.0;
        bool rel_any = false, hit_any = false;
        for (int64_t i = lo + lane; i < hi; i += 32) {
            const int32_t pi = perm[i];
            const double si = scores[pi], ti = truths[pi];
            int rs = 0, rt = 0;
            for (int64_t j = lo; j < hi; ++j) {
                const int32_t pj = perm[j];
                const double sj = scores[pj], tj = truths[pj];
                rs += (sj > si || (sj == si && j < i)) ? 1 : 0;
                rt += (tj > ti || (tj == ti && j < i)) ? 1 : 0;
            }
            if (rs < k_ndcg) dcg += ti * (1.0 / log2((double)(rs + 2)));
            if (rt < k_ndcg) idcg += ti * (1.0 / log2((double)(rt + 2)));
            const bool rel = ti >= thr;
            rel_any |= rel;
            hit_any |= rel && rs < k_hit;
        }
        dcg = warp_sum_d(dcg);
        idcg = warp_sum_d(idcg);
        const bool q = __any_sync(CALS_FULL_MASK, rel_any), h = __any_sync(CALS_FULL_MASK, hit_any);
        if (lane == 0) {
            const bool us = idcg > 0.0;
            qual[u] = q ? 1.0 : 0.0;
            hit[u] = (q && h) ? 1.0 : 0.0;
            used[u] = us ? 1.0 : 0.0;
            ratio[u] = us ? dcg / idcg : 0.0;
        }
    }
}

}  // namespace cals
