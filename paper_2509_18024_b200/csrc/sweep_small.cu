// sweep_small.cu -- the staged-slice (shared-memory) tier of the half-sweep,
// plus the per-sweep quantile table that seeds its selection brackets.
//
// One CTA per regression (persistent over a length-sorted row list):
//   gather  X = source[idx] and y into shared memory          (core.py:215,220)
//   select  per column the s_i largest keys                    (_kernels.py:26-120)
//   gram    G = (P.X)^T X + lam*n*I, b = (P.X)^T y              (_kernels.py:123-146)
//   solve   LU with partial pivoting / SPD when s_i == n_i      (core.py:120-131, als.py:184-205)
//   write   target[i] = w; fused residual on the item side      (als.py:286-288, _kernels.py:219-230)
#include "gram.cuh"
#include "select.cuh"
#include "solve.cuh"
#include "sweep_common.cuh"

namespace cals {

// ---------------------------------------------------------------------------
// Quantile table: per column, abs-bit quantiles of the source values seen by
// this side's ratings (a rating-weighted sample, QS deterministic positions).
// qtab[c][0] = kAbsInf (nothing above), qtab[c][kQ] = 0 (everything >= 0).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) quantile_table_kernel(const int32_t* __restrict__ idx, int64_t nnz,
                                                              const float* __restrict__ src, int ld, int QS,
                                                              uint32_t* __restrict__ qtab) {
    extern __shared__ uint32_t sbuf[];
    const int c = blockIdx.x;
    for (int i = threadIdx.x; i < QS; i += blockDim.x) {
        int64_t pos = (int64_t)(((double)i + 0.5) * (double)nnz / (double)QS);
        if (pos >= nnz) pos = nnz - 1;
        sbuf[i] = abs_bits(src[(int64_t)idx[pos] * ld + c]);
    }
    __syncthreads();
    // bitonic sort, descending
    for (int size = 2; size <= QS; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < QS / 2; i += blockDim.x) {
                int lo = 2 * i - (i & (stride - 1));
                int hi = lo + stride;
                bool desc = (lo & size) == 0;
                uint32_t a = sbuf[lo], b = sbuf[hi];
                if ((a < b) == desc) { sbuf[lo] = b; sbuf[hi] = a; }
            }
            __syncthreads();
        }
    }
    uint32_t* q = qtab + (size_t)c * (kQ + 1);
    for (int j = threadIdx.x; j <= kQ; j += blockDim.x) {
        uint32_t v;
        if (j == 0) v = kAbsInf;
        else if (j == kQ) v = 0u;
        else v = sbuf[(size_t)j * QS / kQ];
        q[j] = v;
    }
}

// ---------------------------------------------------------------------------
// Staged-slice half-sweep kernel.
// NFP: 8/16/32 -> warp-register LU; 0 -> block LU in shared memory (nf > 32).
// ---------------------------------------------------------------------------
template <int NFP>
__global__ void __launch_bounds__(kThreads, 2) small_sweep_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                               int64_t n_list, int N) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int cnt_above[CALS_MAX_NF_DEV], cnt_in[CALS_MAX_NF_DEV];
    __shared__ uint64_t thr[CALS_MAX_NF_DEV];
    __shared__ float wv[CALS_MAX_NF_DEV];
    __shared__ double red[32];
    __shared__ int s_piv[1];
    __shared__ int s_stat[1];

    const int nf = A.nf;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const T1Layout L(N, nf, nt);
    const int sx = L.sx, mw = L.mw, gs = nf + 1;
    float* Xs = reinterpret_cast<float*>(smem);
    unsigned char* R = smem + L.xs;
    uint16_t* cand = reinterpret_cast<uint16_t*>(R);
    uint32_t* mb = reinterpret_cast<uint32_t*>(R);
    float* G = reinterpret_cast<float*>(R + L.mb);
    float* W = reinterpret_cast<float*>(R + L.mb + L.g);
    float* scratch = reinterpret_cast<float*>(R + L.mb + L.g + L.w);
    const FastDiv fdiv((uint32_t)nf);

    for (int64_t li = blockIdx.x; li < n_list; li += gridDim.x) {
        const int row = rows[li];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        const bool full = (s >= n);

        // ---- gather the slice [X | y] (coalesced within each source row) ----
        const int nel = n * nf;
#pragma unroll 4
        for (int e = tid; e < nel; e += nt) {
            const int k = (int)fdiv.div((uint32_t)e);
            const int c = e - k * nf;
            Xs[k * sx + c] = __ldg(A.src + (int64_t)__ldg(A.idx + lo + k) * A.ld_src + c);
        }
        for (int k = tid; k < n; k += nt) {
            Xs[k * sx + nf] = __ldg(A.val + lo + k);
            for (int c = nf + 1; c < sx; ++c) Xs[k * sx + c] = 0.f;
        }
        if (tid < nf) { cnt_above[tid] = 0; cnt_in[tid] = 0; }
        __syncthreads();

        // ---- selection: threshold key per column ----
        if (!full) {
            const bool use_tab = (n > kCap) && (A.qtab != nullptr);
            if (use_tab) {
                const int per = nt / nf;  // threads per column
                if (tid < per * nf) {
                    const int c = tid % nf, j = tid / nf;
                    uint32_t hib, lob;
                    table_bracket(A.qtab + (size_t)c * (kQ + 1), n, s, A.delta_tab, hib, lob);
                    int above = 0;
                    uint16_t* cl = cand + c * kCap;
                    for (int k = j; k < n; k += per) {
                        const uint32_t a = abs_bits(Xs[k * sx + c]);
                        above += (a >= hib);
                        if (a >= lob && a < hib) {
                            int slot = atomicAdd(&cnt_in[c], 1);
                            if (slot < kCap) cl[slot] = (uint16_t)k;
                        }
                    }
                    atomicAdd(&cnt_above[c], above);
                }
                __syncthreads();
            }
            for (int c = warp; c < nf; c += nwarps) {
                uint64_t T;
                uint16_t* cl = cand + c * kCap;
                if (!use_tab) {
                    IdxList<uint16_t> Lst{Xs, sx, c, cl, true};
                    T = warp_select_idx(Lst, n, s, 0ull, ~0ull, lane);
                } else {
                    uint32_t hib, lob;
                    table_bracket(A.qtab + (size_t)c * (kQ + 1), n, s, A.delta_tab, hib, lob);
                    const uint64_t hik = hi_key_of(hib), lok = (uint64_t)lob << 32;
                    const int above = cnt_above[c], in = cnt_in[c];
                    if (above < s && s <= above + in && in <= kCap && lok < hik) {
                        IdxList<uint16_t> Lst{Xs, sx, c, cl, false};
                        T = warp_select_idx(Lst, in, s - above, lok, hik, lane);
                    } else {
                        uint64_t rlo, rhi;
                        int m, need;
                        if (above >= s) { rlo = hik; rhi = ~0ull; m = above; need = s; }
                        else if (above + in < s) { rlo = 0ull; rhi = lok; m = n - above - in; need = s - above - in; }
                        else { rlo = lok; rhi = hik; m = in; need = s - above; }
                        const float* Xc = Xs;
                        auto keyat = [Xc, sx, c](int k) { return make_key(Xc[k * sx + c], (uint32_t)k); };
                        T = warp_select_column(keyat, n, m, need, rlo, rhi, reinterpret_cast<uint64_t*>(cl),
                                               (kCap * (int)sizeof(uint16_t)) / 8, lane);
                    }
                }
                if (lane == 0) thr[c] = T;
            }
        } else if (A.thr_keys != nullptr) {
            // complete sketch: every row kept; report the smallest key per column
            for (int c = warp; c < nf; c += nwarps) {
                uint64_t mn = ~0ull;
                for (int k = lane; k < n; k += 32) {
                    uint64_t kk = make_key(Xs[k * sx + c], (uint32_t)k);
                    mn = kk < mn ? kk : mn;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    uint64_t t = __shfl_xor_sync(CALS_FULL_MASK, mn, o);
                    mn = t < mn ? t : mn;
                }
                if (lane == 0) thr[c] = mn;
            }
        }
        __syncthreads();

        // ---- mask + Gram ----
        build_mask(Xs, sx, n, nf, thr, full, mb, mw);
        __syncthreads();
        tile_gram(Xs, sx, mb, mw, n, nf, G, scratch);
        const float lam_n = (float)(A.lam * (double)n);
        for (int c = tid; c < nf; c += nt) G[c * gs + c] += lam_n;
        __syncthreads();

        // ---- solve ----
        const int st = solve_row<NFP>(G, nf, full, wv, W, A.retry_ws + (size_t)blockIdx.x * A.retry_stride, s_piv,
                                      s_stat);

        // ---- write back, residual, diagnostics ----
        if (st != CALS_ROW_SINGULAR)
            for (int f = tid; f < nf; f += nt) A.tgt[(int64_t)row * A.ld_tgt + f] = wv[f];
        if (tid == 0) { A.status[row] = st; report_status(A, row, st); }
        if (A.thr_keys != nullptr)
            for (int c = tid; c < nf; c += nt) A.thr_keys[(int64_t)row * nf + c] = thr[c];
        if (A.rss_rows != nullptr) {
            double acc = 0.0;
            for (int k = tid; k < n; k += nt) {
                double pred = 0.0;
                for (int f = 0; f < nf; ++f) pred = fma((double)Xs[k * sx + f], (double)wv[f], pred);
                const double d = (double)Xs[k * sx + nf] - pred;
                acc = fma(d, d, acc);
            }
            acc = block_sum_d(acc, red);
            if (tid == 0) A.rss_rows[row] = (st == CALS_ROW_SINGULAR) ? 0.0 : acc;
        }
        __syncthreads();
    }
}

// explicit instantiations used by the launcher
template __global__ void small_sweep_kernel<8>(SweepArgs, const int32_t*, int64_t, int);
template __global__ void small_sweep_kernel<16>(SweepArgs, const int32_t*, int64_t, int);
template __global__ void small_sweep_kernel<32>(SweepArgs, const int32_t*, int64_t, int);
template __global__ void small_sweep_kernel<0>(SweepArgs, const int32_t*, int64_t, int);

}  // namespace cals
