// sweep_small.cu -- the staged-slice (shared-memory) tier of the half-sweep,
// plus the per-sweep quantile table that seeds its selection brackets.
//
// Phase A (this file), one CTA per regression, persistent over a
// length-sorted row list:
//   stage   X = source[idx] (cp.async, 16-byte rows) and y into shared memory
//                                                              (core.py:215,220)
//   resid   optional fused residual of the PREVIOUS iteration's row of this
//           regression: sum_k (y_k - X_k . w_old)^2            (_kernels.py:219-230)
//   select  per column the s_i largest keys -> selection bitmap (_kernels.py:26-120)
//   gram    sparse G = X*^T X + lam*n*I, b = X*^T y -> global  (_kernels.py:123-146)
// Phase B (sweep_solve.cu) solves the batch of normal equations.
#include "gram.cuh"
#include "select.cuh"
#include "sweep_common.cuh"

namespace cals {

// ---------------------------------------------------------------------------
// Quantile table: per column, abs-bit quantiles of the source values seen by
// this side's ratings (a rating-weighted sample at QS deterministic positions).
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
    for (int size = 2; size <= QS; size <<= 1) {  // bitonic sort, descending
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < QS / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool desc = (lo & size) == 0;
                const uint32_t a = sbuf[lo], b = sbuf[hi];
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

// Threshold key of column c (warp-level, see select.cuh).  `cl` (shared
// address) holds the column's bracket candidates and is left intact, `scr`
// is this warp's scratch list.
__device__ __forceinline__ uint64_t resolve_column(const SweepArgs& A, uint32_t xs, int sx, int c, int n, int s,
                                                   bool use_tab, int above, int in, uint32_t cl, uint32_t scr,
                                                   bool& fallback, int lane) {
    fallback = false;
    if (!use_tab) {
        IdxList Lst{xs, sx, c, scr, true};
        return warp_select_idx(Lst, n, s, 0ull, ~0ull, lane);
    }
    const uint32_t* qc = A.qtab + (size_t)c * (kQ + 1);
    int jhi, jlo;
    table_levels(n, s, A.delta_tab, jhi, jlo);
    const uint32_t hib = qc[jhi], lob = qc[jlo];
    uint64_t hik = hi_key_of(hib), lok = (uint64_t)lob << 32;
    if (above < s && s <= above + in && in <= kCap && lok < hik) {
        for (int i = lane; i < in; i += 32) sts_u16(scr + 2u * i, lds_u16(cl + 2u * i));
        __syncwarp();
        IdxList Lst{xs, sx, c, scr, false};
        int m = in, need = s - above;
        warp_prenarrow(Lst, m, need, lok, hik, qc, jhi, jlo, lane);
        return warp_select_idx(Lst, m, need, lok, hik, lane);
    }
    // the table bracket missed (or overflowed): exact column-mode search
    fallback = true;
    uint64_t rlo, rhi;
    int m, need;
    if (above >= s) { rlo = hik; rhi = ~0ull; m = above; need = s; }
    else if (above + in < s) { rlo = 0ull; rhi = lok; m = n - above - in; need = s - above - in; }
    else { rlo = lok; rhi = hik; m = in; need = s - above; }
    auto keyat = [xs, sx, c](int k) { return make_key(lds_f32(xs + 4u * (uint32_t)(k * sx + c)), (uint32_t)k); };
    uint64_t* keybuf = reinterpret_cast<uint64_t*>(__cvta_shared_to_generic(scr));
    return warp_select_column(keyat, n, m, need, rlo, rhi, keybuf, (kCap * (int)sizeof(uint16_t)) / 8, lane);
}

// ---------------------------------------------------------------------------
// Phase A kernel (blockDim 128 or 256).  rows / n_list: this batch; the
// normal equations of rows[li] go to A.gbuf + li * nf * (nf+1).
// N: longest row of the batch; S: largest budget among its incomplete rows.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2) small_gram_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                                 int64_t n_list, int N, int S) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int cnt_above[CALS_MAX_NF_DEV], cnt_in[CALS_MAX_NF_DEV];
    __shared__ uint64_t thr[CALS_MAX_NF_DEV];
    __shared__ float wold[CALS_MAX_NF_DEV];
    __shared__ double red[32];

    const int nf = A.nf;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const T1Layout L(N, S, nf, nt);
    const int sx = L.sx, mw = L.mw, gs = nf + 1;
    float* Xs = reinterpret_cast<float*>(smem);
    float* ys = reinterpret_cast<float*>(smem + L.xs);
    uint32_t* mb = reinterpret_cast<uint32_t*>(smem + L.xs + L.ys);
    const uint32_t s_xs = smem_u32(smem);
    const uint32_t s_ys = s_xs + (uint32_t)L.xs;
    const uint32_t s_mb = s_ys + (uint32_t)L.ys;
    const uint32_t s_cand = s_mb + (uint32_t)L.mb;
    const uint32_t s_lists = s_cand;  // reused once the thresholds are known
    const uint32_t s_scr = s_cand + (uint32_t)L.region + 2u * (uint32_t)(warp * kCap);
    const uint32_t rowb = 4u * (uint32_t)sx;
    const FastDiv fq((uint32_t)xs_chunks(nf));
    const bool ballot_bits = (32 % nf == 0) || (nf % 32 == 0);

    for (int64_t li = blockIdx.x; li < n_list; li += gridDim.x) {
        const int row = rows[li];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        const bool full = (s >= n);

        // ---- stage the slice [X | y]; clear the bitmap ----
        stage_slice(A, lo, 0, n, Xs, ys, fq);
        for (int e = tid; e < n * mw; e += nt) mb[e] = 0u;
        if (tid < nf) {
            cnt_above[tid] = 0;
            cnt_in[tid] = 0;
            if (A.tgt_old != nullptr) wold[tid] = A.tgt_old[(int64_t)row * A.ld_old + tid];
        }
        __syncthreads();

        // ---- fused residual of the previous iteration's row (als.py:287-288) ----
        if (A.rss_rows != nullptr) {
            double acc = 0.0;
            for (int k = tid; k < n; k += nt) {
                const uint32_t rb = s_xs + (uint32_t)k * rowb;
                double pred = 0.0;
                for (int f = 0; f < nf; ++f) pred = fma((double)lds_f32(rb + 4u * f), (double)wold[f], pred);
                const double d = (double)lds_f32(s_ys + 4u * k) - pred;
                acc = fma(d, d, acc);
            }
            acc = block_sum_d(acc, red);
            if (tid == 0) A.rss_rows[row] = acc;
        }

        // ---- selection: threshold key per column, kept-set bitmap ----
        if (!full) {
            const bool use_tab = (n > kCap) && (A.qtab != nullptr);
            if (use_tab) {
                // one pass: keys above the table bracket go straight into the
                // bitmap (ballots), keys inside it are listed per column
                const int per = nt / nf;
                const int c = tid % nf, j = tid / nf;
                const bool active = tid < per * nf;
                uint32_t hib = kAbsInf, lob = kAbsInf;
                if (active) table_bracket(A.qtab + (size_t)c * (kQ + 1), n, s, A.delta_tab, hib, lob);
                const uint32_t cl = s_cand + 2u * (uint32_t)(c * kCap);
                int above = 0;
                const int iters = (n + per - 1) / per;
                const int rsh = (lane / (nf <= 32 ? nf : 32)) * nf;
                const uint32_t rmask = nf >= 32 ? 0xffffffffu : ((1u << nf) - 1u);
                const bool writer = nf <= 32 ? (c == 0) : (lane == 0);
                uint32_t addr = s_xs + (uint32_t)j * rowb + 4u * (uint32_t)c;
                const uint32_t astep = (uint32_t)per * rowb;
                int k = j;
                for (int it = 0; it < iters; ++it, k += per, addr += astep) {
                    const bool ok = active && k < n;
                    const uint32_t a = ok ? (__float_as_uint(lds_f32(addr)) & 0x7FFFFFFFu) : 0u;
                    const bool ab = ok && a >= hib;
                    above += ab;
                    if (ok && a >= lob && a < hib) {
                        const int slot = atomicAdd(&cnt_in[c], 1);
                        if (slot < kCap) sts_u16(cl + 2u * slot, k);
                    }
                    if (ballot_bits) {
                        const uint32_t bal = __ballot_sync(CALS_FULL_MASK, ab);
                        if (writer && ok) sts_u32(s_mb + 4u * (uint32_t)(k * mw + (c >> 5)), (bal >> rsh) & rmask);
                    } else if (ab) {
                        atomicOr(&mb[k * mw + (c >> 5)], 1u << (c & 31));
                    }
                }
                if (active) atomicAdd(&cnt_above[c], above);
                __syncthreads();
            }
            for (int c = warp; c < nf; c += nwarps) {
                bool fallback;
                const uint32_t cl = s_cand + 2u * (uint32_t)(c * kCap);
                const uint64_t T = resolve_column(A, s_xs, sx, c, n, s, use_tab, cnt_above[c], cnt_in[c], cl, s_scr,
                                                  fallback, lane);
                if (lane == 0) thr[c] = T;
                const uint32_t bit = 1u << (c & 31);
                uint32_t* mcol = mb + (c >> 5);
                const uint32_t xcol = s_xs + 4u * (uint32_t)c;
                if (!use_tab || fallback) {
                    // (re)derive column c entirely: kept iff key >= T
                    for (int k = lane; k < n; k += 32) {
                        const bool keep = make_key(lds_f32(xcol + (uint32_t)k * rowb), (uint32_t)k) >= T;
                        if (keep) atomicOr(mcol + k * mw, bit);
                        else if (fallback) atomicAnd(mcol + k * mw, ~bit);
                    }
                } else {
                    // bracket candidates at or above the threshold join the kept set
                    const int in = cnt_in[c];
                    for (int i = lane; i < in; i += 32) {
                        const uint32_t k = lds_u16(cl + 2u * i);
                        if (make_key(lds_f32(xcol + k * rowb), k) >= T) atomicOr(mcol + k * mw, bit);
                    }
                }
            }
        } else if (A.thr_keys != nullptr) {
            // complete sketch: every row kept; report the smallest key per column
            for (int c = warp; c < nf; c += nwarps) {
                uint64_t mn = ~0ull;
                for (int k = lane; k < n; k += 32) {
                    const uint64_t kk = make_key(lds_f32(s_xs + (uint32_t)k * rowb + 4u * c), (uint32_t)k);
                    mn = kk < mn ? kk : mn;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t t = __shfl_xor_sync(CALS_FULL_MASK, mn, o);
                    mn = t < mn ? t : mn;
                }
                if (lane == 0) thr[c] = mn;
            }
        }
        __syncthreads();

        // ---- sparse Gram -> global normal equations ----
        const float lam_n = (float)(A.lam * (double)n);
        sparse_gram(s_xs, sx, s_ys, s_mb, mw, n, nf, s, full, s_lists, S > 0 ? S : 1, lam_n,
                    A.gbuf + (size_t)li * nf * gs, warp, nwarps, lane);
        if (A.thr_keys != nullptr)
            for (int c = tid; c < nf; c += nt) A.thr_keys[(int64_t)row * nf + c] = thr[c];
        __syncthreads();
    }
}

}  // namespace cals
