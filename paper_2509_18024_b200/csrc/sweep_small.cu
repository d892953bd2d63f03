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

// One warp selects column c end to end: threshold key T (the s-th largest
// key, select.cuh), the column's kept-set bitmap words (bit k of word k/32 =
// key(k) >= T) and its ascending kept-row list.  `cand` / `scr` are this
// warp's candidate and scratch lists (shared addresses, kCap entries each).
__device__ __forceinline__ uint64_t select_column(const SweepArgs& A, uint32_t xs, int sx, int c, int n, int s,
                                                  uint32_t words, uint32_t list, uint32_t cand, uint32_t scr,
                                                  int lane) {
    const uint32_t rowb = 4u * (uint32_t)sx;
    const uint32_t xcol = xs + 4u * (uint32_t)c;
    auto keyat = [xcol, rowb](int k) { return make_key(lds_f32(xcol + (uint32_t)k * rowb), (uint32_t)k); };
    const int nwords = (n + 31) >> 5;
    uint64_t T;
    bool rebuild = true;  // derive all bitmap words from T
    if (n <= kCap || A.qtab == nullptr) {
        IdxList Lst{xs, sx, c, scr, true};
        T = warp_select_idx(Lst, n, s, 0ull, ~0ull, lane);
    } else {
        // one pass over the column: keys above the table bracket go straight
        // into the bitmap, keys inside it are listed (ascending k)
        const uint32_t* qc = A.qtab + (size_t)c * (kQ + 1);
        int jhi, jlo;
        table_levels(n, s, A.delta_tab, jhi, jlo);
        const uint32_t hib = qc[jhi], lob = qc[jlo];
        const uint64_t hik = hi_key_of(hib), lok = (uint64_t)lob << 32;
        int above = 0, nin = 0;
        uint32_t addr = xcol + (uint32_t)lane * rowb;
        const uint32_t astep = 32u * rowb;
        for (int k0 = 0; k0 < n; k0 += 32, addr += astep) {
            const int k = k0 + lane;
            const bool ok = k < n;
            const uint32_t a = ok ? (__float_as_uint(lds_f32(addr)) & 0x7FFFFFFFu) : 0u;
            const uint32_t bA = __ballot_sync(CALS_FULL_MASK, ok && a >= hib);
            const bool in = ok && a >= lob && a < hib;
            const uint32_t bI = __ballot_sync(CALS_FULL_MASK, in);
            if (lane == 0) sts_u32(words + 4u * (uint32_t)(k0 >> 5), bA);
            if (in) {
                const int p = nin + __popc(bI & lanemask_lt());
                if (p < kCap) sts_u16(cand + 2u * (uint32_t)p, (uint32_t)k);
            }
            above += __popc(bA);
            nin += __popc(bI);
        }
        __syncwarp();
        if (above < s && s <= above + nin && nin <= kCap && lok < hik) {
            for (int i = lane; i < nin; i += 32) sts_u16(scr + 2u * i, lds_u16(cand + 2u * i));
            __syncwarp();
            IdxList Lst{xs, sx, c, scr, false};
            int m = nin, need = s - above;
            uint64_t lo = lok, hi = hik;
            warp_prenarrow(Lst, m, need, lo, hi, qc, jhi, jlo, lane);
            T = warp_select_idx(Lst, m, need, lo, hi, lane);
            // bracket candidates at or above T join the kept set (above keys already in)
            for (int i = lane; i < nin; i += 32) {
                const uint32_t k = lds_u16(cand + 2u * i);
                if (keyat((int)k) >= T) atoms_or(words + 4u * (k >> 5), 1u << (k & 31));
            }
            __syncwarp();
            rebuild = false;
        } else {
            // the table bracket missed (or overflowed): exact column-mode search
            uint64_t rlo, rhi;
            int m, need;
            if (above >= s) { rlo = hik; rhi = ~0ull; m = above; need = s; }
            else if (above + nin < s) { rlo = 0ull; rhi = lok; m = n - above - nin; need = s - above - nin; }
            else { rlo = lok; rhi = hik; m = nin; need = s - above; }
            uint64_t* keybuf = reinterpret_cast<uint64_t*>(__cvta_shared_to_generic(scr));
            T = warp_select_column(keyat, n, m, need, rlo, rhi, keybuf, (kCap * (int)sizeof(uint16_t)) / 8, lane);
        }
    }
    if (rebuild) {
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            const uint32_t b = __ballot_sync(CALS_FULL_MASK, k < n && keyat(k) >= T);
            if (lane == 0) sts_u32(words + 4u * (uint32_t)(k0 >> 5), b);
        }
        __syncwarp();
    }
    bitmap_to_list(words, nwords, list, lane);
    return T;
}

// ---------------------------------------------------------------------------
// Phase A kernel (blockDim 128 or 256).  rows / n_list: this batch; the
// normal equations of rows[li] go to A.gbuf + li * nf * (nf+1).
// N: longest row of the batch; S: largest budget among its incomplete rows.
// Warp w owns columns w, w + nwarps, ... of every row: selection, bitmap,
// list and Gram rows of a column never leave its warp, so a row costs two
// block barriers (after staging, before the next row's staging).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2) small_gram_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                                 int64_t n_list, int N, int S) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t thr[CALS_MAX_NF_DEV];
    __shared__ float wold[CALS_MAX_NF_DEV];
    __shared__ double red[32];

    const int nf = A.nf;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const T1Layout L(N, S, nf, nt);
    const int sx = L.sx, gs = nf + 1;
    const int Smax = S > 0 ? S : 1;
    float* Xs = reinterpret_cast<float*>(smem);
    float* ys = reinterpret_cast<float*>(smem + L.xs);
    const uint32_t s_xs = smem_u32(smem);
    const uint32_t s_ys = s_xs + (uint32_t)L.xs;
    const uint32_t s_mb = s_ys + (uint32_t)L.ys;
    const uint32_t s_lists = s_mb + (uint32_t)L.mb;
    const uint32_t s_cand = s_lists + (uint32_t)L.lists + 2u * (uint32_t)(warp * kCap);
    const uint32_t s_scr = s_lists + (uint32_t)L.lists + (uint32_t)L.cand + 2u * (uint32_t)(warp * kCap);
    const uint32_t rowb = 4u * (uint32_t)sx;
    const FastDiv fq((uint32_t)xs_chunks(nf));
    const int my_cols = warp < nf ? (nf - 1 - warp) / nwarps + 1 : 0;

    for (int64_t li = blockIdx.x; li < n_list; li += gridDim.x) {
        const int row = rows[li];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        const bool full = (s >= n);

        stage_slice(A, lo, 0, n, Xs, ys, fq);
        if (tid < nf && A.tgt_old != nullptr) wold[tid] = A.tgt_old[(int64_t)row * A.ld_old + tid];
        __syncthreads();

        // ---- fused residual of the previous iteration's row (als.py:287-288) ----
        if (A.rss_rows != nullptr) {
            double acc = 0.0;
            const int nq = xs_chunks(nf);
            for (int k = tid; k < n; k += nt) {
                const uint32_t rb = s_xs + (uint32_t)k * rowb;
                float pred = 0.f;
                for (int q = 0; q < nq; ++q) {
                    const float4 v = lds_f128(rb + 16u * q);
                    const int f = 4 * q;
                    pred = fmaf(v.x, wold[f], pred);
                    if (f + 1 < nf) pred = fmaf(v.y, wold[f + 1], pred);
                    if (f + 2 < nf) pred = fmaf(v.z, wold[f + 2], pred);
                    if (f + 3 < nf) pred = fmaf(v.w, wold[f + 3], pred);
                }
                const double d = (double)lds_f32(s_ys + 4u * k) - (double)pred;
                acc = fma(d, d, acc);
            }
            acc = warp_sum_d(acc);
            if (lane == 0) red[warp] = acc;
        }

        // ---- per owned column: selection -> bitmap -> kept-row list ----
        for (int j = 0; j < my_cols; ++j) {
            const int c = warp + j * nwarps;
            uint64_t T;
            if (!full) {
                T = select_column(A, s_xs, sx, c, n, s, s_mb + 4u * (uint32_t)(c * L.nw),
                                  s_lists + 2u * (uint32_t)(c * Smax), s_cand, s_scr, lane);
            } else {
                T = ~0ull;
                if (A.thr_keys != nullptr) {  // complete sketch: report the smallest key
                    for (int k = lane; k < n; k += 32) {
                        const uint64_t kk = make_key(lds_f32(s_xs + (uint32_t)k * rowb + 4u * c), (uint32_t)k);
                        T = kk < T ? kk : T;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const uint64_t t = __shfl_xor_sync(CALS_FULL_MASK, T, o);
                        T = t < T ? t : T;
                    }
                }
            }
            if (lane == 0) thr[c] = T;
        }

        // ---- sparse Gram of the owned columns -> global normal equations ----
        const float lam_n = (float)(A.lam * (double)n);
        if (my_cols > 0)
            sparse_gram_owned_any(s_xs, sx, s_ys, nf, full ? n : s, full, s_lists, Smax, warp, nwarps, my_cols, lam_n,
                                  A.gbuf + (size_t)li * nf * gs, lane);
        __syncthreads();
        if (A.rss_rows != nullptr && tid == 0) {
            double r = 0.0;
            for (int w = 0; w < nwarps; ++w) r += red[w];
            A.rss_rows[row] = r;
        }
        if (A.thr_keys != nullptr)
            for (int c = tid; c < nf; c += nt) A.thr_keys[(int64_t)row * nf + c] = thr[c];
    }
}

}  // namespace cals
