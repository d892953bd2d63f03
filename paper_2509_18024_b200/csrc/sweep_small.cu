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

// ---------------------------------------------------------------------------
// Phase A kernel (blockDim 128 or 256).  rows / n_list: this batch; the
// normal equations of rows[li] go to A.gbuf + li * nf * (nf+1).
// N: longest row of the batch; S: largest budget among its incomplete rows.
//
// Selection runs SIMT across columns: thread (c, slot) scans column c over
// its slot's k-range (sequential, conflict-free shared loads), writes the
// "above the table bracket" bits of its own bitmap words, lists the keys in
// the bracket and counts them against the table levels inside the bracket.
// One thread per column then picks the sub-bucket holding the target rank,
// the slot threads forward that sub-bucket's keys (typically ~10), and one
// warp per column sorts them to read off the threshold key T.  Keys of the
// bracket at or above T join the bitmap; lists are built from the bitmap.
// Any miss (bracket, capacity) falls back to an exact warp search.
// ---------------------------------------------------------------------------
template <int CPL>
__global__ void __launch_bounds__(512, 1) small_gram_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                                 int64_t n_list, int N, int S) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t thr[CALS_MAX_NF_DEV], c_lo[CALS_MAX_NF_DEV], c_hi[CALS_MAX_NF_DEV];
    __shared__ int c_need[CALS_MAX_NF_DEV], c_flag[CALS_MAX_NF_DEV], c_fc[CALS_MAX_NF_DEV];
    __shared__ float wold[CALS_MAX_NF_DEV];
    __shared__ double red[32];
    __shared__ __align__(8) unsigned long long s_mbar;
    const uint32_t mbar = smem_u32(&s_mbar);
    uint32_t phase = 0;
    if (threadIdx.x == 0) mbar_init(mbar, 1);
    __syncthreads();

    const int nf = A.nf;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const T1Layout L(N, S, nf, nt);
    const SlotMap SM(nf, nt);
    const int sx = L.sx, gs = nf + 1, NW = L.nw, CAPS = L.caps, NFP = SM.NFP, P = SM.P;
    const int Smax = S > 0 ? S : 1;
    float* Xs = reinterpret_cast<float*>(smem);
    float* ys = reinterpret_cast<float*>(smem + L.xs);
    const uint32_t s_xs = smem_u32(smem);
    const uint32_t s_ys = s_xs + (uint32_t)L.xs;
    const uint32_t s_mb = s_ys + (uint32_t)L.ys;
    const uint32_t s_lists = s_mb + (uint32_t)L.mb;
    const uint32_t s_cand = s_lists + (uint32_t)L.lists;
    const uint32_t s_lvl = s_cand + (uint32_t)L.cand;
    const uint32_t s_cnt = s_lvl + (uint32_t)L.lvl;
    const uint32_t s_fb = s_cnt + (uint32_t)L.cnts;
    uint64_t* wscr = reinterpret_cast<uint64_t*>(smem + L.xs + L.ys + L.mb + L.lists + L.cand + L.lvl + L.cnts + L.fb) +
                     warp * kFinalCap;
    const uint32_t rowb = 4u * (uint32_t)sx;
    const FastDiv fq((uint32_t)xs_chunks(nf));
    const int my_cols = warp < nf ? (nf - 1 - warp) / nwarps + 1 : 0;
    const int cl = tid % NFP, slot = tid / NFP;
    const bool col_thread = cl < nf && slot < P;

    for (int64_t li = blockIdx.x; li < n_list; li += gridDim.x) {
        const int row = rows[li];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        const bool full = (s >= n);
        const bool use_tab = !full && A.qtab != nullptr && n > 16;
        int jhi = 0, jlo = 0;
        if (use_tab) table_levels(n, s, A.delta_tab, jhi, jlo);
        const int chunk = SM.chunk(n);

        // 1-D bulk copies pay off for long rows (>= 256 B); short rows stay on cp.async
        if (xs_chunks(nf) >= 16) stage_slice_bulk(A, lo, 0, n, s_xs, ys, mbar, phase);
        else stage_slice(A, lo, 0, n, Xs, ys, fq);
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

        if (use_tab) {
            // ---- S2: per (column, slot) scan of the k-range ----
            if (col_thread) {
                const uint32_t* qc = A.qtab + (size_t)cl * (kQ + 1);
                const uint32_t hib = qc[jhi], lob = qc[jlo];
                const int span = jlo - jhi;
                const int k0 = slot * chunk, k1 = min(n, k0 + chunk);
                int above = 0, nin = 0;
                const uint32_t span_ab = hib > lob ? hib - lob : 0u;
                uint32_t addr = s_xs + (uint32_t)k0 * rowb + 4u * (uint32_t)cl;
                const uint32_t cbase = s_cand + 2u * (uint32_t)(slot * CAPS * NFP + cl);
                // 32 rows per step: two bit words (above the bracket / inside it)
                for (int kb = k0; kb < k1; kb += 32, addr += 32u * rowb) {
                    const int cnt = min(32, k1 - kb);
                    uint32_t wa = 0u, wi = 0u;
                    if (cnt == 32) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const uint32_t a = __float_as_uint(lds_f32(addr + (uint32_t)i * rowb)) & 0x7FFFFFFFu;
                            wa |= (a >= hib) ? (1u << i) : 0u;
                            wi |= (a - lob < span_ab) ? (1u << i) : 0u;
                        }
                    } else {
                        for (int i = 0; i < cnt; ++i) {
                            const uint32_t a = __float_as_uint(lds_f32(addr + (uint32_t)i * rowb)) & 0x7FFFFFFFu;
                            wa |= (a >= hib) ? (1u << i) : 0u;
                            wi |= (a - lob < span_ab) ? (1u << i) : 0u;
                        }
                    }
                    sts_u32(s_mb + 4u * (uint32_t)(cl * NW + (kb >> 5)), wa);
                    above += __popc(wa);
                    while (wi) {
                        const int i = __ffs(wi) - 1;
                        wi &= wi - 1;
                        if (nin < CAPS) sts_u16(cbase + 2u * (uint32_t)(nin * NFP), (uint32_t)(kb + i));
                        ++nin;
                    }
                }
                const uint32_t ci = s_cnt + 4u * (uint32_t)(slot * NFP + cl);
                sts_u16(ci, (uint32_t)above);
                sts_u16(ci + 2u, nin > CAPS ? 0xFFFFu : (uint32_t)nin);
                // counts of the listed keys against the table levels inside the bracket
                uint32_t lev[kSub - 1];
                int lc[kSub - 1];
#pragma unroll
                for (int t = 0; t < kSub - 1; ++t) {
                    lev[t] = qc[jhi + (span * (t + 1)) / kSub];
                    lc[t] = 0;
                }
                const int nl = min(nin, CAPS);
                const uint32_t xcol = s_xs + 4u * (uint32_t)cl;
                for (int i = 0; i < nl; ++i) {
                    const uint32_t k = lds_u16(cbase + 2u * (uint32_t)(i * NFP));
                    const uint32_t a = __float_as_uint(lds_f32(xcol + k * rowb)) & 0x7FFFFFFFu;
#pragma unroll
                    for (int t = 0; t < kSub - 1; ++t) lc[t] += (a >= lev[t]) ? 1 : 0;
                }
#pragma unroll
                for (int t = 0; t < kSub - 1; ++t)
                    sts_u8(s_lvl + (uint32_t)((slot * 8 + t) * NFP + cl), (uint32_t)min(lc[t], 255));
            }
            __syncthreads();
            // ---- S3: per column, the sub-bucket that holds the target rank ----
            if (tid < nf) {
                const int c = tid;
                int above = 0, nin = 0;
                bool over = false;
                int cge[kSub - 1];
#pragma unroll
                for (int t = 0; t < kSub - 1; ++t) cge[t] = 0;
                for (int q = 0; q < P; ++q) {
                    const uint32_t ci = s_cnt + 4u * (uint32_t)(q * NFP + c);
                    above += (int)lds_u16(ci);
                    const uint32_t ni = lds_u16(ci + 2u);
                    over |= (ni == 0xFFFFu);
                    nin += (int)(ni & 0xFFFFu);
#pragma unroll
                    for (int t = 0; t < kSub - 1; ++t) cge[t] += (int)lds_u8(s_lvl + (uint32_t)((q * 8 + t) * NFP + c));
                }
                const uint32_t* qc = A.qtab + (size_t)c * (kQ + 1);
                const uint32_t hib = qc[jhi], lob = qc[jlo];
                const uint64_t hik = hi_key_of(hib), lok = (uint64_t)lob << 32;
                const bool ok = !over && above < s && s <= above + nin && lok < hik;
                c_flag[c] = ok ? 0 : 1;
                if (A.stats != nullptr) {
                    if (over) stat_add(A, kStSmallOver, 1);
                    else if (!ok) stat_add(A, kStSmallMiss, 1);
                }
                c_fc[c] = 0;
                if (ok) {
                    const int need = s - above;
                    const int span = jlo - jhi;
                    int b = 0;
#pragma unroll
                    for (int t = 0; t < kSub - 1; ++t) b += (cge[t] < need) ? 1 : 0;
                    uint64_t bhi = hik, blo = lok;
                    int before = 0;
#pragma unroll
                    for (int t = 0; t < kSub - 1; ++t) {
                        const uint64_t lv = (uint64_t)qc[jhi + (span * (t + 1)) / kSub] << 32;
                        if (t == b - 1) { bhi = lv < hik ? lv : hik; before = cge[t]; }
                        if (t == b) blo = lv > lok ? lv : lok;
                    }
                    c_lo[c] = blo;
                    c_hi[c] = bhi;
                    c_need[c] = need - before;
                }
                if (lane == 0 && A.stats != nullptr) {
                    stat_add(A, kStColumns, 1);
                    stat_add(A, kStCandidates, (unsigned long long)nin);
                }
            }
            __syncthreads();
            // ---- S4: forward the chosen sub-bucket's keys ----
            if (col_thread && c_flag[cl] == 0) {
                const int nin = min((int)lds_u16(s_cnt + 4u * (uint32_t)(slot * NFP + cl) + 2u), CAPS);
                const uint32_t cbase = s_cand + 2u * (uint32_t)(slot * CAPS * NFP + cl);
                const uint64_t blo = c_lo[cl], bhi = c_hi[cl];
                const uint32_t xcol = s_xs + 4u * (uint32_t)cl;
                for (int i = 0; i < nin; ++i) {
                    const uint32_t k = lds_u16(cbase + 2u * (uint32_t)(i * NFP));
                    const uint64_t key = make_key(lds_f32(xcol + k * rowb), k);
                    if (key >= blo && key < bhi) {
                        const int p = atomicAdd(&c_fc[cl], 1);
                        if (p < kFinalCap) sts_u16(s_fb + 2u * (uint32_t)(cl * kFinalCap + p), k);
                    }
                }
            }
            __syncthreads();
        }

        // ---- S5: threshold key per column (warp per column) ----
        for (int j = 0; j < my_cols; ++j) {
            const int c = warp + j * nwarps;
            const uint32_t xcol = s_xs + 4u * (uint32_t)c;
            auto keyat = [xcol, rowb](int k) { return make_key(lds_f32(xcol + (uint32_t)k * rowb), (uint32_t)k); };
            uint64_t T = ~0ull;
            if (full) {
                if (A.thr_keys != nullptr) {  // complete sketch: report the smallest key
                    for (int k = lane; k < n; k += 32) {
                        const uint64_t kk = keyat(k);
                        T = kk < T ? kk : T;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const uint64_t t = __shfl_xor_sync(CALS_FULL_MASK, T, o);
                        T = t < T ? t : T;
                    }
                }
            } else {
                const int m = use_tab ? c_fc[c] : 0;
                const bool exact = !use_tab || c_flag[c] != 0 || m > kFinalCap;
                if (use_tab && c_flag[c] == 0 && m > kFinalCap && lane == 0) stat_add(A, kStFinalOver, 1);
                if (!exact) {
                    const int need = c_need[c];
                    if (m <= 32) {
                        const uint64_t v = lane < m ? keyat((int)lds_u16(s_fb + 2u * (uint32_t)(c * kFinalCap + (lane & 31)))) : 0ull;
                        T = warp_kth_desc(v, m, need, lane);
                    } else {
                        for (int i = lane; i < m; i += 32)
                            wscr[i] = keyat((int)lds_u16(s_fb + 2u * (uint32_t)(c * kFinalCap + i)));
                        __syncwarp();
                        T = warp_select_keys(KeyList{wscr}, m, need, c_lo[c], c_hi[c], lane);
                    }
                } else {
                    if (use_tab && lane == 0) stat_add(A, kStFallback, 1);
                    T = warp_select_column(keyat, n, n, s, 0ull, ~0ull, wscr, kFinalCap, lane);
                    // the whole column's bitmap words from T
                    for (int k0 = 0; k0 < n; k0 += 32) {
                        const int k = k0 + lane;
                        const uint32_t b = __ballot_sync(CALS_FULL_MASK, k < n && keyat(k) >= T);
                        if (lane == 0) sts_u32(s_mb + 4u * (uint32_t)(c * NW + (k0 >> 5)), b);
                    }
                    if (lane == 0) c_flag[c] = 1;
                }
            }
            if (lane == 0) thr[c] = T;
        }
        __syncthreads();

        // ---- S6: bracket keys at or above T join the kept set (own bitmap words) ----
        if (use_tab && col_thread && c_flag[cl] == 0) {
            const int nin = min((int)lds_u16(s_cnt + 4u * (uint32_t)(slot * NFP + cl) + 2u), CAPS);
            const uint32_t cbase = s_cand + 2u * (uint32_t)(slot * CAPS * NFP + cl);
            const uint32_t xcol = s_xs + 4u * (uint32_t)cl;
            const uint64_t T = thr[cl];
            for (int i = 0; i < nin; ++i) {
                const uint32_t k = lds_u16(cbase + 2u * (uint32_t)(i * NFP));
                if (make_key(lds_f32(xcol + k * rowb), k) >= T) {
                    const uint32_t wa = s_mb + 4u * (uint32_t)(cl * NW + (k >> 5));
                    sts_u32(wa, lds_u32(wa) | (1u << (k & 31)));
                }
            }
        }
        __syncthreads();

        // ---- S7: kept-row lists + sparse Gram of the owned columns -> global ----
        if (!full)
            for (int j = 0; j < my_cols; ++j) {
                const int c = warp + j * nwarps;
                bitmap_to_list(s_mb + 4u * (uint32_t)(c * NW), (n + 31) >> 5, s_lists + 2u * (uint32_t)(c * Smax),
                               lane);
            }
        const float lam_n = (float)(A.lam * (double)n);
        if (my_cols > 0)
            sparse_gram_owned<CPL>(s_xs, sx, s_ys, nf, full ? n : s, full, s_lists, Smax, warp, nwarps, my_cols, lam_n,
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

template __global__ void small_gram_kernel<1>(SweepArgs, const int32_t*, int64_t, int, int);
template __global__ void small_gram_kernel<2>(SweepArgs, const int32_t*, int64_t, int, int);
template __global__ void small_gram_kernel<4>(SweepArgs, const int32_t*, int64_t, int, int);
template __global__ void small_gram_kernel<8>(SweepArgs, const int32_t*, int64_t, int, int);

// ---------------------------------------------------------------------------
// Tiny regressions (n <= 64): one warp per row, no block barriers.  Per column
// the n keys are bitonic-sorted across the warp (one or two per lane) and the
// s-th is the threshold; kept rows come out of a ballot in ascending k.  The
// warp then runs the same sparse Gram over all columns and writes the normal
// equations for the batched solve.  kTinyN rows x sx floats per warp.
// ---------------------------------------------------------------------------
constexpr int kTinyN = 64;
constexpr int kTinyWarps = 4;

__host__ __device__ inline size_t tiny_warp_bytes(int nf) {
    return align16((size_t)kTinyN * xs_stride(nf) * 4) + align16(kTinyN * 4) + align16((size_t)nf * 4) +
           align16((size_t)nf * kTinyN * 2);
}

template <int CPL>
__global__ void __launch_bounds__(kTinyWarps * 32) tiny_gram_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                                    int64_t n_list) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int nf = A.nf, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sx = xs_stride(nf), gs = nf + 1;
    unsigned char* base = smem + (size_t)warp * tiny_warp_bytes(nf);
    float* Xs = reinterpret_cast<float*>(base);
    float* ys = reinterpret_cast<float*>(base + align16((size_t)kTinyN * sx * 4));
    float* wold = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(ys) + align16(kTinyN * 4));
    const uint32_t s_xs = smem_u32(Xs), s_ys = smem_u32(ys);
    const uint32_t s_lists = smem_u32(reinterpret_cast<unsigned char*>(wold) + align16((size_t)nf * 4));
    const uint32_t rowb = 4u * (uint32_t)sx;
    const int nq = xs_chunks(nf);
    const int64_t gw = (int64_t)blockIdx.x * kTinyWarps + warp;
    const int64_t stride = (int64_t)gridDim.x * kTinyWarps;
    for (int64_t li = gw; li < n_list; li += stride) {
        const int row = rows[li];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        const bool full = s >= n;
        __syncwarp();
        // stage (warp-level cp.async)
        for (int e = lane; e < n * nq; e += 32) {
            const int kk = e / nq, q = e - kk * nq;
            const int64_t r = __ldg(A.idx + lo + kk);
            cp_async16(s_xs + (uint32_t)kk * rowb + 16u * q, A.src + r * A.ld_src + 4 * q);
        }
        for (int kk = lane; kk < n; kk += 32) ys[kk] = __ldg(A.val + lo + kk);
        if (A.tgt_old != nullptr)
            for (int c = lane; c < nf; c += 32) wold[c] = A.tgt_old[(int64_t)row * A.ld_old + c];
        cp_async_wait_all();
        __syncwarp();
        // fused residual of the previous iteration's row
        if (A.rss_rows != nullptr) {
            double acc = 0.0;
            for (int kk = lane; kk < n; kk += 32) {
                float pred = 0.f;
                for (int f = 0; f < nf; ++f) pred = fmaf(lds_f32(s_xs + (uint32_t)kk * rowb + 4u * f), wold[f], pred);
                const double d = (double)ys[kk] - (double)pred;
                acc = fma(d, d, acc);
            }
            acc = warp_sum_d(acc);
            if (lane == 0) A.rss_rows[row] = acc;
        }
        // per column: threshold key by a warp sort, kept rows by ballot
        for (int c = 0; c < nf; ++c) {
            const uint32_t xcol = s_xs + 4u * (uint32_t)c;
            auto keyat = [xcol, rowb](int kk) { return make_key(lds_f32(xcol + (uint32_t)kk * rowb), (uint32_t)kk); };
            const uint64_t k0 = lane < n ? keyat(lane) : 0ull;
            const uint64_t k1 = lane + 32 < n ? keyat(lane + 32) : 0ull;
            uint64_t T;
            if (full) {
                uint64_t mn = lane < n ? k0 : ~0ull;
                if (lane + 32 < n) mn = k1 < mn ? k1 : mn;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t t2 = __shfl_xor_sync(CALS_FULL_MASK, mn, o);
                    mn = t2 < mn ? t2 : mn;
                }
                T = mn;
            } else if (s <= 8) {
                // small budgets: extract the s largest keys one warp max at a time
                uint64_t v0 = lane < n ? k0 : 0ull, v1 = lane + 32 < n ? k1 : 0ull;
                for (int q = 0; q < s; ++q) {
                    uint64_t m = v0 > v1 ? v0 : v1;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const uint64_t t2 = __shfl_xor_sync(CALS_FULL_MASK, m, o);
                        m = t2 > m ? t2 : m;
                    }
                    T = m;  // keys are unique: exactly one lane holds m
                    if (v0 == m) v0 = 0ull;
                    if (v1 == m) v1 = 0ull;
                }
            } else if (n <= 32) {
                const uint64_t v = warp_sort_desc(k0, lane);
                T = __shfl_sync(CALS_FULL_MASK, v, s - 1);
            } else {
                uint64_t v0 = k0, v1 = k1;
                warp_sort64_desc(v0, v1, lane);
                T = s - 1 < 32 ? __shfl_sync(CALS_FULL_MASK, v0, s - 1) : __shfl_sync(CALS_FULL_MASK, v1, s - 1 - 32);
            }
            if (A.thr_keys != nullptr && lane == 0) A.thr_keys[(int64_t)row * nf + c] = T;
            if (!full) {
                const uint32_t L = s_lists + 2u * (uint32_t)(c * kTinyN);
                const bool a0 = lane < n && k0 >= T, a1 = lane + 32 < n && k1 >= T;
                const uint32_t b0 = __ballot_sync(CALS_FULL_MASK, a0), b1 = __ballot_sync(CALS_FULL_MASK, a1);
                if (a0) sts_u16(L + 2u * (uint32_t)__popc(b0 & lanemask_lt()), (uint32_t)lane);
                if (a1) sts_u16(L + 2u * (uint32_t)(__popc(b0) + __popc(b1 & lanemask_lt())), (uint32_t)(lane + 32));
            }
        }
        __syncwarp();
        const float lam_n = (float)(A.lam * (double)n);
        sparse_gram_owned<CPL>(s_xs, sx, s_ys, nf, full ? n : s, full, s_lists, kTinyN, 0, 1, nf, lam_n,
                               A.gbuf + (size_t)li * nf * gs, lane);
    }
}

template __global__ void tiny_gram_kernel<1>(SweepArgs, const int32_t*, int64_t);
template __global__ void tiny_gram_kernel<2>(SweepArgs, const int32_t*, int64_t);
template __global__ void tiny_gram_kernel<4>(SweepArgs, const int32_t*, int64_t);
template __global__ void tiny_gram_kernel<8>(SweepArgs, const int32_t*, int64_t);

}  // namespace cals
