// sweep_big.cu -- the tiled tier of the half-sweep: regressions whose slice
// does not fit in shared memory (the reference's long rows, which it handles
// with the presort walk, core.py:167-170,209-213).
//
// A big row is cut into work items of `item_rows` slice rows, processed in
// shared-memory chunks.  Per half-sweep:
//   big_scan2    counts per column above / inside the table bracket, a
//                32-bucket histogram of the bracket, and appends the
//                bracket's keys to a per-(row, column) list (one share per item)
//   big_resolve  one warp per (row, column): the histogram names the bucket
//                holding the target rank, one filtering pass keeps its keys,
//                a warp select finishes (or an exact whole-column search if
//                the bracket missed: always correct)
//   big_gram     sparse partial Gram per item from per-chunk kept-row lists
//                (fixed order), plus the item's share of the fused residual
//   big_reduce   fixed-order fp64 sum of the partials, + lam*n*I -> normal
//                equations for the batched solve (sweep_solve.cu)
#include "gram.cuh"
#include "select.cuh"
#include "solve.cuh"
#include "sweep_common.cuh"

namespace cals {


__device__ __forceinline__ int find_row(const int64_t* tile_ptr, int64_t n_big, int64_t t) {
    int64_t lo = 0, hi = n_big - 1;  // largest r with tile_ptr[r] <= t
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (tile_ptr[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return (int)lo;
}

// Row-local bracket calibration for long rows: the table describes the
// rating-weighted population of source values, and a long row's own values
// can sit systematically above or below it (a popular item is rated by
// nearly every user, not by an activity-weighted draw).  A deterministic
// strided sample of kCalibSamples slice rows is counted against the table
// levels of each column; the bracket levels are the sample's rank estimates
// of the target fraction s/n, +- kCalibZ sampling sigmas.  A miss is still
// caught (and resolved exactly) by big_resolve.
constexpr int kCalibSamples = 4096;
constexpr float kCalibZ = 5.5f;
constexpr int kCalibCols = 32;  // columns per shared-memory pass

__global__ void __launch_bounds__(kThreads) big_calib_kernel(SweepArgs A, BigArgs B, int64_t n_rows) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* qs = reinterpret_cast<uint32_t*>(smem);  // [kCalibCols][kQ + 1]
    uint32_t* hist = qs + kCalibCols * (kQ + 1);         // [kCalibCols][kQ + 1]
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        if (s >= n) continue;
        const int m = min(B.calib_samples > 0 ? B.calib_samples : kCalibSamples, max(1024, n / 4));  // n > 4096 here
        const double p = (double)s / (double)n;
        const double sig = sqrt(p * (1.0 - p) / (double)m * (double)(n - m) / (double)max(n - 1, 1));
        const double z = B.calib_z > 0.f ? B.calib_z : kCalibZ;
        const int t_lo = (int)floor((p - z * sig) * (double)m);
        const int t_hi = (int)ceil((p + z * sig) * (double)m);
        for (int c0 = 0; c0 < nf; c0 += kCalibCols) {
            const int gc = min(kCalibCols, nf - c0);
            __syncthreads();
            for (int e = tid; e < gc * (kQ + 1); e += nt) {
                qs[e] = A.qtab[(size_t)c0 * (kQ + 1) + e];
                hist[e] = 0;
            }
            __syncthreads();
            for (int j = tid; j < m; j += nt) {
                const int k = (int)(((2 * (int64_t)j + 1) * n) / (2 * (int64_t)m));
                const float* xr = A.src + (int64_t)__ldg(A.idx + lo + k) * A.ld_src + c0;
#pragma unroll 4
                for (int g = 0; g < gc; ++g) {
                    const uint32_t v = abs_bits(__ldg(xr + g));
                    const uint32_t q = smem_u32(qs + g * (kQ + 1));
                    // branchless search for the last level with q[pos] > v (q[0] = inf, q[kQ] = 0)
                    int pos = 0;
#pragma unroll
                    for (int step = kQ / 2; step > 0; step >>= 1)
                        pos += (lds_u32(q + 4u * (uint32_t)(pos + step)) > v) ? step : 0;
                    atomicAdd(&hist[g * (kQ + 1) + pos + 1], 1u);
                }
            }
            __syncthreads();
            for (int g = warp; g < gc; g += nt >> 5) {
                // cnt(j) = sample values >= q[j] = sum_{L <= j} hist[L] (nondecreasing in j)
                int run = 0, n_le = 0, n_lt = 0;
                for (int j0 = 0; j0 <= kQ; j0 += 32) {
                    const int j = j0 + lane;
                    int v = j <= kQ ? (int)hist[g * (kQ + 1) + j] : 0;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t2 = __shfl_up_sync(CALS_FULL_MASK, v, o);
                        if (lane >= o) v += t2;
                    }
                    const int cnt = run + v;
                    n_le += __popc(__ballot_sync(CALS_FULL_MASK, j <= kQ && cnt <= t_lo));
                    n_lt += __popc(__ballot_sync(CALS_FULL_MASK, j <= kQ && cnt < t_hi));
                    run += __shfl_sync(CALS_FULL_MASK, v, 31);
                }
                if (lane == 0) {
                    const int jhi = t_lo < 0 ? 0 : n_le - 1;
                    const int jlo = t_hi > m ? kQ : min(n_lt, kQ);
                    ((uint32_t*)B.brk)[(size_t)r * nf + c0 + g] = (uint32_t)jhi | ((uint32_t)jlo << 16);
                }
            }
        }
    }
}

// Threshold of one column whose bracket held the target rank (above < s <= above + in, the
// in-bracket keys complete in one contiguous list cl[0, in)): the sub-bucket of the target rank
// from the histogram (cnt_b: the calling lane's bucket, lane 0 = highest), that bucket's keys
// kept in the warp's shared-memory list while they number <= 32, else compacted in place in
// cl, and the need-th largest of them.  Used by big_scan2_kernel for single-item rows, right
// after their only item: the keys are still in L2 and the counts in shared memory
// (big_resolve_kernel keeps the per-item-share form for multi-item rows).
__device__ __forceinline__ uint64_t resolve_one_list(uint64_t* __restrict__ cl, int in, int need, int cnt_b, uint32_t hib,
                                                     uint32_t lob, uint64_t* __restrict__ keep_w, int lane) {
    const uint64_t hik = hi_key_of(hib);
    int incl = cnt_b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t2 = __shfl_up_sync(CALS_FULL_MASK, incl, o);
        if (lane >= o) incl += t2;
    }
    const uint32_t hit = __ballot_sync(CALS_FULL_MASK, incl >= need);
    const int L = __ffs(hit) - 1;  // first lane whose prefix reaches need
    const int before = __shfl_sync(CALS_FULL_MASK, incl - cnt_b, L);
    const int bT = kHB - 1 - L;
    const int sh = hb_shift(hib - lob);
    const uint64_t blo = hb_lower_key(bT, lob, sh);
    const uint64_t bhi = min(hb_lower_key(bT + 1, lob, sh), hik);
    int m = 0;
    bool spill = false;
    for (int i0 = 0; i0 < in; i0 += 128) {
        uint64_t kk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + 32 * u + lane;
            kk[u] = i < in ? cl[i] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + 32 * u + lane;
            const bool keep = i < in && kk[u] >= blo && kk[u] < bhi;
            const uint32_t bal = __ballot_sync(CALS_FULL_MASK, keep);
            const int cnt = __popc(bal);
            if (!spill && m + cnt <= 32) {
                if (keep) keep_w[m + __popc(bal & lanemask_lt())] = kk[u];
            } else {
                if (!spill) {
                    __syncwarp();
                    if (lane < m) cl[lane] = keep_w[lane];
                    spill = true;
                }
                __syncwarp();
                if (keep) cl[m + __popc(bal & lanemask_lt())] = kk[u];
            }
            m += cnt;
        }
    }
    __syncwarp();
    uint64_t T;
    if (spill) {
        T = warp_select_keys(KeyList{cl}, m, need - before, blo, bhi, lane);
    } else {
        // rank of the lane's key among the m kept keys (broadcast reads of the list)
        const uint64_t v = lane < m ? keep_w[lane] : 0ull;
        int gt = 0;
        for (int jj = 0; jj < m; ++jj) gt += (keep_w[jj] > v) ? 1 : 0;
        const uint32_t hit2 = __ballot_sync(CALS_FULL_MASK, lane < m && gt == need - before - 1);
        T = __shfl_sync(CALS_FULL_MASK, v, __ffs(hit2) - 1);
        __syncwarp();  // keep_w is free for the warp's next column
    }
    return T;
}

// Tiled tier pass 1, pipelined: persistent CTAs claim work items from a counter
// (B.item_ctr, zeroed before the launch; longest rows first), each item's slice is
// streamed in chunks of B.chunk rows through two shared-memory buffers (the bulk
// copies of chunk i+1 are in flight while chunk i is counted; slice-row ids are loaded
// a chunk earlier still), and the count pass is compiled for the headline shape (PER
// threads per column, row stride SXT floats, KCT-row chunks) without bounds checks on
// full chunks.  An item writes its in-bracket keys into its own equal share of the
// row's column region (cand_item_cap), reserving positions with shared-memory
// counters: no global atomics per chunk and one block barrier per chunk.  Per (row,
// column) outputs: count above the bracket, the in-bracket
// histogram and total, and per item its in-bracket count (B.icnt; a share that
// overflowed sends that column to big_resolve's exact search).
template <int PER, int SXT, int KCT>
__global__ void __launch_bounds__(kThreads, 4) big_scan2_kernel(SweepArgs A, BigArgs B) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_above[CALS_MAX_NF_DEV], s_pos[CALS_MAX_NF_DEV];
    __shared__ uint32_t s_hib[CALS_MAX_NF_DEV], s_lob[CALS_MAX_NF_DEV];
    __shared__ __align__(8) unsigned long long s_mbar[2];
    __shared__ int s_item;
    __shared__ uint64_t s_keep[kThreads / 32][32];  // fused resolve of single-item rows (resolve_one_list)
    __shared__ unsigned char s_done[CALS_MAX_NF_DEV];
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x;
    const int sx = SXT > 0 ? SXT : xs_stride(nf);
    const int per = PER > 0 ? PER : nt / nf;  // threads per column
    const int KC = KCT > 0 ? KCT : B.chunk;   // staged slice rows per buffer (<= blockDim.x)
    const uint32_t rowb = 4u * (uint32_t)sx;
    const uint32_t bufb = (uint32_t)align16((size_t)KC * sx * 4);
    const uint32_t s_xs = smem_u32(smem);
    int* s_hist = reinterpret_cast<int*>(smem + 2 * (size_t)bufb);  // [nf][kHB]
    const uint32_t rowbytes = 16u * (uint32_t)xs_chunks(nf);
    if (tid == 0) {
        mbar_init(smem_u32(&s_mbar[0]), 1);
        mbar_init(smem_u32(&s_mbar[1]), 1);
    }
    __syncthreads();
    uint32_t phases = 0u;  // bit b: parity of buffer b's barrier
    const int c = tid % nf, j = tid / nf;
    const bool col_thread = tid < per * nf;
    // chunk rows into buffer b: every thread copies its row (id in `rid`)
    auto stage = [&](int b, int kn, int rid) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // prior generic reads of the buffer
        if (tid == 0) mbar_expect_tx(smem_u32(&s_mbar[b]), (uint32_t)kn * rowbytes);
        if (tid < kn) bulk_g2s(s_xs + (uint32_t)b * bufb + (uint32_t)tid * rowb, A.src + (int64_t)rid * A.ld_src,
                               rowbytes, smem_u32(&s_mbar[b]));
    };
    for (;;) {
        __syncthreads();  // previous item done with s_item, buffers, counters, histogram
        if (tid == 0) s_item = atomicAdd(B.item_ctr, 1);
        __syncthreads();
        const int64_t t = s_item;
        if (t >= B.n_tiles) break;
        const int64_t T_abs = B.tile_base + t;
        const int r = B.tile_row != nullptr ? (int)(__ldg(B.tile_row + T_abs) - B.row_base)
                                            : find_row(B.tile_ptr, B.n_big, T_abs);
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        if (s >= n) continue;  // complete sketch: nothing to select (uniform per block)
        const int t_loc = (int)(T_abs - B.tile_ptr[r]);
        const int kbeg = t_loc * B.item_rows;
        const int kend = min(n, kbeg + B.item_rows);
        const int32_t* idx = A.idx + lo;
        const int kn0 = min(KC, kend - kbeg);
        const int rid0 = tid < kn0 ? __ldg(idx + kbeg + tid) : 0;
        if (tid < nf) {
            uint32_t hib, lob;
            big_bracket(A, B, r, tid, n, s, hib, lob);
            s_hib[tid] = hib;
            s_lob[tid] = lob;
            s_above[tid] = 0;
            s_pos[tid] = 0;
        }
        for (int e = tid; e < nf * kHB; e += nt) s_hist[e] = 0;
        const int capB = (int)((B.cand_ptr[r + 1] - B.cand_ptr[r]) / nf);
        const int capI = cand_item_cap(capB, (int)(B.tile_ptr[r + 1] - B.tile_ptr[r]));
        uint64_t* cl = B.cand + (B.cand_ptr[r] - B.cand_base) + (int64_t)c * capB + (int64_t)t_loc * capI;
        stage(0, kn0, rid0);
        const int kn1_0 = kbeg + KC < kend ? min(KC, kend - kbeg - KC) : 0;
        int rid_next = tid < kn1_0 ? __ldg(idx + kbeg + KC + tid) : 0;  // chunk 1's row
        int my_above = 0;
        int ci = 0;
        for (int k0 = kbeg; k0 < kend; k0 += KC, ++ci) {
            const int b = ci & 1;
            const int kn = min(KC, kend - k0);
            const int k1 = k0 + KC, kn1 = k1 < kend ? min(KC, kend - k1) : 0;
            const int k2 = k1 + KC, kn2 = k2 < kend ? min(KC, kend - k2) : 0;
            const int rid2 = tid < kn2 ? __ldg(idx + k2 + tid) : 0;  // two chunks ahead
            mbar_wait(smem_u32(&s_mbar[b]), (phases >> b) & 1u);
            phases ^= 1u << b;
            __syncthreads();  // chunk ci landed for every thread; buffer b^1 free (chunk ci-1 emitted)
            if (kn1 > 0) stage(b ^ 1, kn1, rid_next);
            rid_next = rid2;
            const uint32_t xb = s_xs + (uint32_t)b * bufb;
            uint32_t inmask = 0;  // bit i: row j + i * per is inside the bracket
            if (col_thread) {
                const uint32_t hib = s_hib[c], lob = s_lob[c], span = hib - lob;
                const uint32_t colb = xb + 4u * (uint32_t)c + (uint32_t)j * rowb;
                if (KCT > 0 && kn == KCT) {
                    // full chunk, compile-time row stride: immediate-offset loads, no bounds checks
#pragma unroll
                    for (int i = 0; i < KCT / PER; ++i) {
                        const uint32_t a = abs_bits(lds_f32(colb + (uint32_t)(i * PER * SXT * 4)));
                        my_above += a >= hib ? 1 : 0;
                        inmask |= (a - lob < span) ? (1u << i) : 0u;
                    }
                } else {
                    const int rows_t = (KC + per - 1) / per;
                    const uint32_t stepb = (uint32_t)per * rowb;
#pragma unroll 8
                    for (int i = 0; i < rows_t; ++i) {
                        const int k = j + i * per;
                        const uint32_t a = k < kn ? abs_bits(lds_f32(colb + (uint32_t)i * stepb)) : 0u;
                        my_above += (k < kn && a >= hib) ? 1 : 0;
                        inmask |= (k < kn && a - lob < span) ? (1u << i) : 0u;
                    }
                }
                const int my_in = __popc(inmask);
                if (my_in) {
                    // a contiguous run in the item's share of the column region
                    int pos = atomicAdd(&s_pos[c], my_in);
                    const uint32_t lob2 = lob;
                    const int sh = hb_shift(span);
                    while (inmask) {
                        const int i = __ffs(inmask) - 1;
                        inmask &= inmask - 1;
                        const int k = j + i * per;
                        const float x = lds_f32(xb + (uint32_t)k * rowb + 4u * c);
                        atomicAdd(&s_hist[c * kHB + (int)((abs_bits(x) - lob2) >> sh)], 1);
                        if (pos < capI) cl[pos] = make_key(x, (uint32_t)(k0 + k));
                        ++pos;
                    }
                }
            }
        }
        if (col_thread && my_above) atomicAdd(&s_above[c], my_above);
        __syncthreads();
        // A single-item row is resolved right here: its counts and histogram are in shared memory and
        // its in-bracket keys (written by this CTA a moment ago) in L2, so the columns whose bracket held
        // the target rank get their threshold without the round trip through big_resolve_kernel (which
        // skips them: in-count -1) -- no dependent header loads, no second pass over the keys from HBM.
        const bool single = B.tile_ptr[r + 1] - B.tile_ptr[r] == 1;
        if (single) {
            const int warp = tid >> 5, lane = tid & 31;
            uint64_t* cl0 = B.cand + (B.cand_ptr[r] - B.cand_base);
            for (int c2 = warp; c2 < nf; c2 += nt >> 5) {
                const int above = s_above[c2], in = s_pos[c2];
                const uint32_t hib = s_hib[c2], lob = s_lob[c2];
                const bool ok = above < s && s <= above + in && in <= capB && ((uint64_t)lob << 32) < hi_key_of(hib);
                if (ok) {
                    const uint64_t T = resolve_one_list(cl0 + (int64_t)c2 * capB, in, s - above,
                                                        s_hist[c2 * kHB + (kHB - 1 - lane)], hib, lob, s_keep[warp], lane);
                    if (lane == 0) {
                        stat_add(A, kStBigColumns, 1);
                        B.thr[(size_t)r * nf + c2] = T;
                        if (A.thr_keys != nullptr) A.thr_keys[(int64_t)row * nf + c2] = T;
                    }
                }
                if (lane == 0) s_done[c2] = ok ? 1 : 0;
            }
            __syncthreads();
        }
        if (tid < nf) {
            if (single && s_done[tid]) {
                B.cnt[((size_t)r * nf + tid) * 2 + 1] = -1;  // resolved: big_resolve_kernel skips the column
            } else {
                if (s_above[tid]) atomicAdd(&B.cnt[((size_t)r * nf + tid) * 2], s_above[tid]);
                if (s_pos[tid]) atomicAdd(&B.cnt[((size_t)r * nf + tid) * 2 + 1], s_pos[tid]);
            }
            B.icnt[(size_t)t * nf + tid] = s_pos[tid];
        }
        for (int e = tid; e < nf * kHB; e += nt)
            if (s_hist[e] && !(single && s_done[e / kHB])) atomicAdd(&B.hist[(size_t)r * nf * kHB + e], s_hist[e]);
    }
}
template __global__ void big_scan2_kernel<4, 68, 64>(SweepArgs, BigArgs);
template __global__ void big_scan2_kernel<0, 0, 0>(SweepArgs, BigArgs);

__global__ void __launch_bounds__(kThreads) big_resolve_kernel(SweepArgs A, BigArgs B) {
    // per warp: the target bucket's keys while they number <= 32 (each keeping lane stores its key
    // at its rank; lane p then picks up key p -- a find-nth-set-bit + shuffle per lane and round
    // cost 29 % of this kernel's instructions)
    __shared__ uint64_t s_keep[kThreads / 32][32];
    const int nf = A.nf;
    const int lane = threadIdx.x & 31;
    uint64_t* keep_w = s_keep[threadIdx.x >> 5];
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwork = B.n_big * nf;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = gw; w < nwork; w += wstride) {
        const int r = (int)(w / nf), c = (int)(w % nf);
        if (B.cnt[((size_t)r * nf + c) * 2 + 1] < 0) continue;  // resolved by big_scan2_kernel (single-item row)
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        const float* src = A.src;
        const int32_t* idx = A.idx + lo;
        const int ld = A.ld_src;
        auto keyat = [src, idx, ld, c](int k) {
            return make_key(__ldg(src + (int64_t)__ldg(idx + k) * ld + c), (uint32_t)k);
        };
        uint64_t T;
        if (s >= n) {
            uint64_t mn = ~0ull;
            if (A.thr_keys != nullptr) {
                for (int k = lane; k < n; k += 32) {
                    const uint64_t kk = keyat(k);
                    mn = kk < mn ? kk : mn;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t t2 = __shfl_xor_sync(CALS_FULL_MASK, mn, o);
                    mn = t2 < mn ? t2 : mn;
                }
            }
            T = (A.thr_keys != nullptr) ? mn : 0ull;
        } else {
            const int above = B.cnt[((size_t)r * nf + c) * 2];
            const int in = B.cnt[((size_t)r * nf + c) * 2 + 1];
            const int64_t cbase = B.cand_ptr[r] - B.cand_base;
            const int capB = (int)((B.cand_ptr[r + 1] - B.cand_ptr[r]) / nf);
            uint64_t* cl = B.cand + cbase + (int64_t)c * capB;
            uint32_t hib, lob;
            big_bracket(A, B, r, c, n, s, hib, lob);
            const uint64_t hik = hi_key_of(hib), lok = (uint64_t)lob << 32;
            // the column's keys: one contiguous list, or (scan2, multi-item rows) one share per item
            const int n_items = (int)(B.tile_ptr[r + 1] - B.tile_ptr[r]);
            const int capI = B.icnt != nullptr ? cand_item_cap(capB, n_items) : capB;
            const int64_t t0 = B.tile_ptr[r] - B.tile_base;  // batch-relative first item of the row
            const int nseg = B.icnt != nullptr ? n_items : 1;
            bool seg_over = false;
            if (B.icnt != nullptr)
                for (int q = 0; q < nseg; ++q) seg_over |= B.icnt[(size_t)(t0 + q) * nf + c] > capI;
            if (above < s && s <= above + in && in <= capB && !seg_over && lok < hik) {
                // bucket holding the target rank: inclusive scan of the histogram from the top
                const int need = s - above;
                const int bl = kHB - 1 - lane;  // lane 0 = highest bucket
                const int cnt_b = B.hist[((size_t)r * nf + c) * kHB + bl];
                int incl = cnt_b;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t2 = __shfl_up_sync(CALS_FULL_MASK, incl, o);
                    if (lane >= o) incl += t2;
                }
                const uint32_t hit = __ballot_sync(CALS_FULL_MASK, incl >= need);
                const int L = __ffs(hit) - 1;  // first lane whose prefix reaches need
                const int before = __shfl_sync(CALS_FULL_MASK, incl - cnt_b, L);
                const int bT = kHB - 1 - L;
                const int sh = hb_shift(hib - lob);
                const uint64_t blo = hb_lower_key(bT, lob, sh);
                const uint64_t bhi = min(hb_lower_key(bT + 1, lob, sh), hik);
                // keep that bucket's keys, then select among them: in registers (one key
                // per lane) while they fit, else compacted in place in the candidate list.
                // Four 32-key loads are in flight per round (the list streams from HBM).
                int m = 0;
                bool spill = false;
                uint64_t v = 0ull;
                for (int q = 0; q < nseg; ++q) {
                const int cnt_q = B.icnt != nullptr ? B.icnt[(size_t)(t0 + q) * nf + c] : in;
                const uint64_t* sl = cl + (int64_t)q * capI;
                for (int i0 = 0; i0 < cnt_q; i0 += 128) {
                    uint64_t kk[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = i0 + 32 * u + lane;
                        kk[u] = i < cnt_q ? sl[i] : 0ull;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = i0 + 32 * u + lane;
                        const bool keep = i < cnt_q && kk[u] >= blo && kk[u] < bhi;
                        const uint32_t bal = __ballot_sync(CALS_FULL_MASK, keep);
                        const int cnt = __popc(bal);
                        if (!spill && m + cnt <= 32) {
                            if (keep) keep_w[m + __popc(bal & lanemask_lt())] = kk[u];
                        } else {
                            if (!spill) {
                                __syncwarp();
                                if (lane < m) cl[lane] = keep_w[lane];
                                spill = true;
                            }
                            __syncwarp();
                            if (keep) cl[m + __popc(bal & lanemask_lt())] = kk[u];
                        }
                        m += cnt;
                    }
                }
                }
                __syncwarp();
                if (lane == 0) stat_add(A, kStBigColumns, 1);
                if (spill) {
                    T = warp_select_keys(KeyList{cl}, m, need - before, blo, bhi, lane);
                } else {
                    // rank of the lane's key among the m kept keys (broadcast reads of the list)
                    v = lane < m ? keep_w[lane] : 0ull;
                    int gt = 0;
                    for (int j = 0; j < m; ++j) gt += (keep_w[j] > v) ? 1 : 0;
                    const uint32_t hit = __ballot_sync(CALS_FULL_MASK, lane < m && gt == need - before - 1);
                    T = __shfl_sync(CALS_FULL_MASK, v, __ffs(hit) - 1);
                    __syncwarp();  // keep_w is free for the warp's next column
                }
            } else {
                if (lane == 0) {
                    stat_add(A, kStBigFallback, 1);
                    stat_add(A, above >= s ? kStBigMissAbove : (above + in < s ? kStBigMissBelow : kStBigOverflow), 1);
                    stat_add(A, kStBigFallbackN, (unsigned long long)n);
                }
                uint64_t rlo, rhi;
                int m, need;
                if (above >= s) { rlo = hik; rhi = ~0ull; m = above; need = s; }
                else if (above + in < s) { rlo = 0ull; rhi = lok; m = n - above - in; need = s - above - in; }
                else { rlo = lok; rhi = hik; m = in; need = s - above; }
                T = warp_select_column(keyat, n, m, need, rlo, rhi, cl, capB, lane);
            }
        }
        if (lane == 0) {
            B.thr[(size_t)r * nf + c] = T;
            if (A.thr_keys != nullptr) A.thr_keys[(int64_t)row * nf + c] = T;
        }
    }
}

// Partial normal equations of one work item: per staged chunk, warp w builds
// the kept-row lists of its columns (ballots on key >= T) and accumulates
// their sparse Gram rows -- in registers across the item's chunks when the
// warp's columns fit one lane-group round (nf <= 64), else in shared memory;
// the item's partial goes to global.
// n_f > 64 (CPL 8) runs 512-thread CTAs: 16 warps own <= 8 columns each, so the
// accumulators stay register-resident (owned_single_round) instead of in shared memory.
constexpr int big_gram_threads(int cpl) { return cpl >= 8 ? 512 : kThreads; }
// staged chunks summed in fp32 before a fold into the float64 accumulators (~50 kept terms at rate 0.1)
constexpr int kFoldChunks = 4;

template <int CPL, bool FAST, bool F64 = false>
__global__ void __launch_bounds__(big_gram_threads(CPL), CPL <= 4 ? (F64 ? 2 : 3) : 1) big_gram_kernel(SweepArgs A, BigArgs B) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t s_thr[CALS_MAX_NF_DEV];
    __shared__ unsigned long long s_amax[FAST ? CALS_MAX_NF_DEV : 1];
    __shared__ int s_cnt[FAST ? CALS_MAX_NF_DEV : 1];
    __shared__ __align__(8) unsigned long long s_mbar;
    const uint32_t mbar = smem_u32(&s_mbar);
    uint32_t phase = 0;
    if (threadIdx.x == 0) mbar_init(mbar, 1);
    __syncthreads();
    __shared__ float wold[CALS_MAX_NF_DEV];
    __shared__ double red[32];
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const int sx = xs_stride(nf), gs = nf + 1;
    const int CH = B.chunk, nw = CH / 32;
    const bool persist = owned_single_round(nf, nwarps);
    float* Xs = reinterpret_cast<float*>(smem);
    float* ys = reinterpret_cast<float*>(smem + align16((size_t)CH * sx * 4));
    unsigned char* after_ys = reinterpret_cast<unsigned char*>(ys) + align16((size_t)CH * 4);
    float* G = reinterpret_cast<float*>(after_ys);  // shared-memory accumulation (!persist only)
    unsigned char* after_g = after_ys + (persist ? 0 : align16((size_t)nf * gs * 4));
    const uint32_t s_xs = smem_u32(Xs), s_ys = smem_u32(ys);
    const uint32_t s_bits = smem_u32(after_g);                       // [nf][nw] kept-row bitmap words
    const uint32_t s_lists = s_bits + 4u * (uint32_t)(nf * nw);      // [nf][CH] u16 (!persist only)
    const uint32_t s_lens = s_lists + 2u * (uint32_t)(nf * CH);      // [nf] u32 (!persist only)
    // FAST: staged global-sketch mask words of the chunk's rows, [CH][gwords]
    const uint32_t s_gm = persist ? s_bits + 4u * (uint32_t)(nf * nw) : s_lens + 4u * (uint32_t)nf;
    // float64 accumulators of the work item's Gram (persist path only), after the FAST mask words
    double* G64 = reinterpret_cast<double*>(after_g + align16((size_t)nf * nw * 4 +
                                                              (FAST ? (size_t)CH * B.gwords * 4 : 0)));
    const uint32_t rowb = 4u * (uint32_t)sx;
    const FastDiv fq((uint32_t)xs_chunks(nf));
    const int my_cols = warp < nf ? (nf - 1 - warp) / nwarps + 1 : 0;
    const OwnedMap M(nf, warp, nwarps, my_cols, lane);
    OwnedAcc<CPL, typename std::conditional<F64, double, float>::type> S;
    for (int64_t t = blockIdx.x; t < B.n_tiles; t += gridDim.x) {
        const int64_t T_abs = B.tile_base + t;
        const int r = B.tile_row != nullptr ? (int)(__ldg(B.tile_row + T_abs) - B.row_base)
                                            : find_row(B.tile_ptr, B.n_big, T_abs);
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const bool full = A.budget[row] >= n;
        const int kbeg = (int)(T_abs - B.tile_ptr[r]) * B.item_rows;
        const int kend = min(n, kbeg + B.item_rows);
        __syncthreads();
        if (tid < nf) {
            if (!FAST) s_thr[tid] = B.thr[(size_t)r * nf + tid];
            if (A.tgt_old != nullptr) wold[tid] = A.tgt_old[(int64_t)row * A.ld_old + tid];
            if (FAST) {
                s_cnt[tid] = 0;
                s_amax[tid] = 0ull;
            }
        }
        S.zero();
        if (persist)
            for (int e = tid; e < nf * gs; e += nt) G64[e] = 0.0;  // the tile-start barrier above orders the reuse
        double racc = 0.0;
        for (int k0 = kbeg; k0 < kend; k0 += CH) {
            const int kn = min(CH, kend - k0);
            __syncthreads();
            stage_slice_bulk(A, lo, k0, kn, s_xs, ys, mbar, phase);
            if (FAST && !full) {
                for (int e = tid; e < kn * B.gwords; e += nt) {
                    const int k = e / B.gwords, wi = e - k * B.gwords;
                    sts_u32(s_gm + 4u * (uint32_t)e,
                            __ldg(B.gmask + (int64_t)__ldg(A.idx + lo + k0 + k) * B.gwords + wi));
                }
            }
            __syncthreads();
            if (A.rss_rows != nullptr) {
                for (int k = tid; k < kn; k += nt) {
                    double pred = 0.0;
                    for (int f = 0; f < nf; ++f)
                        pred = fma((double)lds_f32(s_xs + (uint32_t)k * rowb + 4u * f), (double)wold[f], pred);
                    const double d = (double)lds_f32(s_ys + 4u * k) - pred;
                    racc = fma(d, d, racc);
                }
            }
            if (!full) {
                // kept-row bitmap words: thread (c, wd) builds word wd of column c from 32
                // sequential rows (a warp reads 32 adjacent columns of one row: no bank
                // conflicts); keep <=> key >= T <=> abs > Ta, or abs == Ta and row <= Tk
                const int nwk = (kn + 31) >> 5;
                for (int e = tid; e < nf * nwk; e += nt) {
                    const int wd = e / nf, c = e - wd * nf;
                    const int kb = 32 * wd, ke = min(kn, kb + 32);
                    uint32_t addr = s_xs + (uint32_t)kb * rowb + 4u * (uint32_t)c;
                    uint32_t word = 0u;
                    if (FAST) {
                        // kept bits from the whole-source sketch; the column's largest key
                        // (first largest |x|) is the fallback row of an empty column
                        unsigned long long kmax = 0ull;
                        const uint32_t gm = s_gm + 4u * (uint32_t)(c >> 5), gsh = (uint32_t)(c & 31);
                        for (int k = kb; k < ke; ++k, addr += rowb) {
                            const uint32_t a = abs_bits(lds_f32(addr));
                            const unsigned long long kk = ((unsigned long long)a << 32) | (0xFFFFFFFFu - (uint32_t)(k0 + k));
                            kmax = kk > kmax ? kk : kmax;
                            word |= ((lds_u32(gm + 4u * (uint32_t)(k * B.gwords)) >> gsh) & 1u) << (k - kb);
                        }
                        atomicMax(&s_amax[c], kmax);
                        if (word) atomicAdd(&s_cnt[c], __popc(word));
                    } else {
                        const uint64_t T = s_thr[c];
                        const uint32_t Ta = (uint32_t)(T >> 32), Tk = 0xFFFFFFFFu - (uint32_t)T;
                        for (int k = kb; k < ke; ++k, addr += rowb) {
                            const uint32_t a = abs_bits(lds_f32(addr));
                            const bool keep = a > Ta || (a == Ta && (uint32_t)(k0 + k) <= Tk);
                            word |= (uint32_t)keep << (k - kb);
                        }
                    }
                    sts_u32(s_bits + 4u * (uint32_t)(c * nw + wd), word);
                }
                __syncthreads();
                if (!persist) {
                    for (int j = 0; j < my_cols; ++j) {
                        const int c = warp + j * nwarps;
                        bitmap_to_list(s_bits + 4u * (uint32_t)(c * nw), nwk, s_lists + 2u * (uint32_t)(c * CH), lane);
                        if (lane == 0) {
                            int w = 0;
                            for (int wd = 0; wd < nwk; ++wd) w += __popc(lds_u32(s_bits + 4u * (uint32_t)(c * nw + wd)));
                            sts_u32(s_lens + 4u * c, (uint32_t)w);
                        }
                    }
                    __syncwarp();
                }
            }
            if (persist) {
                if constexpr (F64) {
                    owned_accumulate_f64<CPL>(S, M, s_xs, sx, s_ys, nf, kn, full, s_bits, nw);
                } else {
                owned_accumulate<CPL>(S, M, s_xs, sx, s_ys, nf, kn, full, s_bits, nw);
                // fold every kFoldChunks chunks and at the item's end (entries owned by this lane only)
                const int fold = B.fold_chunks > 0 ? B.fold_chunks : kFoldChunks;
                if (((k0 - kbeg) / CH) % fold == fold - 1 || k0 + CH >= kend)
                    owned_fold<CPL>(S, M, nf, G64);
                }
            } else {
                for (int j = 0; j < my_cols; ++j) {
                    const int c = warp + j * nwarps;
                    const int lc = full ? kn : (int)lds_u32(s_lens + 4u * c);
                    sparse_gram_owned<CPL>(s_xs, sx, s_ys, nf, lc, full, s_lists, CH, c, nwarps, 1, 0.f, G, lane,
                                           k0 != kbeg);
                }
            }
        }
        // single-item rows: finished normal equations (+ lam*n*I) straight into gbuf
        const bool direct = r >= B.n_multi;
        double* out = direct ? A.gbuf + (size_t)r * nf * gs : B.part + (size_t)t * nf * gs;
        const float lam_n = direct ? (float)(A.lam * (double)n) : 0.f;
        if (persist) {
            if constexpr (F64) owned_flush_f64<CPL>(S, M, nf, out, direct ? A.lam * (double)n : 0.0);
            else owned_flush64<CPL>(M, nf, G64, out, direct ? A.lam * (double)n : 0.0);
        } else {
            __syncthreads();
            for (int e = tid; e < nf * gs; e += nt) {
                const int c = e / gs, f = e - c * gs;
                out[e] = G[e] + ((c == f) ? lam_n : 0.f);
            }
        }
        if (A.rss_rows != nullptr) {
            racc = block_sum_d(racc, red);
            if (tid == 0) {
                if (direct) A.rss_rows[row] = racc;
                else B.rss_part[t] = racc;
            }
        }
        if (FAST && !full) {
            __syncthreads();  // flushed rows (global) and the column counts are complete
            if (direct) {
                // empty sketched columns: the first largest-|x| slice row alone (_kernels.py:196-211)
                for (int c = warp; c < nf; c += nwarps) {
                    if (s_cnt[c] != 0) continue;
                    const int k = (int)(0xFFFFFFFFu - (uint32_t)s_amax[c]);
                    const float* xr = A.src + (int64_t)__ldg(A.idx + lo + k) * A.ld_src;
                    const float v = __ldg(xr + c);
                    double* grow = out + (size_t)c * gs;
                    for (int f = lane; f < nf; f += 32) grow[f] = fma((double)v, (double)__ldg(xr + f), grow[f]);
                    if (lane == 0) grow[nf] = fma((double)v, (double)__ldg(A.val + lo + k), grow[nf]);
                }
            } else if (tid < nf) {
                atomicAdd(&B.fcnt[(size_t)r * nf + tid], s_cnt[tid]);
                atomicMax(&B.famax[(size_t)r * nf + tid], s_amax[tid]);
            }
        }
    }
}

// fast_core, multi-item rows [0, n_multi): the empty-column fallback on the
// reduced normal equations (gbuf slot r), warp per (row, column).
__global__ void __launch_bounds__(kThreads) fast_fix_kernel(SweepArgs A, BigArgs B) {
    const int nf = A.nf, gs = nf + 1;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = gw; w < B.n_multi * nf; w += wstride) {
        const int r = (int)(w / nf), c = (int)(w % nf);
        if (B.fcnt[(size_t)r * nf + c] != 0) continue;
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int k = (int)(0xFFFFFFFFu - (uint32_t)B.famax[(size_t)r * nf + c]);
        const float* xr = A.src + (int64_t)__ldg(A.idx + lo + k) * A.ld_src;
        const float v = __ldg(xr + c);
        double* grow = A.gbuf + (size_t)r * nf * gs + (size_t)c * gs;
        for (int f = lane; f < nf; f += 32) grow[f] = fma((double)v, (double)__ldg(xr + f), grow[f]);
        if (lane == 0) grow[nf] = fma((double)v, (double)__ldg(A.val + lo + k), grow[nf]);
    }
}

// ---- whole-source sketch (method 'fast_core', core.py:276-286) ---------------
// Per column the s-th largest key (abs_bits << 32 | ~row) of the source by an
// 8-pass MSD radix select (8 bits per pass): histogram of the undecided byte of
// the keys that match the decided prefix, then one warp per column picks the
// byte holding rank s.  Columns in groups of 32 per block (32 x 256 counters).
__global__ void __launch_bounds__(256) fast_hist_kernel(const float* __restrict__ src, int64_t n_src, int ld, int nf,
                                                       int pass, const unsigned long long* __restrict__ prefix,
                                                       unsigned int* __restrict__ hist) {
    __shared__ unsigned int h[32 * 256];
    __shared__ unsigned long long pre[32];
    const int c0 = blockIdx.y * 32, gc = min(32, nf - c0);
    const int sh = 56 - 8 * pass;
    for (int e = threadIdx.x; e < 32 * 256; e += blockDim.x) h[e] = 0u;
    if (threadIdx.x < gc) pre[threadIdx.x] = prefix[c0 + threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (lane < gc) {
        const unsigned long long p = pre[lane];
        for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < n_src;
             j += (int64_t)gridDim.x * (blockDim.x >> 5)) {
            const unsigned long long key =
                ((unsigned long long)abs_bits(__ldg(src + j * ld + c0 + lane)) << 32) | (0xFFFFFFFFu - (uint32_t)j);
            if (pass == 0 || (key >> (sh + 8)) == (p >> (sh + 8)))
                atomicAdd(&h[lane * 256 + (int)((key >> sh) & 255u)], 1u);
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < gc * 256; e += blockDim.x)
        if (h[e]) atomicAdd(&hist[(size_t)c0 * 256 + e], h[e]);
}

__global__ void __launch_bounds__(256) fast_pick_kernel(int nf, int64_t s, int pass, unsigned long long* prefix,
                                                       unsigned long long* above, unsigned int* hist) {
    const int lane = threadIdx.x & 31;
    const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (c >= nf) return;
    const int sh = 56 - 8 * pass;
    unsigned int* hc = hist + (size_t)c * 256;
    unsigned long long ab = above[c];
    // bins from the top: lane l owns bins 255 - 8l .. 248 - 8l
    unsigned long long part = 0;
    unsigned int cnt[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        cnt[i] = hc[255 - 8 * lane - i];
        part += cnt[i];
    }
    unsigned long long incl = part;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const unsigned long long before = incl - part;  // keys in higher bins (this pass)
    const bool here = ab + before < (unsigned long long)s && (unsigned long long)s <= ab + incl;
    const uint32_t who = __ballot_sync(0xffffffffu, here);
    if (who && lane == __ffs(who) - 1) {
        unsigned long long acc = ab + before;
        int bin = 255 - 8 * lane;
        for (int i = 0; i < 8; ++i) {
            if (acc + cnt[i] >= (unsigned long long)s) { bin = 255 - 8 * lane - i; break; }
            acc += cnt[i];
        }
        prefix[c] |= (unsigned long long)bin << sh;
        above[c] = acc;
    }
    __syncwarp();
    for (int i = lane; i < 256; i += 32) hc[i] = 0u;
}

__global__ void __launch_bounds__(256) fast_mask_kernel(const float* __restrict__ src, int64_t n_src, int ld, int nf,
                                                       const unsigned long long* __restrict__ thr, int gwords,
                                                       uint32_t* __restrict__ gmask) {
    const int64_t total = n_src * gwords;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / gwords;
        const int wi = (int)(e - j * gwords);
        uint32_t word = 0u;
        const int cb = 32 * wi, ce = min(nf, cb + 32);
        for (int c = cb; c < ce; ++c) {
            const unsigned long long key =
                ((unsigned long long)abs_bits(__ldg(src + j * ld + c)) << 32) | (0xFFFFFFFFu - (uint32_t)j);
            word |= (key >= __ldg(thr + c) ? 1u : 0u) << (c - cb);
        }
        gmask[e] = word;
    }
}

template __global__ void big_gram_kernel<1, false>(SweepArgs, BigArgs);
template __global__ void big_gram_kernel<2, false>(SweepArgs, BigArgs);
template __global__ void big_gram_kernel<4, false>(SweepArgs, BigArgs);
template __global__ void big_gram_kernel<8, false>(SweepArgs, BigArgs);
template __global__ void big_gram_kernel<1, true>(SweepArgs, BigArgs);
template __global__ void big_gram_kernel<2, true>(SweepArgs, BigArgs);
template __global__ void big_gram_kernel<4, true>(SweepArgs, BigArgs);
template __global__ void big_gram_kernel<8, true>(SweepArgs, BigArgs);
template __global__ void big_gram_kernel<4, false, true>(SweepArgs, BigArgs);

// Big rows [r0, r0 + count): fixed-order float64 sum of the item partials,
// + lam*n*I on the diagonal -> A.gbuf slot (r - r0); residual partial sums.
__global__ void __launch_bounds__(kThreads) big_reduce_kernel(SweepArgs A, BigArgs B, int64_t r0, int64_t count) {
    const int nf = A.nf, gs = nf + 1, nout = nf * gs;
    for (int64_t q = blockIdx.x; q < count; q += gridDim.x) {
        const int64_t r = r0 + q;
        const int row = B.rows[r];
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const int64_t t0 = B.tile_ptr[r] - B.tile_base, t1 = B.tile_ptr[r + 1] - B.tile_base;
        const double lam_n = A.lam * (double)n;
        double* G = A.gbuf + (size_t)q * nout;
        for (int e = threadIdx.x; e < nout; e += blockDim.x) {
            double v = 0.0;
            for (int64_t t = t0; t < t1; ++t) v += B.part[(size_t)t * nout + e];
            const int c = e / gs, f = e - c * gs;
            G[e] = v + ((c == f) ? lam_n : 0.0);
        }
        if (A.rss_rows != nullptr && threadIdx.x == 0) {
            double v = 0.0;
            for (int64_t t = t0; t < t1; ++t) v += B.rss_part[t];
            A.rss_rows[row] = v;
        }
    }
}

}  // namespace cals
