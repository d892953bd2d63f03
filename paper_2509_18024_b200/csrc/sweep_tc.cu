// sweep_tc.cu -- the tiled tier's sketched Gram on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, accumulators in TMEM), for 32 < n_f <= 64.
//
// The reference's gram_rhs_global (_kernels.py:123-146) sums, per column c,
// G[c][:] += x_kc * [x_k | y_k] over the slice rows k kept for c -- a masked
// contraction G = (P o X)^T [X | y] with a different kept set per column.  On
// the tensor cores it runs DENSE (1/rate times the kept work), exactly:
//
//   * every factor column c (and the ratings y) is scaled by a power of two
//     alpha_c so |x / alpha_c| < 1/2, rounded to a 32-bit fixed-point integer
//     X = rint(x * 2^32 / alpha_c) and split into four signed bytes,
//     x / alpha_c = sum_{L=1..4} d_L 2^(-8L)  (Ozaki-style digit split; the
//     only approximation is that rounding, |err| <= 2^-33 alpha_c, about
//     2^-31 of the column maximum);
//   * digit products are exact int8 x int8 -> int32 and accumulate exactly in
//     TMEM (no fp32 sums anywhere: the summation error that made an fp32 Gram
//     miss the 1e-4 contract on ill-conditioned long rows is gone);
//   * the level pairs (a, b) with a + b <= 5 (plus a few of 6) are covered by
//     three M=128 x N=144 x K=32 MMAs per 32 slice rows: the M side stacks two
//     levels of the MASKED digits p_kc * x_kc (rows (level, c)), the N side two
//     levels of the unmasked digits of x_kf and y_k (columns (level, f), y at
//     f = 64), so the right-hand side b = X*^T y comes out of the same MMAs;
//   * the work item's G and b are recombined once, in float64, from the TMEM
//     integers and the power-of-two weights (exact products, one rounding per
//     term).
//
// Numerically this is a float64-quality Gram (measured: 2^-31-relative inputs,
// exact sums; a numpy emulation at cond ~1e6 gives ~5e-7 factor error where
// fp32 products give ~2e-4).
//
// Pipeline per CTA (one per SM, 14 warps, warp-specialised, mbarrier handoffs):
//   * warp 13, scheduler: resolves 32 work items at a time lane-parallel (row,
//     rating range, slice rows) into an 8-deep item ring, and copies each
//     item's selection thresholds and previous row into it with cp.async (the
//     ring slot's barrier completes when they land: no warp waits on memory);
//   * warps 0..7, digit pass: every lane gathers ITS OWN 64 bytes of a slice
//     row (four 16-byte cp.async, three chunks ahead, swizzled lane-private
//     staging) and its rating, then turns them into kept bits, fixed point and
//     the 4 signed digits, written into one of two K-step tile sets;
//   * warp 12, lane 0: issues the chunk's 3 MMAs per 32 rows once its tile
//     set is complete and commits them to that set's "empty" barrier;
//   * warps 8..11, epilogue (one TMEM lane quarter each): drain the
//     accumulators into float64 (then the next item's MMAs may start), add
//     the exception rows, write the normal equations, release the ring slot.
#include "sweep_common.cuh"
#include "tc.cuh"

namespace cals {

constexpr int kTcKC = 64;                       // slice rows per chunk (two K-steps of 32)
constexpr int kTcCW = 8;                        // digit-pass warps
constexpr int kTcRW = kTcKC / kTcCW;            // slice rows per digit-pass warp per chunk (4)
constexpr int kTcLPR = 32 / kTcRW;              // lanes per slice row (8)
constexpr int kTcNG = 64 / (4 * kTcLPR);        // groups of 4 columns per lane (2)
constexpr int kTcEW = 4;                        // epilogue warps (TMEM lane quarters)
constexpr int kTcMmaWarp = kTcCW + kTcEW;       // MMA issue
constexpr int kTcSchedWarp = kTcMmaWarp + 1;    // work-item scheduler
constexpr int kTcThreads = (kTcSchedWarp + 1) * 32;
constexpr int kTcStages = 5;                    // lane-private cp.async staging ring
constexpr int kTcAhead = kTcStages - 1;         // chunks gathered ahead of the digit pass
constexpr int kTcRing = 16;                     // index ring slots (>= 2 kTcAhead + 1)
constexpr int kTcStageX = kTcKC * 64 * 4;       // 64 rows x 64 floats (lane-private 64-byte segments)
constexpr int kTcN = 144;                       // N side: two levels x (64 factor columns + y + 7 zero pad)
constexpr int kTcLvl = 72;                      // N columns per level
constexpr int kTcATile = 4096;                  // M = 128 (two levels x 64 columns) x 32 K bytes
constexpr int kTcBTile = 4608;                  // N = 144 x 32 K bytes
constexpr int kTcKStepBytes = 2 * kTcATile + 2 * kTcBTile;  // A12 A34 B12 B34
constexpr int kTcDigitBuf = 2 * kTcKStepBytes;              // one chunk (two K-steps)
constexpr int kTcAccB = 256;                    // TMEM column of the second accumulator (levels 4..6)
constexpr int kTcItems = 16;                    // work-item ring
constexpr int kTcGrab = 8;                      // work items claimed per counter increment
constexpr int kTcExcSlots = 4;                  // exception masks: items in flight past the epilogue <= 3
constexpr int kTcMaxChunks = 256;               // chunks per work item (item_rows <= 16384)
constexpr int kTcExcBatch = 32;                 // exception rows staged per epilogue round (half a chunk)
constexpr float kTcLimit = 2.13e9f;             // |x * 2^32 / alpha| below this keeps the top digit in int8

struct TcItem {             // one work item in the ring (written by the scheduler warp)
    uint64_t T[64];         // selection thresholds (~0: padding column, never kept)
    float wold[64];         // previous row (fused residual)
    int64_t lo;             // first rating of the row
    int64_t t;              // batch-relative work item; -1 ends the CTA's list
    int n, kbeg, kend, r, row, pad[3];
};

struct TcSmem {
    static constexpr int stage_x = 0;                                          // [4] lane-private rows
    static constexpr int ring = stage_x + kTcStages * kTcStageX;               // [R][64] idx, [R][64] f32 y
    static constexpr int digits = (ring + 2 * kTcRing * kTcKC * 4 + 1023) & ~1023;  // [2] tile sets
    static constexpr int xchg = digits + 2 * kTcDigitBuf;                      // [64][72] f64
    static constexpr int exc_x = xchg + 64 * kTcLvl * 8;                       // [64][72] f32 (+ y, k)
    static constexpr int exc_mask = exc_x + kTcExcBatch * kTcLvl * 4;          // [4][256][2] u32
    static constexpr int items = exc_mask + kTcExcSlots * kTcMaxChunks * 8;    // [8] TcItem
    static constexpr int rss = items + kTcItems * (int)sizeof(TcItem);         // [8][kTcCW] f64
    static constexpr int total = rss + kTcItems * kTcCW * 8;
};
static_assert(sizeof(TcItem) % 16 == 0, "item ring alignment");

// item-ring threshold slot of column c: the digit pass reads columns 4q .. 4q+3 (q = 8g + lane
// group) as two 16-byte words; lanes 0..7 of a row read 128 contiguous bytes per word
__host__ __device__ constexpr int tperm(int c) {
    return (((c >> 5) * 2 + ((c >> 1) & 1)) * 8 + ((c >> 2) & 7)) * 2 + (c & 1);
}

__host__ __device__ constexpr uint32_t tc_mn_off(uint32_t mn, uint32_t k) {
    return (mn >> 4) * 512u + (k >> 3) * 128u + (k & 7u) * 16u + (mn & 15u);
}

// low bytes of four words -> one word
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mbar) : "memory");
}
// arrive on `mbar` once every cp.async this thread issued so far has landed (counts as one of
// the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(uint32_t mbar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t saddr, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem));
}

// Digit scales of one half-sweep.  Factor column c: alpha_c = 2^E with alpha_c > 32.25 q_c,
// q_c the table's top level (the rating-weighted 1/256 quantile of |source[:, c]|), so
// values up to ~16 q_c keep the top digit in int8; ratings: alpha_y > 8.06 m_y, m_y the
// maximum of a strided sample.  Larger values (heavy-tailed factor rows) are exceptions:
// their slice rows leave the MMAs and are added exactly in float64 at the item's end.
// out_scale[c] = 2^(32 - E_c) (x -> fixed point), out_alpha[c] = 2^E_c; index 64 = y.
__global__ void __launch_bounds__(256) tc_scales_kernel(const uint32_t* __restrict__ qtab, int nf,
                                                        const float* __restrict__ val, int64_t nnz,
                                                        float* __restrict__ out_scale, double* __restrict__ out_alpha) {
    __shared__ float red[8];
    float m = 0.f;
    const int S = 4096;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        const int64_t pos = nnz > 0 ? (int64_t)(((double)i + 0.5) * (double)nnz / S) : 0;
        if (nnz > 0) m = fmaxf(m, fabsf(val[min(pos, nnz - 1)]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(CALS_FULL_MASK, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    auto put = [&](int c, float bound) {
        int e = -60;
        if (bound > 0.f) {
            frexpf(bound, &e);
            e = max(e, -60);
        }
        out_scale[c] = ldexpf(1.0f, 32 - e);
        out_alpha[c] = ldexp(1.0, e);
    };
    if (threadIdx.x == 0) {
        float my = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) my = fmaxf(my, red[w]);
        put(64, my * 8.0625f);
    }
    if (threadIdx.x < 64) {
        const int c = threadIdx.x;
        const float q = c < nf ? __uint_as_float(qtab[(size_t)c * (kQ + 1) + 1]) : 0.f;
        if (c < nf) put(c, q * 32.25f);
        else { out_scale[c] = 0.f; out_alpha[c] = 0.0; }
    }
}

// profiling trace (tc_debug 8, CALS_TC_TRACE builds): timestamps of CTA 0 of launch A.stats[49149]
// into A.stats (>= 49152 words; A.stats[49150] counts launches)
#ifndef CALS_TC_TRACE
#define CALS_TC_TRACE 0
#endif
#define TC_TRACE(slot, cond)                                                                   \
    do {                                                                                       \
        if (CALS_TC_TRACE && trace && (cond)) A.stats[(slot)] = (unsigned long long)clock64(); \
    } while (0)

// Long waits of the role warps (a whole work item).  A try_wait loop is the default: each
// attempt blocks the warp for a few tens of cycles in hardware, so a waiting warp issues ~0.1
// instructions per cycle; the nanosleep(128) poll it replaces returned at once and its four
// epilogue warps + scheduler took ~45 % of the kernel's issue slots (ncu, r02).  tc_debug
// 256: try_wait with a suspend-time hint; 512: the old test + nanosleep poll.
__device__ __forceinline__ void tc_long_wait(uint32_t mbar, uint32_t phase, int dbg) {
    if (dbg & 256) mbar_wait_hint(mbar, phase);
    else if (dbg & 512) mbar_wait_backoff(mbar, phase);
    else mbar_wait(mbar, phase);
}

// Work-item cursor of the digit-pass warps (item ring position + chunk start).
struct TcCur {
    int i;       // item sequence number (ring slot i % kTcItems)
    int k0;      // first slice row of the chunk
    int kbeg, kend;
    int64_t lo;
    bool ok;     // false past the CTA's last item
};

__device__ __forceinline__ void tc_enter(TcCur& c, const TcItem* items, uint32_t full_base) {
    const int sl = c.i % kTcItems;
    mbar_wait(full_base + 8u * (uint32_t)sl, (uint32_t)((c.i / kTcItems) & 1));
    const TcItem& d = items[sl];
    c.ok = d.t >= 0;
    c.kbeg = d.kbeg;
    c.kend = d.kend;
    c.k0 = d.kbeg;
    c.lo = d.lo;
}
__device__ __forceinline__ void tc_advance(TcCur& c, const TcItem* items, uint32_t full_base) {
    c.k0 += kTcKC;
    if (c.k0 >= c.kend) {
        ++c.i;
        tc_enter(c, items, full_base);
    }
}

__global__ void __launch_bounds__(kTcThreads, 1) big_gram_tc_kernel(SweepArgs A, BigArgs B,
                                                                    const float* __restrict__ g_scale,
                                                                    const double* __restrict__ g_alpha, int dbg) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(16) float s_scale[68];
    __shared__ double s_alpha[65];
    __shared__ uint32_t s_tmem;
    __shared__ uint32_t exc_any[kTcExcSlots];  // item had an exception row (the epilogue scans its masks)
    // every mbarrier in one array, addressed as full_base + a compile-time offset (separate arrays cost a
    // generic-to-shared conversion per use inside the role loops): item_full[kTcItems], item_empty[kTcItems],
    // item_done[kTcItems], full_tl[2], empty_tl[2], tmem_full, tmem_empty
    __shared__ __align__(8) unsigned long long bars[3 * kTcItems + 6];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nf = A.nf, gs = nf + 1;
    const bool want_rss = A.rss_rows != nullptr;
    // tracing (tc_debug 3): CTA 0 of the first launch after the buffer was cleared
    const bool trace = (dbg & 8) && blockIdx.x == 0 && A.stats != nullptr && A.stats[49150] == A.stats[49149];
    const uint32_t sbase = tc::smem_addr(smem);
    unsigned char* digits = smem + TcSmem::digits;
    double* xchg = reinterpret_cast<double*>(smem + TcSmem::xchg);
    float* exc_x = reinterpret_cast<float*>(smem + TcSmem::exc_x);
    uint32_t* exc_mask = reinterpret_cast<uint32_t*>(smem + TcSmem::exc_mask);  // [slot][chunk][2]
    TcItem* items = reinterpret_cast<TcItem*>(smem + TcSmem::items);
    double* rss_part = reinterpret_cast<double*>(smem + TcSmem::rss);
    const uint32_t full_base = smem_u32(&bars[0]);

    // ---- setup, then the roles never meet at a block barrier again
    for (int e = tid; e < 2 * kTcDigitBuf / 16; e += blockDim.x)
        reinterpret_cast<uint4*>(digits)[e] = make_uint4(0u, 0u, 0u, 0u);  // padding bytes stay zero
    for (int e = tid; e < kTcExcSlots * kTcMaxChunks * 2; e += blockDim.x) exc_mask[e] = 0u;
    for (int e = tid; e < kTcStages * kTcStageX / 16; e += blockDim.x)
        reinterpret_cast<uint4*>(smem + TcSmem::stage_x)[e] = make_uint4(0u, 0u, 0u, 0u);  // padding columns stay 0
    if (tid < kTcExcSlots) exc_any[tid] = 0u;
    if (tid < 68) s_scale[tid] = tid < 65 ? g_scale[tid] : 0.f;
    if (tid < 65) {
        s_alpha[tid] = g_alpha[tid];
    }
    if (warp == 0) tc::tmem_alloc<512>(&s_tmem);
    if (tid == 0) {
        for (int s = 0; s < kTcItems; ++s) {
            mbar_init((full_base + 8u * (uint32_t)(0 + (s))), 64);  // 32 lanes x (descriptor writes + their copies)
            mbar_init((full_base + 8u * (uint32_t)(kTcItems + (s))), 1);
            mbar_init((full_base + 8u * (uint32_t)(2 * kTcItems + (s))), kTcCW);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init((full_base + 8u * (uint32_t)(3 * kTcItems + (s))), kTcCW);
            mbar_init((full_base + 8u * (uint32_t)(3 * kTcItems + 2 + (s))), 1);
        }
        mbar_init((full_base + 8u * (uint32_t)(3 * kTcItems + 4)), 1);
        mbar_init((full_base + 8u * (uint32_t)(3 * kTcItems + 5)), 1);
    }
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == kTcSchedWarp) {
        // ================= scheduler: work items -> ring (lane-parallel resolution) =================
        // items are claimed kTcGrab at a time from one counter (longest first: rows are sorted by
        // length), so CTAs that start late or draw long items simply claim fewer
        int i = 0;
        bool more = true;
        while (more) {
            int base = 0;
            if (lane == 0) base = atomicAdd(B.item_ctr, kTcGrab);
            base = __shfl_sync(CALS_FULL_MASK, base, 0);
            const int64_t t = (int64_t)base + lane;
            int r = 0, row = 0, n = 0, kbeg = 0, kend = 0;
            int64_t lo = 0;
            if (lane < kTcGrab && t < B.n_tiles) {
                const int64_t T_abs = B.tile_base + t;
                if (B.tile_row != nullptr) {
                    r = (int)(__ldg(B.tile_row + T_abs) - B.row_base);
                } else {
                    int64_t a = 0, b = B.n_big - 1;
                    while (a < b) {
                        const int64_t mid = (a + b + 1) >> 1;
                        if (B.tile_ptr[mid] <= T_abs) a = mid; else b = mid - 1;
                    }
                    r = (int)a;
                }
                row = B.rows[r];
                lo = A.ptr[row];
                n = (int)(A.ptr[row + 1] - lo);
                kbeg = (int)(T_abs - B.tile_ptr[r]) * B.item_rows;
                kend = min(n, kbeg + B.item_rows);
            }
            for (int l = 0; l < kTcGrab && more; ++l, ++i) {
                const int64_t tl = __shfl_sync(CALS_FULL_MASK, t, l);
                const bool valid = tl < B.n_tiles;
                const int rl = __shfl_sync(CALS_FULL_MASK, r, l), rowl = __shfl_sync(CALS_FULL_MASK, row, l);
                const int nl = __shfl_sync(CALS_FULL_MASK, n, l), kbl = __shfl_sync(CALS_FULL_MASK, kbeg, l);
                const int kel = __shfl_sync(CALS_FULL_MASK, kend, l);
                const int64_t lol = __shfl_sync(CALS_FULL_MASK, lo, l);
                const int sl = i % kTcItems;
                if (i >= kTcItems) tc_long_wait((full_base + 8u * (uint32_t)(kTcItems + (sl))), (uint32_t)(((i / kTcItems) - 1) & 1), dbg);
                TcItem& d = items[sl];
                if (lane == 0) {
                    d.t = valid ? tl : -1;
                    d.lo = lol;
                    d.n = nl;
                    d.kbeg = kbl;
                    d.kend = kel;
                    d.r = rl;
                    d.row = rowl;
                }
                if (valid) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = lane + 32 * h;
                        if (c < nf) cp_async8(smem_u32(&d.T[tperm(c)]), B.thr + (size_t)rl * nf + c);
                        else d.T[tperm(c)] = ~0ull;
                        if (want_rss && c < nf) cp_async4(smem_u32(&d.wold[c]), A.tgt_old + (int64_t)rowl * A.ld_old + c);
                        else d.wold[c] = 0.f;
                    }
                }
                const uint32_t fb = (full_base + 8u * (uint32_t)(0 + (sl)));
                TC_TRACE(40960 + i, lane == 0 && i < 8192);
                mbar_arrive(fb);           // this lane's descriptor / padding writes
                cp_async_mbar_arrive(fb);  // and, asynchronously, its copies
                more = valid;
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ================= MMA issue (one thread) =================
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_i8(128, kTcN) | (1u << 15) | (1u << 16);  // MN-major A and B
            int64_t j = 0;
            for (int i = 0;; ++i) {
                const int sl = i % kTcItems;
                mbar_wait(full_base + 8u * (uint32_t)sl, (uint32_t)((i / kTcItems) & 1));
                const TcItem& d = items[sl];
                if (d.t < 0) break;
                const int kbeg = d.kbeg, kend = d.kend;
                for (int k0 = kbeg; k0 < kend; k0 += kTcKC, ++j) {
                    const int db = (int)(j & 1);
                    if (dbg & 16) mbar_wait_hint((full_base + 8u * (uint32_t)(3 * kTcItems + (db))), (uint32_t)((j >> 1) & 1));
                    else if (dbg & 64) {
                        while (!mbar_test((full_base + 8u * (uint32_t)(3 * kTcItems + (db))), (uint32_t)((j >> 1) & 1))) __nanosleep(20);
                    } else mbar_wait((full_base + 8u * (uint32_t)(3 * kTcItems + (db))), (uint32_t)((j >> 1) & 1));
                    TC_TRACE(j * 8 + 4, j < 4096);
                    if (k0 == kbeg && i > 0) mbar_wait((full_base + 8u * (uint32_t)(3 * kTcItems + 5)), (uint32_t)((i - 1) & 1));
                    TC_TRACE(j * 8 + 5, j < 4096);
                    if (trace && j < 4096) A.stats[j * 8 + 6] = (unsigned long long)i;
                    tc::fence_after();
                    const int nks = (min(kTcKC, kend - k0) + 31) >> 5;
                    for (int ks = 0; ks < ((dbg & 1) ? 0 : nks); ++ks) {
                        const uint32_t base = sbase + TcSmem::digits + (uint32_t)(db * kTcDigitBuf + ks * kTcKStepBytes);
                        const uint64_t a12 = tc::sdesc(base, 128, 512), a34 = tc::sdesc(base + kTcATile, 128, 512);
                        const uint64_t b12 = tc::sdesc(base + 2 * kTcATile, 128, 512);
                        const uint64_t b34 = tc::sdesc(base + 2 * kTcATile + kTcBTile, 128, 512);
                        const uint32_t acc = (k0 == kbeg && ks == 0) ? 0u : 1u;
                        tc::mma_i8_ss(tmem, a12, b12, idesc, acc);
                        tc::mma_i8_ss(tmem + kTcAccB, a12, b34, idesc, acc);
                        tc::mma_i8_ss(tmem + kTcAccB, a34, b12, idesc, 1u);
                    }
                    tc::commit((full_base + 8u * (uint32_t)(3 * kTcItems + 2 + (db))));
                    if (k0 + kTcKC >= kend) tc::commit((full_base + 8u * (uint32_t)(3 * kTcItems + 4)));
                }
            }
        }
    } else if (warp >= kTcCW) {
        // ================= epilogue (warps 8..11 = TMEM lane quarters 0..3) =================
        const int ew = warp - kTcCW, et = tid - kTcCW * 32;
        const uint32_t lrow = (uint32_t)(32 * ew) << 16;
        for (int i = 0;; ++i) {
            const int sl = i % kTcItems, xs = i % kTcExcSlots;
            mbar_wait(full_base + 8u * (uint32_t)sl, (uint32_t)((i / kTcItems) & 1));
            const TcItem& d = items[sl];
            if (d.t < 0) break;
            TC_TRACE(32768 + i * 8 + 0, et == 0 && i < 1024);
            tc_long_wait((full_base + 8u * (uint32_t)(2 * kTcItems + (sl))), (uint32_t)((i / kTcItems) & 1), dbg);
            TC_TRACE(32768 + i * 8 + 1, et == 0 && i < 1024);
            mbar_wait((full_base + 8u * (uint32_t)(3 * kTcItems + 4)), (uint32_t)(i & 1));
            TC_TRACE(32768 + i * 8 + 2, et == 0 && i < 1024);
            tc::fence_after();
            // per TMEM row (level h of column c) and column f, the four accumulators combine exactly
            // in 64-bit integers: I = a0 2^24 + a1 2^16 + b0 2^8 + b1 (|a| < 2^29: |I| < 2^53, so its
            // conversion to float64 is exact); G[c][f] = alpha_c alpha_f (2^-40 I_level1 + 2^-48 I_level2)
            auto drain = [&](int f0, uint32_t (&a0)[8], uint32_t (&a1)[8], uint32_t (&b0)[8], uint32_t (&b1)[8]) {
                tc::ld_32x32b_x8(tmem + lrow + f0, a0);
                tc::ld_32x32b_x8(tmem + lrow + kTcLvl + f0, a1);
                tc::ld_32x32b_x8(tmem + lrow + kTcAccB + f0, b0);
                tc::ld_32x32b_x8(tmem + lrow + kTcAccB + kTcLvl + f0, b1);
                tc::ld_wait();
            };
            auto combine = [](uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
                const long long I = ((long long)(int)a0 << 24) + ((long long)(int)a1 << 16) +
                                    ((long long)(int)b0 << 8) + (long long)(int)b1;
                return (double)I;
            };
            // both warp pairs drain at once, on opposite column halves: level-1 warps (TMEM rows 0..63) take
            // columns [0, 40) first, level-2 warps (rows 64..127) [40, 72); after the barrier they swap.  The
            // first visitor of (c, f) leaves its exact scaled integer, the second adds its own with one
            // rounding and applies alpha_c alpha_f -- the same value in either order -- so TMEM is held for
            // 5 + 5 column blocks instead of 9 + 9 (the next item's MMAs wait on this drain)
            {
                const bool lvl2 = ew >= 2;
                const int cr = 32 * (ew & 1) + lane;
                const double ac = s_alpha[cr];
                const double wscale = lvl2 ? 0x1p-48 : 0x1p-40;
                for (int f0 = lvl2 ? 40 : 0; f0 < (lvl2 ? kTcLvl : 40); f0 += 8) {
                    uint32_t a0[8], a1[8], b0[8], b1[8];
                    drain(f0, a0, a1, b0, b1);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        xchg[cr * kTcLvl + f0 + q] = combine(a0[q], a1[q], b0[q], b1[q]) * wscale;  // exact
                }
                named_bar(1, 128);
                for (int f0 = lvl2 ? 0 : 40; f0 < (lvl2 ? 40 : kTcLvl); f0 += 8) {
                    uint32_t a0[8], a1[8], b0[8], b1[8];
                    drain(f0, a0, a1, b0, b1);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int f = f0 + q;
                        const double p = fma(combine(a0[q], a1[q], b0[q], b1[q]), wscale, xchg[cr * kTcLvl + f]);
                        xchg[cr * kTcLvl + f] = ac * s_alpha[f <= 64 ? f : 64] * p;
                    }
                }
            }
            tc::fence_before();
            named_bar(1, 128);
            if (et == 0) mbar_arrive((full_base + 8u * (uint32_t)(3 * kTcItems + 5)));  // the next item's MMAs may start
            TC_TRACE(32768 + i * 8 + 3, et == 0 && i < 1024);
            // exception rows (a value past its column's digit range), chunk by chunk in slice
            // order: their exact float64 contributions, G[c][:] += x_kc [x_k | y_k] if k is kept for c
            const int nchunks = (d.kend - d.kbeg + kTcKC - 1) / kTcKC;
            uint32_t* em = exc_mask + xs * kTcMaxChunks * 2;
            const bool any_exc = exc_any[xs] != 0u;
            for (int q = 0; q < (any_exc ? 2 * nchunks : 0); ++q) {  // 32-row halves of the chunks, in slice order
                const uint32_t m = em[q];
                if (m == 0u) continue;
                named_bar(1, 128);  // exc_x free, mask read by every epilogue thread
                if (et == 0) em[q] = 0u;
                const int ne = __popc(m);
                for (int e = et; e < ne * kTcLvl; e += 128) {
                    const int ii = e / kTcLvl, f = e - ii * kTcLvl;
                    const int k = d.kbeg + 32 * q + (int)__fns(m, 0, ii + 1);
                    float v = 0.f;
                    if (f < nf) v = __ldg(A.src + (int64_t)__ldg(A.idx + d.lo + k) * A.ld_src + f);
                    else if (f == 64) v = __ldg(A.val + d.lo + k);
                    else if (f == 65) v = __int_as_float(k);
                    exc_x[ii * kTcLvl + f] = v;
                }
                named_bar(1, 128);
                if (et < nf) {
                    const int cr = et;
                    const uint64_t T = d.T[tperm(cr)];
                    const uint32_t Ta = (uint32_t)(T >> 32), Tk = 0xFFFFFFFFu - (uint32_t)T;
                    for (int ii = 0; ii < ne; ++ii) {
                        const float* xr = exc_x + ii * kTcLvl;
                        const float xc = xr[cr];
                        const uint32_t a = abs_bits(xc), kgl = (uint32_t)__float_as_int(xr[65]);
                        if (!(a > Ta || (a == Ta && kgl <= Tk))) continue;
                        const double xd = (double)xc;
                        double* grow = xchg + cr * kTcLvl;
                        for (int f = 0; f < nf; ++f) grow[f] = fma(xd, (double)xr[f], grow[f]);
                        grow[64] = fma(xd, (double)xr[64], grow[64]);
                    }
                }
            }
            named_bar(1, 128);
            if (et == 0) exc_any[xs] = 0u;
            TC_TRACE(32768 + i * 8 + 4, et == 0 && i < 1024);
            // the normal equations (+ lam*n on the diagonal of a finished row) and the residual
            const bool direct = d.r >= B.n_multi;
            double* out = direct ? A.gbuf + (size_t)d.r * nf * gs : B.part + (size_t)d.t * nf * gs;
            const double lam_n = direct ? A.lam * (double)d.n : 0.0;
            for (int cr = ew; cr < nf; cr += kTcEW) {  // a warp per row: coalesced, no division
                double* orow = out + (size_t)cr * gs;
                const double* xr = xchg + cr * kTcLvl;
                for (int f = lane; f < nf; f += 32) orow[f] = xr[f] + (f == cr ? lam_n : 0.0);
                if (lane == 0) orow[nf] = xr[64];
            }
            if (et == 0 && want_rss) {
                double v = 0.0;
                for (int w = 0; w < kTcCW; ++w) v += rss_part[sl * kTcCW + w];
                if (direct) A.rss_rows[d.row] = v;
                else B.rss_part[d.t] = v;
            }
            named_bar(1, 128);
            TC_TRACE(32768 + i * 8 + 5, et == 0 && i < 1024);
            if (et == 0) mbar_arrive((full_base + 8u * (uint32_t)(kTcItems + (sl))));
        }
    } else {
        // ================= digit pass (warps 0..15): gather, select, split =================
        // lane (kl, fql): slice row kRW * warp + kl of the chunk, columns 4 (kLPR g + fql) + 0..3
        const int kl = lane / kTcLPR, fql = lane % kTcLPR;
        const int krel = kTcRW * warp + kl;  // slice row of this lane within the chunk
        // row-major staging (256 bytes per slice row): the 8 lanes of a row copy and read one
        // contiguous 128-byte segment per group (one shared-memory wavefront each way)
        const uint32_t sx_lane = sbase + TcSmem::stage_x + (uint32_t)krel * 256u;
        // index ring: the slice-row ids and ratings of chunk t in slot t % kTcRing, copied 2 kTcAhead
        // chunks ahead by the row's first lane (so the gathers never wait on an index load)
        const uint32_t ring_idx = sbase + TcSmem::ring + 4u * (uint32_t)krel;
        const uint32_t ring_val = ring_idx + kTcRing * kTcKC * 4;
        // 16-byte segment (kLPR g + fql) of the row; with fewer than 8 lanes per row, odd rows
        // swap 64-byte halves so the rows sharing a quarter-warp phase hit different banks
        auto seg = [&](int g) {
            const uint32_t sg = (uint32_t)(kTcLPR * g + fql) ^ (kTcLPR < 8 ? (uint32_t)(krel & 1) * 4u : 0u);
            return 16u * sg;
        };
        // digit-store offsets of this lane within a tile set: K part (its slice row) + MN part
        // (its first column, per stacked level half); group g adds 1024 bytes (32 columns)
        const uint32_t kk = (uint32_t)(krel & 31);
        const uint32_t dig_lane = sbase + TcSmem::digits + (uint32_t)(krel >> 5) * kTcKStepBytes + tc_mn_off(0u, kk);
        auto mn_part = [](uint32_t mn) { return (mn >> 4) * 512u + (mn & 15u); };
        const uint32_t off_a0 = mn_part(4u * fql), off_a1 = mn_part(64u + 4u * fql);
        const uint32_t off_b0 = off_a0, off_b1 = mn_part(kTcLvl + 4u * fql);
        const uint32_t off_y0 = mn_part(64u), off_y1 = mn_part(kTcLvl + 64u);
        auto issue_idx = [&](const TcCur& q, int slot) {
            if (fql == 0) {
                const uint32_t o = (uint32_t)slot * (kTcKC * 4);
                if (q.ok && q.k0 + krel < q.kend) {
                    cp_async4(ring_idx + o, A.idx + q.lo + q.k0 + krel);
                    cp_async4(ring_val + o, A.val + q.lo + q.k0 + krel);
                } else {
                    sts_u32(ring_idx + o, 0xFFFFFFFFu);  // -1: no row
                }
            }
        };
        auto issue_data = [&](int stage, int slot) {
            const int idx = (int)lds_u32(ring_idx + (uint32_t)slot * (kTcKC * 4));
            if (idx >= 0 && !(dbg & 128)) {
                const float* srow = A.src + (int64_t)idx * A.ld_src;
#pragma unroll
                for (int g = 0; g < kTcNG; ++g) {
                    const int c0 = 4 * (kTcLPR * g + fql);
                    if (c0 < nf) cp_async16(sx_lane + (uint32_t)stage * kTcStageX + seg(g), srow + c0);
                }
            }
        };
        // group t (t >= -kTcAhead) = {indices of chunk t + 2 kTcAhead, rows of chunk t + kTcAhead}
        TcCur q{};
        q.i = 0;
        tc_enter(q, items, full_base);
        auto adv = [&](TcCur& x) {
            if (x.ok) tc_advance(x, items, full_base);
        };
#pragma unroll 1
        for (int t = 0; t < kTcAhead; ++t) {
            issue_idx(q, t);
            adv(q);
            cp_async_commit();
        }
        cp_async_wait<0>();
        __syncwarp();
#pragma unroll 1
        for (int t = 0; t < kTcAhead; ++t) {
            issue_idx(q, kTcAhead + t);
            adv(q);
            issue_data(t, t);
            cp_async_commit();
        }
        TcCur c{};
        c.i = 0;
        tc_enter(c, items, full_base);
        double racc = 0.0;
        // loop-invariant operands in registers: the lane's column scales for the whole launch, its
        // 8 selection thresholds for as long as the work item lasts (reloaded when c.i changes);
        // 135.1 -> 132.9 ms per 500M iteration (the previous row's values as well: 128 registers spill, 142.6)
        float4 scr[kTcNG];
#pragma unroll
        for (int g = 0; g < kTcNG; ++g) scr[g] = *reinterpret_cast<const float4*>(s_scale + 4 * (kTcLPR * g + fql));
        const float sc_y = s_scale[64];
        ulonglong2 thr01[kTcNG], thr23[kTcNG];
        int thr_item = -1;
#pragma unroll 1
        // j: chunks done by this CTA (32-bit: far below 2^32 per launch); s = j % kTcStages kept
        // incrementally (a 64-bit j cost two emulated 64-bit modulo-by-5 sequences per chunk)
        int s = 0;
        for (uint32_t j = 0; c.ok; ++j, s = (s + 1 == kTcStages) ? 0 : s + 1) {
            // group j - kTcAhead landed: the rows of chunk j and the indices of chunk j + kTcAhead
            TC_TRACE(j * 8 + 0, warp == 0 && lane == 0 && j < 4096);
            cp_async_wait<kTcAhead - 1>();
            __syncwarp();
            TC_TRACE(j * 8 + 1, warp == 0 && lane == 0 && j < 4096);
            issue_idx(q, (int)((j + 2 * kTcAhead) % kTcRing));
            adv(q);
            issue_data(s == 0 ? kTcStages - 1 : s - 1, (int)((j + kTcAhead) % kTcRing));  // (j + kTcAhead) % kTcStages
            cp_async_commit();
            TC_TRACE(j * 8 + 7, warp == 0 && lane == 0 && j < 4096);
            const int db = (int)(j & 1);
            const int sl = c.i % kTcItems;
            const TcItem& it_d = items[sl];
            const int kn = min(kTcKC, c.kend - c.k0);
            const bool last = c.k0 + kTcKC >= c.kend;
            const int ci = (c.k0 - c.kbeg) / kTcKC;
            const bool krow = krel < kn;
            const uint32_t kg = (uint32_t)(c.k0 + krel);
            const uint32_t sx = sx_lane + (uint32_t)s * kTcStageX;
            // the lane's 8 elements (2 groups of 4 consecutive columns): fixed point X = rint(x * 2^32 /
            // alpha_c), its four signed digits all at once -- byte i of (X + 0x80808080) ^ 0x80 is the
            // digit of weight 2^(8i) (the +0x80 per byte carries exactly the borrows of a signed-digit
            // split) -- transposed into one word per level; kept bits from the 64-bit selection key
            const uint32_t lo_key = 0xFFFFFFFFu - kg;
            const uint32_t row_on = krow ? 0xFFFFFFFFu : 0u;
            if (dbg & 2) {
                if (j >= 2) mbar_wait((full_base + 8u * (uint32_t)(3 * kTcItems + 2 + (db))), (uint32_t)(((j - 2) >> 1) & 1));
                __syncwarp();
                if (lane == 0) mbar_arrive((full_base + 8u * (uint32_t)(3 * kTcItems + (db))));
                if (last) {
                    if (lane == 0) rss_part[sl * kTcCW + warp] = 0.0;
                    __syncwarp();
                    if (lane == 0) mbar_arrive((full_base + 8u * (uint32_t)(2 * kTcItems + (sl))));
                }
                tc_advance(c, items, full_base);
                continue;
            }
            if (c.i != thr_item) {
                thr_item = c.i;
#pragma unroll
                for (int g = 0; g < kTcNG; ++g) {
                    const int c0 = 4 * (kTcLPR * g + fql);
                    thr01[g] = *reinterpret_cast<const ulonglong2*>(&it_d.T[tperm(c0)]);
                    thr23[g] = *reinterpret_cast<const ulonglong2*>(&it_d.T[tperm(c0 + 2)]);
                }
            }
            uint32_t lev[kTcNG][4];  // [group][level 1..4]
            uint32_t km[kTcNG];
            float amax = 0.f, pdot = 0.f;
#pragma unroll
            for (int g = 0; g < kTcNG; ++g) {
                const int c0 = 4 * (kTcLPR * g + fql);
                const float4 x = lds_f128(sx + seg(g));  // zero in padding columns
                const float4 sc = scr[g];
                const ulonglong2 t01 = thr01[g], t23 = thr23[g];
                const float t0 = x.x * sc.x, t1 = x.y * sc.y, t2 = x.z * sc.z, t3 = x.w * sc.w;
                amax = fmaxf(amax, fmaxf(fmaxf(fabsf(t0), fabsf(t1)), fmaxf(fabsf(t2), fabsf(t3))));
                const uint32_t z0 = (uint32_t)__float2int_rn(t0) + 0x80808080u;
                const uint32_t z1 = (uint32_t)__float2int_rn(t1) + 0x80808080u;
                const uint32_t z2 = (uint32_t)__float2int_rn(t2) + 0x80808080u;
                const uint32_t z3 = (uint32_t)__float2int_rn(t3) + 0x80808080u;
                const uint32_t lo01 = __byte_perm(z0, z1, 0x5140), hi01 = __byte_perm(z0, z1, 0x7362);
                const uint32_t lo23 = __byte_perm(z2, z3, 0x5140), hi23 = __byte_perm(z2, z3, 0x7362);
                lev[g][3] = __byte_perm(lo01, lo23, 0x5410);  // level 4: weight 2^0
                lev[g][2] = __byte_perm(lo01, lo23, 0x7632);  // level 3
                lev[g][1] = __byte_perm(hi01, hi23, 0x5410);  // level 2
                lev[g][0] = __byte_perm(hi01, hi23, 0x7632);  // level 1: weight 2^24
                const bool k0 = (((uint64_t)abs_bits(x.x) << 32) | lo_key) >= t01.x;
                const bool k1 = (((uint64_t)abs_bits(x.y) << 32) | lo_key) >= t01.y;
                const bool k2 = (((uint64_t)abs_bits(x.z) << 32) | lo_key) >= t23.x;
                const bool k3 = (((uint64_t)abs_bits(x.w) << 32) | lo_key) >= t23.y;
                km[g] = (k0 ? 0xFFu : 0u) | (k1 ? 0xFF00u : 0u) | (k2 ? 0xFF0000u : 0u) | (k3 ? 0xFF000000u : 0u);  // & zero_row below
                if (want_rss) {
                    const float4 wo = *reinterpret_cast<const float4*>(&it_d.wold[c0]);  // in registers too: spills
                    pdot = fmaf(x.x, wo.x, pdot);
                    pdot = fmaf(x.y, wo.y, pdot);
                    pdot = fmaf(x.z, wo.z, pdot);
                    pdot = fmaf(x.w, wo.w, pdot);
                }
            }
            float yv = 0.f;
            uint32_t zy = 0x80808080u;
            if (fql == 0) {
                yv = krow ? lds_f32(ring_val + (uint32_t)(j % kTcRing) * (kTcKC * 4)) : 0.f;
                const float ty = yv * sc_y;
                amax = fmaxf(amax, fabsf(ty));
                zy = (uint32_t)__float2int_rn(ty) + 0x80808080u;
            }
            // the row's exception flag and dot over its lanes
            const bool exc = ((__ballot_sync(CALS_FULL_MASK, amax >= kTcLimit) >> (kTcLPR * kl)) & ((1u << kTcLPR) - 1u)) != 0u;
            if (want_rss) {
#pragma unroll
                for (int o = 1; o < kTcLPR; o <<= 1) pdot += __shfl_xor_sync(CALS_FULL_MASK, pdot, o);
                if (fql == 0 && krow) {
                    const double dd = (double)yv - (double)pdot;
                    racc = fma(dd, dd, racc);
                }
            }
            const uint32_t zero_row = exc ? 0u : row_on;
            TC_TRACE(j * 8 + 2, warp == 0 && lane == 0 && j < 4096);
            if (j >= 2) {
                if (dbg & 32) mbar_wait_hint((full_base + 8u * (uint32_t)(3 * kTcItems + 2 + (db))), (uint32_t)(((j - 2) >> 1) & 1));
                else mbar_wait((full_base + 8u * (uint32_t)(3 * kTcItems + 2 + (db))), (uint32_t)(((j - 2) >> 1) & 1));
            }
            TC_TRACE(j * 8 + 3, warp == 0 && lane == 0 && j < 4096);
            const uint32_t dbase = dig_lane + (uint32_t)db * kTcDigitBuf;
            uint32_t kmz[kTcNG];
#pragma unroll
            for (int g = 0; g < kTcNG; ++g) kmz[g] = km[g] & zero_row;
#pragma unroll
            for (int g = 0; g < ((dbg & 4) ? 0 : kTcNG); ++g) {
#pragma unroll
                for (int L = 1; L <= 4; ++L) {
                    // un-bias (^ 0x80 per byte) and mask in one LOP3 per stored word
                    const uint32_t w = (lev[g][L - 1] ^ 0x80808080u) & zero_row;
                    const uint32_t pair = (uint32_t)((L - 1) >> 1), half = (uint32_t)((L - 1) & 1);
                    const uint32_t gofs = 128u * kTcLPR * (uint32_t)g;  // 4 kLPR columns further
                    sts_u32(dbase + 2 * kTcATile + pair * kTcBTile + (half ? off_b1 : off_b0) + gofs, w);
                    sts_u32(dbase + pair * kTcATile + (half ? off_a1 : off_a0) + gofs,
                            (lev[g][L - 1] ^ 0x80808080u) & kmz[g]);
                }
            }
            if (fql == 0) {
                // the rating's digits (level L = byte 4 - L), one byte per level word (the rest is padding)
#pragma unroll
                for (int L = 1; L <= 4; ++L) {
                    const uint32_t pair = (uint32_t)((L - 1) >> 1), half = (uint32_t)((L - 1) & 1);
                    const uint32_t yb = ((zy >> (8 * (4 - L))) & 0xFFu) ^ 0x80u;
                    sts_u32(dbase + 2 * kTcATile + pair * kTcBTile + (half ? off_y1 : off_y0), yb & zero_row);
                }
                if (exc && krow) {
                    atomicOr(&exc_mask[((c.i % kTcExcSlots) * kTcMaxChunks + ci) * 2 + (krel >> 5)], 1u << (krel & 31));
                    exc_any[c.i % kTcExcSlots] = 1u;
                }
            }
            tc::fence_smem_async();
            __syncwarp();
                        if (lane == 0) mbar_arrive((full_base + 8u * (uint32_t)(3 * kTcItems + (db))));
            if (last) {
                // per-warp residual partial, then this warp is done with the item
                double v = racc;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CALS_FULL_MASK, v, o);
                if (lane == 0) rss_part[sl * kTcCW + warp] = v;
                racc = 0.0;
                __syncwarp();
                if (lane == 0) mbar_arrive((full_base + 8u * (uint32_t)(2 * kTcItems + (sl))));
            }
            tc_advance(c, items, full_base);
        }
        cp_async_wait<0>();
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tmem);
    if ((dbg & 8) && blockIdx.x == 0 && tid == 0 && A.stats != nullptr) A.stats[49150] += 1ull;
}

}  // namespace cals
