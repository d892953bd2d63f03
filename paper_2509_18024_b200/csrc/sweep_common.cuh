// sweep_common.cuh -- pieces shared by the half-sweep kernels.
#pragma once
#include "common.cuh"

namespace cals {

#define CALS_MAX_NF_DEV 128
#define CALS_MAX_WARPS 16
constexpr int kThreads = 256;       // max threads per sweep CTA (launch bound)
constexpr int kCap = 256;           // per-column candidate capacity (shared-memory tier)
constexpr int kQ = 256;             // quantile-table resolution (levels per column)
constexpr int kSub = 8;             // sub-buckets used to pre-narrow a bracket
constexpr uint32_t kAbsInf = 0x80000000u;  // sentinel above every abs_bits value

struct SweepArgs {
    const int64_t* ptr;
    const int32_t* idx;
    const float* val;
    int64_t nnz;
    const int32_t* budget;
    const float* src;
    int64_t n_src;
    int ld_src;   // multiple of 4 (16-byte rows for cp.async gathers)
    int nf;
    float* tgt;            // solved rows (the new target matrix)
    int ld_tgt;
    const float* tgt_old;  // previous-iteration rows for the fused residual (nullable)
    int ld_old;
    double lam;
    double* rss_rows;      // residual of tgt_old rows per regression (nullable)
    double* pen_rows;      // n_i * |w_i|^2 of the new rows (nullable)
    uint64_t* thr_keys;    // nullable
    int32_t* status;
    const uint32_t* qtab;  // [nf][kQ+1] abs-bit quantiles of the source, or null
    float delta_tab;       // quantile-table sampling margin (rank units)
    unsigned long long* summary;  // nullable: max over rows of (status << 32 | ~row)
    double* gbuf;                 // normal equations of the current batch: [slot][nf][nf+1], float64
                                  // (the fp32 solve rounds them; the float64 refinement needs them exact)
    unsigned long long* stats;    // nullable debug counters (cals_debug_stats)
    int* rf_cnt;                  // rows deferred to the float64 refinement (sweep_refine.cu) that
    int64_t* rf_list;             // need their stored normal equations: (row << 32 | slot), per batch
    int* rs_cnt;                  // rows deferred that rebuild their Gram from the slice: refined once
    int32_t* rs_list;             // after the tier's last batch (one launch, no per-batch latency)
    int rf_slice_max;             // rows up to this length rebuild from the slice (0: none)
    int* ir_cnt;                  // 32 < n_f <= 64: systems the fp32 solve hands to the mixed-precision
    int64_t* ir_list;             // solve (sweep_solve_ir.cu), (row << 32 | slot), per batch
    float ill_ratio;              // pivot-magnitude spread that defers a system (ill_ratio_for)
};

// Hand a system the fp32 solve cannot hold to the float64 refinement.
__device__ __forceinline__ void defer_refine(const SweepArgs& A, int row, int64_t slot) {
    const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
    if (n <= A.rf_slice_max) {
        A.rs_list[atomicAdd(A.rs_cnt, 1)] = row;
    } else {
        const int at = atomicAdd(A.rf_cnt, 1);
        A.rf_list[at] = ((int64_t)row << 32) | (int64_t)(uint32_t)slot;
    }
}

// 32 < n_f <= 64: an ill-conditioned system first goes to the fp32 LU + float64 iterative
// refinement (which defers to the float64 elimination what it cannot hold).
__device__ __forceinline__ void defer_ir(const SweepArgs& A, int row, int64_t slot) {
    A.ir_list[atomicAdd(A.ir_cnt, 1)] = ((int64_t)row << 32) | (int64_t)(uint32_t)slot;
}

// Debug counters (only when A.stats != nullptr): see cals_debug_stats.
enum StatId { kStColumns = 0, kStFallback, kStCandidates, kStAfterPrenarrow, kStSelectRounds, kStRows,
              kStBigColumns, kStBigFallback, kStSmallOver, kStSmallMiss, kStFinalOver, kStBigMissAbove,
              kStBigMissBelow, kStBigOverflow, kStBigFallbackN, kStRefined, kStCount = 16 };
__device__ __forceinline__ void stat_add(const SweepArgs& A, int id, unsigned long long v) {
    if (A.stats != nullptr) atomicAdd(A.stats + id, v);
}

__device__ __forceinline__ void report_status(const SweepArgs& A, int row, int st) {
    if (st != 0 && A.summary != nullptr)
        atomicMax(A.summary, ((unsigned long long)st << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)row));
}

// Work description of the tiled (big-row) tier.
struct BigArgs {
    const int32_t* rows;      // [n_big] row ids
    const int64_t* tile_ptr;  // [n_big + 1] item prefix per row
    const int64_t* cand_ptr;  // [n_big + 1] candidate key offsets (nf equal column regions)
    int64_t n_big;            // rows of this batch
    int64_t n_multi;          // rows [0, n_multi) span >= 2 work items (partials + big_reduce); the
                              // rest write their normal equations straight into gbuf slot r
    int64_t n_tiles;          // work items of this batch
    int64_t tile_base;        // absolute index of the batch's first work item
    int64_t cand_base;        // absolute offset of the batch's first candidate key
    int item_rows;            // slice rows per work item
    int chunk;                // slice rows staged per shared-memory chunk
    int* cnt;                 // [n_big][nf][2]  (above, in)
    uint64_t* cand;           // [cand_total]
    uint64_t* thr;            // [n_big][nf]
    double* part;             // [n_tiles][nf][nf+1] float64 partial normal equations
    float* wbig;              // [n_big][nf]
    double* rss_part;         // [n_tiles]
    int* hist;                // [n_big][nf][kHB] in-bracket counts per sub-bucket
    const uint32_t* brk;      // [n_big][nf] calibrated levels jhi | jlo << 16, or ~0u (use the table margin)
    const int32_t* tile_row;  // nullable: absolute big row of each absolute work item
    int64_t row_base;         // absolute index of the batch's first big row
    // method 'fast_core' (big_gram_kernel<CPL, true>): kept bits come from one sketch of
    // the whole source instead of per-row thresholds
    const uint32_t* gmask;    // [n_src][gwords] bit c%32 of word c/32: source row kept for column c
    int gwords;
    int fold_chunks;          // big_gram: chunks summed in fp32 before a float64 fold (0: kFoldChunks)
    int calib_samples;        // tuning overrides (0: defaults kCalibSamples / kCalibZ)
    float calib_z;
    int* fcnt;                // [n_big][nf] kept slice rows per column (multi-item rows)
    unsigned long long* famax;  // [n_big][nf] max key (abs_bits << 32 | ~k) per column (fallback row)
    int* item_ctr;            // big_gram_tc / big_scan2: next unclaimed work item (zeroed before the launch)
    int* icnt;                // [n_tiles][nf] in-bracket keys of each work item (big_scan2): a multi-item
                              // row's column region is split into equal per-item sub-regions
};

// Candidate sub-region of work item t_local (0-based within its row) of a row with
// n_items items, in a column region of capB keys.
__host__ __device__ inline int cand_item_cap(int capB, int n_items) { return capB / max(n_items, 1); }

constexpr int kHB = 32;  // sub-buckets of a big row's bracket (linear in abs-bit space)

// Sub-buckets of a bracket [lob, hib) are power-of-two wide: width 2^sh with
// sh the smallest shift mapping span - 1 below kHB (so 16..32 buckets are used).
__device__ __forceinline__ int hb_shift(uint32_t span) {
    const int bits = span > 1 ? 32 - __clz((int)(span - 1)) : 0;
    return bits > 5 ? bits - 5 : 0;  // kHB == 32
}
// Sub-bucket of an in-bracket abs value a.
__device__ __forceinline__ int hb_bucket(uint32_t a, uint32_t lob, int sh) { return (int)((a - lob) >> sh); }
// Key range [lo, hi) of sub-bucket b (hi capped at the bracket's top key).
__device__ __forceinline__ uint64_t hb_lower_key(int b, uint32_t lob, int sh) {
    return ((uint64_t)lob + ((uint64_t)b << sh)) << 32;
}

__host__ __device__ inline int round_up4(int x) { return (x + 3) & ~3; }
// Staged row stride (floats): 16-byte aligned rows for cp.async / LDS.128,
// padded so that consecutive rows start in different bank groups.
__host__ __device__ inline int xs_stride(int nf) {
    const int r = round_up4(nf);
    return (r % 8 == 0) ? r + 4 : r;
}
__host__ __device__ inline int xs_chunks(int nf) { return (nf + 3) >> 2; }  // 16-byte chunks holding data
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// Table levels [jhi, jlo] around the target rank of a row:
// keys with abs_bits >= qtab[jhi] are "above", the bracket is
// [qtab[jlo], qtab[jhi]).  Margin: 3 binomial sigmas + table sampling error.
__device__ __forceinline__ void table_levels(int n, int s, float delta_tab, int& jhi, int& jlo) {
    const float p = (float)s / (float)n;
    // tiled rows get a wider margin: a miss there costs whole-column passes
    const float ks = n > 2048 ? 4.0f : 3.0f, kt = n > 2048 ? 1.5f : 1.0f;
    const float d = ks * sqrtf(p * (1.0f - p) / (float)n) + kt * delta_tab + 0.5f / (float)kQ;
    jhi = (int)floorf((p - d) * (float)kQ);
    jlo = (int)ceilf((p + d) * (float)kQ);
    jhi = jhi < 0 ? 0 : (jhi > kQ ? kQ : jhi);
    jlo = jlo < 0 ? 0 : (jlo > kQ ? kQ : jlo);
}

__device__ __forceinline__ void table_bracket(const uint32_t* qtab_c, int n, int s, float delta_tab,
                                              uint32_t& hib, uint32_t& lob) {
    int jhi, jlo;
    table_levels(n, s, delta_tab, jhi, jlo);
    hib = qtab_c[jhi];
    lob = qtab_c[jlo];
}

// Bracket of big row r (batch-relative), column c: the row's own calibrated
// table levels when it has them (big_calib_kernel), else the table margin.
__device__ __forceinline__ void big_bracket(const SweepArgs& A, const BigArgs& B, int r, int c, int n, int s,
                                            uint32_t& hib, uint32_t& lob) {
    const uint32_t* q = A.qtab + (size_t)c * (kQ + 1);
    const uint32_t v = B.brk != nullptr ? B.brk[(size_t)r * A.nf + c] : ~0u;
    if (v != ~0u) {
        hib = q[v & 0xFFFFu];
        lob = q[v >> 16];
    } else {
        table_bracket(q, n, s, A.delta_tab, hib, lob);
    }
}

__device__ __forceinline__ uint64_t hi_key_of(uint32_t hib) {
    return hib >= kAbsInf ? ~0ull : ((uint64_t)hib << 32);
}

// cp.async 16-byte global -> shared copy (L2-only caching: gathers are streamed)
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
}

// Stage slice rows [k0, k0 + kn) of the regression whose ratings start at
// `lo`: X rows (16-byte chunks, cp.async) into Xs (stride sx) and y into ys.
// The caller synchronises the block afterwards.
__device__ __forceinline__ void stage_slice(const SweepArgs& A, int64_t lo, int k0, int kn, float* Xs, float* ys,
                                            const FastDiv& fq) {
    const int sx = xs_stride(A.nf), nq = xs_chunks(A.nf);
    const int nt = blockDim.x;
    const int nel = kn * nq;
    const uint32_t xs_base = smem_u32(Xs);
    const int32_t* idx = A.idx + lo + k0;
    const float* src = A.src;
    const int64_t ld = A.ld_src;
#pragma unroll 4
    for (int e = threadIdx.x; e < nel; e += nt) {
        const int k = (int)fq.div((uint32_t)e);
        const int q = e - k * nq;
        const int64_t r = __ldg(idx + k);
        cp_async16(xs_base + (uint32_t)((k * sx + 4 * q) * 4), src + r * ld + 4 * q);
    }
    if (ys != nullptr)
        for (int k = threadIdx.x; k < kn; k += nt) ys[k] = __ldg(A.val + lo + k0 + k);
    cp_async_wait_all();
}

__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Asynchronous variant for double-buffered chunk loops: issue the copies of
// slice rows [k0, k0 + kn) (X into xs_base, y into ys_base unless 0) as one
// cp.async group and return; the caller waits with cp_async_wait<N>() and
// synchronises the block before reading.
__device__ __forceinline__ void stage_slice_issue(const SweepArgs& A, int64_t lo, int k0, int kn, uint32_t xs_base,
                                                  uint32_t ys_base, const FastDiv& fq) {
    const int sx = xs_stride(A.nf), nq = xs_chunks(A.nf);
    const int nt = blockDim.x;
    const int nel = kn * nq;
    const int32_t* idx = A.idx + lo + k0;
    const float* src = A.src;
    const int64_t ld = A.ld_src;
#pragma unroll 4
    for (int e = threadIdx.x; e < nel; e += nt) {
        const int k = (int)fq.div((uint32_t)e);
        const int q = e - k * nq;
        const int64_t r = __ldg(idx + k);
        cp_async16(xs_base + (uint32_t)((k * sx + 4 * q) * 4), src + r * ld + 4 * q);
    }
    if (ys_base != 0u)
        for (int k = threadIdx.x; k < kn; k += nt) cp_async4(ys_base + 4u * (uint32_t)k, A.val + lo + k0 + k);
    cp_async_commit();
}

// ---- 1-D bulk (TMA) staging of gathered rows ----------------------------------
// One cp.async.bulk per slice row (its 16*nq data bytes), all completing on one
// mbarrier: warp 0 issues, every thread waits on the barrier's phase.
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mbar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
// waiter for role warps that wait long (a whole work item): polls with a short sleep in
// between so its spinning does not take issue slots from the warps doing the work
__device__ __forceinline__ bool mbar_test(uint32_t mbar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(mbar), "r"(phase)
        : "memory");
    return ok != 0u;
}
// try_wait with a suspend-time hint: the thread may be suspended until the phase completes
__device__ __forceinline__ void mbar_wait_hint(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            mbar),
        "r"(phase), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_backoff(uint32_t mbar, uint32_t phase) {
    while (!mbar_test(mbar, phase)) __nanosleep(128);
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            mbar),
        "r"(phase)
        : "memory");
}

// Stage slice rows [k0, k0 + kn) like stage_slice, X by bulk copies (warp 0
// issues one per row) and y by plain loads; returns after the copies landed.
// `phase` is the barrier's current parity (flipped here).  The caller
// synchronises the block before (buffer free) and after (y visible).
__device__ __forceinline__ void stage_slice_bulk(const SweepArgs& A, int64_t lo, int k0, int kn, uint32_t xs_base,
                                                 float* ys, uint32_t mbar, uint32_t& phase) {
    const int sx = xs_stride(A.nf);
    const uint32_t rowbytes = 16u * (uint32_t)xs_chunks(A.nf);
    // every thread issues the copies of its rows; the barrier's single arrival (thread 0,
    // with the expected byte count) may come before or after them: the phase cannot
    // complete while that arrival is pending
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // prior generic reads of the buffer
    if (threadIdx.x == 0) mbar_expect_tx(mbar, (uint32_t)kn * rowbytes);
    const int32_t* idx = A.idx + lo + k0;
    for (int k = threadIdx.x; k < kn; k += blockDim.x)
        bulk_g2s(xs_base + (uint32_t)(k * sx * 4), A.src + (int64_t)__ldg(idx + k) * A.ld_src, rowbytes, mbar);
    if (ys != nullptr)
        for (int k = threadIdx.x; k < kn; k += blockDim.x) ys[k] = __ldg(A.val + lo + k0 + k);
    mbar_wait(mbar, phase);
    phase ^= 1u;
}

// Column lanes / slots of the staged-slice kernel: thread t handles column
// t % NFP over the k-range of slot t / NFP (ranges are multiples of 32 rows,
// so every bitmap word has a single owner).
struct SlotMap {
    int NFP, P;
    __host__ __device__ SlotMap(int nf, int threads) {
        if (nf <= 32) {
            NFP = 1;
            while (NFP < nf) NFP <<= 1;
        } else {
            NFP = (nf + 31) / 32 * 32;
        }
        P = threads / NFP;
        if (P < 1) P = 1;
    }
    __host__ __device__ int chunk(int n) const { return ((n + P - 1) / P + 31) / 32 * 32; }
    __host__ __device__ int caps(int chunk_rows) const {
        const int c = 16 + chunk_rows / 4;
        return c < chunk_rows ? c : chunk_rows;
    }
};

constexpr int kFinalCap = 64;  // per-column candidates of the chosen sub-bucket

// Shared-memory footprint of the staged-slice kernel for rows of length <= N
// whose sketch budget is <= S:
//   Xs [N][sx] | ys [N] | bitmap [nf][ceil(N/32)] (column-major) | lists [nf][S] |
//   slot candidates [P][CAPS][NFP] u16 | slot level counts [P][8][NFP] u8 |
//   slot above/in counts [P][NFP] 2 x u16 | final buffers [nf][kFinalCap] u16 |
//   per-warp key scratch [kFinalCap] u64
struct T1Layout {
    size_t xs, ys, mb, lists, cand, lvl, cnts, fb, scr, total;
    int sx, nw, caps;
    __host__ __device__ T1Layout(int N, int S, int nf, int threads) {
        const SlotMap M(nf, threads);
        sx = xs_stride(nf);
        nw = (N + 31) / 32;
        caps = M.caps(M.chunk(N));
        const int warps = threads / 32;
        xs = align16((size_t)N * sx * sizeof(float));
        ys = align16((size_t)N * sizeof(float));
        mb = align16((size_t)nf * nw * sizeof(uint32_t));
        lists = align16((size_t)nf * (S > 0 ? S : 1) * sizeof(uint16_t));
        cand = align16((size_t)M.P * caps * M.NFP * sizeof(uint16_t));
        lvl = align16((size_t)M.P * 8 * M.NFP);
        cnts = align16((size_t)M.P * M.NFP * 2 * sizeof(uint16_t));
        fb = align16((size_t)nf * kFinalCap * sizeof(uint16_t));
        scr = align16((size_t)warps * kFinalCap * sizeof(uint64_t));
        total = xs + ys + mb + lists + cand + lvl + cnts + fb + scr;
    }
};

}  // namespace cals
