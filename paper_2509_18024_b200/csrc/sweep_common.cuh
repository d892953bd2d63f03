// sweep_common.cuh -- pieces shared by the half-sweep kernels.
#pragma once
#include "common.cuh"

namespace cals {

#define CALS_MAX_NF_DEV 128
constexpr int kThreads = 256;       // threads per sweep CTA
constexpr int kCap = 256;           // per-column candidate capacity (shared-memory tier)
constexpr int kQ = 256;             // quantile-table resolution (levels per column)
constexpr uint32_t kAbsInf = 0x80000000u;  // sentinel above every abs_bits value

struct SweepArgs {
    const int64_t* ptr;
    const int32_t* idx;
    const float* val;
    const int32_t* budget;
    const float* src;
    int64_t n_src;
    int ld_src;
    int nf;
    float* tgt;
    int ld_tgt;
    double lam;
    double* rss_rows;      // nullable
    uint64_t* thr_keys;    // nullable
    int32_t* status;
    const uint32_t* qtab;  // [nf][kQ+1] abs-bit quantiles of the source, or null
    float delta_tab;       // quantile-table sampling margin (rank units)
    unsigned long long* summary;  // nullable: max over rows of (status << 32 | ~row)
    double* retry_ws;             // per-CTA float64 jitter-retry scratch (retry_stride doubles each)
    int retry_stride;
};

__device__ __forceinline__ void report_status(const SweepArgs& A, int row, int st) {
    if (st != 0 && A.summary != nullptr)
        atomicMax(A.summary, ((unsigned long long)st << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)row));
}

// Work description of the tiled (big-row) tier.
struct BigArgs {
    const int32_t* rows;      // [n_big] row ids
    const int64_t* tile_ptr;  // [n_big + 1] item prefix per row
    const int64_t* cand_ptr;  // [n_big + 1] candidate key offsets (nf equal column regions)
    int64_t n_big;
    int64_t n_tiles;
    int item_rows;            // slice rows per work item
    int chunk;                // slice rows staged per shared-memory chunk
    int* cnt;                 // [n_big][nf][2]  (above, in)
    uint64_t* cand;           // [cand_total]
    uint64_t* thr;            // [n_big][nf]
    float* part;              // [n_tiles][nf][nf+1]
    float* wbig;              // [n_big][nf]
    double* rss_part;         // [n_tiles]
};

__host__ __device__ inline int round_up4(int x) { return (x + 3) & ~3; }
__host__ __device__ inline int xs_stride(int nf) { return round_up4(nf + 1); }  // X | y | pad
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// Bracket [lob, hib) in abs-bit space around the target rank of a row,
// read from the column's quantile table.  Keys >= (hib << 32) are "above".
__device__ __forceinline__ void table_bracket(const uint32_t* qtab_c, int n, int s, float delta_tab,
                                              uint32_t& hib, uint32_t& lob) {
    float p = (float)s / (float)n;
    float d = 3.0f * sqrtf(p * (1.0f - p) / (float)n) + delta_tab + 0.5f / (float)kQ;
    int jhi = (int)floorf((p - d) * (float)kQ);
    int jlo = (int)ceilf((p + d) * (float)kQ);
    jhi = jhi < 0 ? 0 : (jhi > kQ ? kQ : jhi);
    jlo = jlo < 0 ? 0 : (jlo > kQ ? kQ : jlo);
    hib = qtab_c[jhi];
    lob = qtab_c[jlo];
}

__device__ __forceinline__ uint64_t hi_key_of(uint32_t hib) {
    return hib >= kAbsInf ? ~0ull : ((uint64_t)hib << 32);
}

// Shared-memory footprint of the staged-slice kernel for rows of length <= N.
struct T1Layout {
    size_t xs, cand, mb, g, w, scratch, region, total;
    int sx, mw;
    __host__ __device__ T1Layout(int N, int nf, int threads) {
        sx = xs_stride(nf);
        mw = (nf + 31) / 32;
        xs = align16((size_t)N * sx * sizeof(float));
        cand = align16((size_t)nf * kCap * sizeof(uint16_t));
        mb = align16((size_t)N * mw * sizeof(uint32_t));
        g = align16((size_t)nf * (nf + 1) * sizeof(float));
        w = nf > 32 ? g : 0;
        scratch = align16((size_t)threads * 16 * sizeof(float));
        size_t after = mb + g + w + scratch;
        region = cand > after ? cand : after;
        total = xs + region;
    }
};

}  // namespace cals

