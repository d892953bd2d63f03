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
// fp32 products give ~2e-4, tools/ozaki_emul.py).
//
// Pipeline per CTA (one per SM, 16 warps): a 4-deep ring of fp32 slice chunks
// (64 rows, one cp.async.bulk per gathered row, mbarrier completion) feeds a
// digit pass (all warps: kept bits from the selection thresholds, digits,
// masked copies -> two double-buffered K-step tile sets in shared memory), and
// thread 0 issues the chunk's MMAs and commits them to that tile set's
// mbarrier, so the tensor cores run one chunk behind the digit pass.
#include "sweep_common.cuh"
#include "tc.cuh"

namespace cals {

constexpr int kTcCW = 8;                      // compute warps: 8 whole slice rows each per chunk
constexpr int kTcThreads = (kTcCW + 1) * 32;  // + the control warp (bulk-copy producer, MMA issue)
constexpr int kTcKC = 64;                     // slice rows per chunk (two K-steps of 32)
constexpr int kTcStages = 4;                  // fp32 staging ring depth
constexpr int kTcSX = 80;                     // staged row stride in floats (320 B: conflict-free float4 reads)
constexpr int kTcN = 144;                     // N side: two levels x (64 factor columns + y + 7 zero pad)
constexpr int kTcLvl = 72;                    // N columns per level
constexpr int kTcATile = 4096;                // M = 128 (two levels x 64 columns) x 32 K bytes
constexpr int kTcBTile = 4608;                // N = 144 x 32 K bytes
constexpr int kTcKStepBytes = 2 * kTcATile + 2 * kTcBTile;  // A12 A34 B12 B34
constexpr int kTcDigitBuf = 2 * kTcKStepBytes;              // one chunk (two K-steps)
constexpr int kTcAccB = 256;                  // TMEM column of the second accumulator (levels 4..6)
constexpr int kTcSlots = 4;                   // work items in flight (finalize lags <= 2 chunks)
constexpr int kTcMaxChunks = 256;             // chunks per work item (item_rows <= 16384)
constexpr int kTcExcBatch = 64;               // exception rows staged per finalize round (one chunk)
constexpr float kTcLimit = 2.13e9f;           // |x * 2^32 / alpha| below this keeps the top digit in int8

struct TcMeta {             // per staged chunk: its work item's thresholds and previous rows
    uint64_t T[64];
    float wold[64];
};

struct TcSmem {
    static constexpr int stage_x = 0;                                          // [4][64][kTcSX] f32
    static constexpr int stage_y = stage_x + kTcStages * kTcKC * kTcSX * 4;     // [4][64] f32
    static constexpr int meta = stage_y + kTcStages * kTcKC * 4;               // [4] TcMeta
    static constexpr int digits = (meta + kTcStages * (int)sizeof(TcMeta) + 1023) & ~1023;  // [2] tile sets
    static constexpr int xchg = digits + 2 * kTcDigitBuf;                      // [64][72] f64
    static constexpr int exc_x = xchg + 64 * kTcLvl * 8;                       // [32][72] f32 (+ y, k)
    static constexpr int exc_mask = exc_x + kTcExcBatch * kTcLvl * 4;          // [slots][256] u64
    static constexpr int rss = exc_mask + kTcSlots * kTcMaxChunks * 8;         // [slots][kTcCW] f64
    static constexpr int fin_T = rss + kTcSlots * kTcCW * 8;                   // [slots][64] u64
    static constexpr int total = fin_T + kTcSlots * 64 * 8;
};

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

struct TcCursor {
    int64_t t;   // work item index (batch-relative); >= n_tiles when done
    int k0;      // first slice row of the chunk
    int kbeg, kend;
    int r, row;  // batch row, row id
    int64_t lo;  // first rating of the row
    int n;
};

__device__ __forceinline__ void tc_cursor_item(const SweepArgs& A, const BigArgs& B, TcCursor& c) {
    if (c.t >= B.n_tiles) return;
    const int64_t T_abs = B.tile_base + c.t;
    int r;
    if (B.tile_row != nullptr) {
        r = (int)(__ldg(B.tile_row + T_abs) - B.row_base);
    } else {
        int64_t lo = 0, hi = B.n_big - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (B.tile_ptr[mid] <= T_abs) lo = mid; else hi = mid - 1;
        }
        r = (int)lo;
    }
    c.r = r;
    c.row = B.rows[r];
    c.lo = A.ptr[c.row];
    c.n = (int)(A.ptr[c.row + 1] - c.lo);
    c.kbeg = (int)(T_abs - B.tile_ptr[r]) * B.item_rows;
    c.kend = min(c.n, c.kbeg + B.item_rows);
    c.k0 = c.kbeg;
}

__device__ __forceinline__ void tc_cursor_next(const SweepArgs& A, const BigArgs& B, TcCursor& c) {
    c.k0 += kTcKC;
    if (c.k0 >= c.kend) {
        c.t += gridDim.x;
        tc_cursor_item(A, B, c);
    }
}

__global__ void __launch_bounds__(kTcThreads, 1) big_gram_tc_kernel(SweepArgs A, BigArgs B,
                                                                    const float* __restrict__ g_scale,
                                                                    const double* __restrict__ g_alpha) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ float s_scale[65];
    __shared__ double s_alpha[65];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long bar_full_st[kTcStages], bar_empty_st[kTcStages];
    __shared__ __align__(8) unsigned long long bar_full_tl[2], bar_empty_tl[2];
    __shared__ __align__(8) unsigned long long bar_tmem_full, bar_tmem_empty, bar_item[kTcSlots];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nf = A.nf, gs = nf + 1;
    const bool want_rss = A.rss_rows != nullptr;
    const uint32_t sbase = tc::smem_addr(smem);
    unsigned char* digits = smem + TcSmem::digits;
    double* xchg = reinterpret_cast<double*>(smem + TcSmem::xchg);
    float* exc_x = reinterpret_cast<float*>(smem + TcSmem::exc_x);
    uint32_t* exc_mask = reinterpret_cast<uint32_t*>(smem + TcSmem::exc_mask);  // [slot][chunk][2]
    double* rss_part = reinterpret_cast<double*>(smem + TcSmem::rss);
    uint64_t* fin_T = reinterpret_cast<uint64_t*>(smem + TcSmem::fin_T);

    // ---- setup (every thread), then the roles never meet at a block barrier again
    for (int e = tid; e < 2 * kTcDigitBuf / 16; e += blockDim.x)
        reinterpret_cast<uint4*>(digits)[e] = make_uint4(0u, 0u, 0u, 0u);  // padding bytes stay zero
    for (int e = tid; e < kTcSlots * kTcMaxChunks * 2; e += blockDim.x) exc_mask[e] = 0u;
    if (tid < 65) {
        s_scale[tid] = g_scale[tid];
        s_alpha[tid] = g_alpha[tid];
    }
    if (warp == 0) tc::tmem_alloc<512>(&s_tmem);
    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(smem_u32(&bar_full_st[s]), 1);
            mbar_init(smem_u32(&bar_empty_st[s]), kTcCW);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&bar_full_tl[s]), kTcCW);
            mbar_init(smem_u32(&bar_empty_tl[s]), 1);
        }
        mbar_init(smem_u32(&bar_tmem_full), 1);
        mbar_init(smem_u32(&bar_tmem_empty), 1);
        for (int s = 0; s < kTcSlots; ++s) mbar_init(smem_u32(&bar_item[s]), kTcCW);
    }
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == kTcCW) {
        // ================= control warp: producer of the staging ring + MMA issue =================
        const uint32_t idesc = tc::idesc_i8(128, kTcN) | (1u << 15) | (1u << 16);  // MN-major A and B
        const uint32_t rowbytes = 16u * (uint32_t)xs_chunks(nf);
        TcCursor p{}, m{};
        p.t = m.t = blockIdx.x;
        tc_cursor_item(A, B, p);
        m = p;
        int64_t jp = 0, jm = 0, item = 0;
        bool m_first = true;
        while (m.t < B.n_tiles) {
            // produce up to kTcStages chunks ahead of the MMAs
            while (p.t < B.n_tiles && jp < jm + kTcStages) {
                const int s = (int)(jp % kTcStages);
                if (jp >= kTcStages) mbar_wait(smem_u32(&bar_empty_st[s]), (uint32_t)((jp / kTcStages - 1) & 1));
                const int kn = min(kTcKC, p.kend - p.k0);
                TcMeta* meta = reinterpret_cast<TcMeta*>(smem + TcSmem::meta) + s;
                float* ys = reinterpret_cast<float*>(smem + TcSmem::stage_y) + s * kTcKC;
                for (int c = lane; c < 64; c += 32) {
                    meta->T[c] = c < nf ? B.thr[(size_t)p.r * nf + c] : ~0ull;
                    meta->wold[c] = (want_rss && c < nf) ? A.tgt_old[(int64_t)p.row * A.ld_old + c] : 0.f;
                }
                for (int k = lane; k < kTcKC; k += 32) ys[k] = k < kn ? __ldg(A.val + p.lo + p.k0 + k) : 0.f;
                __syncwarp();
                const uint32_t fb = smem_u32(&bar_full_st[s]);
                if (lane == 0) mbar_expect_tx(fb, (uint32_t)kn * rowbytes);
                const uint32_t sx = sbase + TcSmem::stage_x + (uint32_t)s * (kTcKC * kTcSX * 4u);
                for (int k = lane; k < kn; k += 32)
                    bulk_g2s(sx + (uint32_t)k * (kTcSX * 4u),
                             A.src + (int64_t)__ldg(A.idx + p.lo + p.k0 + k) * A.ld_src, rowbytes, fb);
                tc_cursor_next(A, B, p);
                ++jp;
            }
            // MMAs of chunk jm
            const int db = (int)(jm & 1);
            const int kn = min(kTcKC, m.kend - m.k0);
            const bool last = m.k0 + kTcKC >= m.kend;
            if (lane == 0) {
                mbar_wait(smem_u32(&bar_full_tl[db]), (uint32_t)((jm >> 1) & 1));
                if (m_first && item > 0) mbar_wait(smem_u32(&bar_tmem_empty), (uint32_t)((item - 1) & 1));
                tc::fence_after();
                const int nks = (kn + 31) >> 5;
                for (int ks = 0; ks < nks; ++ks) {
                    const uint32_t base = sbase + TcSmem::digits + (uint32_t)(db * kTcDigitBuf + ks * kTcKStepBytes);
                    const uint64_t a12 = tc::sdesc(base, 128, 512), a34 = tc::sdesc(base + kTcATile, 128, 512);
                    const uint64_t b12 = tc::sdesc(base + 2 * kTcATile, 128, 512);
                    const uint64_t b34 = tc::sdesc(base + 2 * kTcATile + kTcBTile, 128, 512);
                    const uint32_t acc = (m_first && ks == 0) ? 0u : 1u;
                    tc::mma_i8_ss(tmem, a12, b12, idesc, acc);
                    tc::mma_i8_ss(tmem + kTcAccB, a12, b34, idesc, acc);
                    tc::mma_i8_ss(tmem + kTcAccB, a34, b12, idesc, 1u);
                }
                tc::commit(smem_u32(&bar_empty_tl[db]));
                if (last) tc::commit(smem_u32(&bar_tmem_full));
            }
            __syncwarp();
            if (last) ++item;
            m_first = last;
            tc_cursor_next(A, B, m);
            ++jm;
        }
    } else {
        // ================= compute warps: digits (+ finalize on warps 0..3) =================
        TcCursor c{};
        c.t = blockIdx.x;
        tc_cursor_item(A, B, c);
        const int kl = lane >> 2, fql = lane & 3;
        const int krel = 8 * warp + kl;  // slice row of this lane within the chunk
        int64_t j = 0, item = 0;
        double racc = 0.0;
        while (c.t < B.n_tiles) {
            const int s = (int)(j % kTcStages), db = (int)(j & 1), slot = (int)(item % kTcSlots);
            const int kn = min(kTcKC, c.kend - c.k0);
            const bool last = c.k0 + kTcKC >= c.kend;
            const int ci = (c.k0 - c.kbeg) / kTcKC;
            mbar_wait(smem_u32(&bar_full_st[s]), (uint32_t)((j / kTcStages) & 1));
            if (j >= 2) mbar_wait(smem_u32(&bar_empty_tl[db]), (uint32_t)(((j - 2) >> 1) & 1));
            const float* Xs = reinterpret_cast<const float*>(smem + TcSmem::stage_x) + s * kTcKC * kTcSX;
            const float* ys = reinterpret_cast<const float*>(smem + TcSmem::stage_y) + s * kTcKC;
            const TcMeta* meta = reinterpret_cast<const TcMeta*>(smem + TcSmem::meta) + s;
            const bool krow = krel < kn;
            const uint32_t kg = (uint32_t)(c.k0 + krel);
            // fixed point of the lane's 16 elements, kept bits, exception flag, residual dot
            int X[16];
            uint32_t keepm[4];
            bool exc = false;
            float pdot = 0.f;
#pragma unroll
            for (int it = 0; it < 4; ++it) {
                const int c0 = 4 * (4 * it + fql);
                float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                if (krow && c0 < nf) x = *reinterpret_cast<const float4*>(Xs + krel * kTcSX + c0);
                const float xv[4] = {x.x, x.y, x.z, x.w};
                uint32_t km = 0u;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int cc = c0 + e;
                    const float v = cc < nf ? xv[e] : 0.f;
                    const float t = v * s_scale[cc];
                    exc |= fabsf(t) >= kTcLimit;
                    X[4 * it + e] = __float2int_rn(t);
                    if (want_rss) pdot = fmaf(v, meta->wold[cc], pdot);
                    const uint64_t T = meta->T[cc];
                    const uint32_t a = abs_bits(v), Ta = (uint32_t)(T >> 32), Tk = 0xFFFFFFFFu - (uint32_t)T;
                    const bool keep = krow && cc < nf && (a > Ta || (a == Ta && kg <= Tk));
                    km |= keep ? (0xFFu << (8 * e)) : 0u;
                }
                keepm[it] = km;
            }
            float yv = 0.f;
            int Xy = 0;
            if (fql == 0) {
                yv = krow ? ys[krel] : 0.f;
                const float ty = yv * s_scale[64];
                exc |= fabsf(ty) >= kTcLimit;
                Xy = __float2int_rn(ty);
            }
            // the row's flag and dot over its four lanes
            exc = ((__ballot_sync(CALS_FULL_MASK, exc) >> (4 * kl)) & 0xFu) != 0u;
            if (want_rss) {
                pdot += __shfl_xor_sync(CALS_FULL_MASK, pdot, 1);
                pdot += __shfl_xor_sync(CALS_FULL_MASK, pdot, 2);
                if (fql == 0 && krow) {
                    const double d = (double)yv - (double)pdot;
                    racc = fma(d, d, racc);
                }
            }
            const uint32_t zero_row = exc ? 0u : 0xFFFFFFFFu;
            unsigned char* dbuf = digits + db * kTcDigitBuf + (krel >> 5) * kTcKStepBytes;
            const uint32_t kk = (uint32_t)(krel & 31);
#pragma unroll
            for (int it = 0; it < 4; ++it) {
                const int c0 = 4 * (4 * it + fql);
                uint32_t Y[4][4];  // [element][Y0..Y3]: Y0 = X, Y_{i+1} = (Y_i + 128) >> 8; level L byte = Y[4 - L]
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int x0 = X[4 * it + e];
                    const int y1 = (x0 + 128) >> 8, y2 = (y1 + 128) >> 8, y3 = (y2 + 128) >> 8;
                    Y[e][0] = (uint32_t)x0;
                    Y[e][1] = (uint32_t)y1;
                    Y[e][2] = (uint32_t)y2;
                    Y[e][3] = (uint32_t)y3;
                }
#pragma unroll
                for (int L = 1; L <= 4; ++L) {
                    const uint32_t w = pack4(Y[0][4 - L], Y[1][4 - L], Y[2][4 - L], Y[3][4 - L]) & zero_row;
                    const int pair = (L - 1) >> 1, half = (L - 1) & 1;
                    *reinterpret_cast<uint32_t*>(dbuf + 2 * kTcATile + pair * kTcBTile +
                                                 tc_mn_off((uint32_t)(half * kTcLvl + c0), kk)) = w;
                    *reinterpret_cast<uint32_t*>(dbuf + pair * kTcATile + tc_mn_off((uint32_t)(half * 64 + c0), kk)) =
                        w & keepm[it];
                }
            }
            if (fql == 0) {
                const int y1 = (Xy + 128) >> 8, y2 = (y1 + 128) >> 8, y3 = (y2 + 128) >> 8;
                const uint32_t yl[4] = {(uint32_t)y3, (uint32_t)y2, (uint32_t)y1, (uint32_t)Xy};  // levels 1..4
#pragma unroll
                for (int L = 1; L <= 4; ++L) {
                    const int pair = (L - 1) >> 1, half = (L - 1) & 1;
                    *reinterpret_cast<uint32_t*>(dbuf + 2 * kTcATile + pair * kTcBTile +
                                                 tc_mn_off((uint32_t)(half * kTcLvl + 64), kk)) = yl[L - 1] & 0xFFu & zero_row;
                }
                if (exc && krow) atomicOr(&exc_mask[(slot * kTcMaxChunks + ci) * 2 + (krel >> 5)], 1u << (krel & 31));
            }
            if (last && warp < 4) {
                // the finalize reads the item's thresholds after this stage is recycled
                for (int cc = lane + 32 * warp; cc < 64; cc += 128) fin_T[slot * 64 + cc] = meta->T[cc];
            }
            tc::fence_smem_async();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(smem_u32(&bar_empty_st[s]));
                mbar_arrive(smem_u32(&bar_full_tl[db]));
            }
            if (last) {
                // per-warp residual partial, then this warp is done with the item
                double v = racc;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CALS_FULL_MASK, v, o);
                if (lane == 0) rss_part[slot * kTcCW + warp] = v;
                racc = 0.0;
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bar_item[slot]));
                if (warp < 4) {
                    // ===== finalize (warps 0..3 = the four TMEM lane quarters) =====
                    mbar_wait(smem_u32(&bar_item[slot]), (uint32_t)((item / kTcSlots) & 1));
                    mbar_wait(smem_u32(&bar_tmem_full), (uint32_t)(item & 1));
                    tc::fence_after();
                    const uint32_t lrow = (uint32_t)(32 * warp) << 16;
                    if (warp >= 2) {
                        // second stacked level (ra = 1): weights 2^-8(beta + 1 + rb), beta 2 / 4
                        const int cr = 32 * (warp - 2) + lane;
                        const double wA0 = ldexp(1.0, -24), wA1 = ldexp(1.0, -32), wB0 = ldexp(1.0, -40),
                                     wB1 = ldexp(1.0, -48);
                        for (int f0 = 0; f0 < kTcLvl; f0 += 8) {
                            uint32_t a0[8], a1[8], b0[8], b1[8];
                            tc::ld_32x32b_x8(tmem + lrow + f0, a0);
                            tc::ld_32x32b_x8(tmem + lrow + kTcLvl + f0, a1);
                            tc::ld_32x32b_x8(tmem + lrow + kTcAccB + f0, b0);
                            tc::ld_32x32b_x8(tmem + lrow + kTcAccB + kTcLvl + f0, b1);
                            tc::ld_wait();
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                xchg[cr * kTcLvl + f0 + q] = wA0 * (double)(int)a0[q] + wA1 * (double)(int)a1[q] +
                                                             wB0 * (double)(int)b0[q] + wB1 * (double)(int)b1[q];
                        }
                    }
                    named_bar(1, 128);
                    if (warp < 2) {
                        const int cr = 32 * warp + lane;
                        const double wA0 = ldexp(1.0, -16), wA1 = ldexp(1.0, -24), wB0 = ldexp(1.0, -32),
                                     wB1 = ldexp(1.0, -40);
                        for (int f0 = 0; f0 < kTcLvl; f0 += 8) {
                            uint32_t a0[8], a1[8], b0[8], b1[8];
                            tc::ld_32x32b_x8(tmem + lrow + f0, a0);
                            tc::ld_32x32b_x8(tmem + lrow + kTcLvl + f0, a1);
                            tc::ld_32x32b_x8(tmem + lrow + kTcAccB + f0, b0);
                            tc::ld_32x32b_x8(tmem + lrow + kTcAccB + kTcLvl + f0, b1);
                            tc::ld_wait();
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const int f = f0 + q;
                                const double p = wA0 * (double)(int)a0[q] + wA1 * (double)(int)a1[q] +
                                                 wB0 * (double)(int)b0[q] + wB1 * (double)(int)b1[q];
                                xchg[cr * kTcLvl + f] = s_alpha[cr] * s_alpha[f <= 64 ? f : 64] * (p + xchg[cr * kTcLvl + f]);
                            }
                        }
                    }
                    tc::fence_before();
                    named_bar(1, 128);
                    if (tid == 0) mbar_arrive(smem_u32(&bar_tmem_empty));  // the next item's MMAs may start
                    // exception rows (a value past its column's digit range), chunk by chunk in slice
                    // order: their exact float64 contributions, G[c][:] += x_kc [x_k | y_k] if k is kept for c
                    const int nchunks = (c.kend - c.kbeg + kTcKC - 1) / kTcKC;
                    uint32_t* em = exc_mask + slot * kTcMaxChunks * 2;
                    for (int q = 0; q < nchunks; ++q) {
                        const uint32_t m0 = em[2 * q], m1 = em[2 * q + 1];
                        if ((m0 | m1) == 0u) continue;
                        named_bar(1, 128);  // exc_x free, masks read by every finalize thread
                        if (tid == 0) em[2 * q] = em[2 * q + 1] = 0u;
                        const int n0 = __popc(m0), ne = n0 + __popc(m1);
                        for (int e = tid; e < ne * kTcLvl; e += 128) {
                            const int i = e / kTcLvl, f = e - i * kTcLvl;
                            const uint32_t mm = i < n0 ? m0 : m1;
                            const int bit = (int)__fns(mm, 0, (i < n0 ? i : i - n0) + 1);
                            const int k = c.kbeg + q * kTcKC + (i < n0 ? 0 : 32) + bit;
                            float v = 0.f;
                            if (f < nf) v = __ldg(A.src + (int64_t)__ldg(A.idx + c.lo + k) * A.ld_src + f);
                            else if (f == 64) v = __ldg(A.val + c.lo + k);
                            else if (f == 65) v = __int_as_float(k);
                            exc_x[i * kTcLvl + f] = v;
                        }
                        named_bar(1, 128);
                        if (tid < nf) {
                            const int cr = tid;
                            const uint64_t T = fin_T[slot * 64 + cr];
                            const uint32_t Ta = (uint32_t)(T >> 32), Tk = 0xFFFFFFFFu - (uint32_t)T;
                            for (int i = 0; i < ne; ++i) {
                                const float* xr = exc_x + i * kTcLvl;
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
                    // write the normal equations (+ lam*n on the diagonal of a finished row) and the residual
                    const bool direct = c.r >= B.n_multi;
                    double* out = direct ? A.gbuf + (size_t)c.r * nf * gs : B.part + (size_t)c.t * nf * gs;
                    const double lam_n = direct ? A.lam * (double)c.n : 0.0;
                    for (int e = tid; e < nf * gs; e += 128) {
                        const int cr = e / gs, f = e - cr * gs;
                        out[e] = f == nf ? xchg[cr * kTcLvl + 64] : xchg[cr * kTcLvl + f] + (f == cr ? lam_n : 0.0);
                    }
                    if (tid == 0 && want_rss) {
                        double v = 0.0;
                        for (int w = 0; w < kTcCW; ++w) v += rss_part[slot * kTcCW + w];
                        if (direct) A.rss_rows[c.row] = v;
                        else B.rss_part[c.t] = v;
                    }
                    named_bar(1, 128);
                }
                ++item;
            }
            tc_cursor_next(A, B, c);
            ++j;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

}  // namespace cals
