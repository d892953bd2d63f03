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

constexpr int kTcThreads = 512;
constexpr int kTcKC = 64;        // slice rows per chunk (two K-steps of 32)
constexpr int kTcStages = 4;     // fp32 staging ring depth
constexpr int kTcSX = 80;        // staged row stride in floats (320 B: conflict-free float4 reads)
constexpr int kTcN = 144;        // N side: two levels x (64 factor columns + y + 7 zero pad)
constexpr int kTcLvl = 72;       // N columns per level
constexpr int kTcATile = 4096;   // M = 128 (two levels x 64 columns) x 32 K bytes
constexpr int kTcBTile = 4608;   // N = 144 x 32 K bytes
constexpr int kTcKStepBytes = 2 * kTcATile + 2 * kTcBTile;  // A12 A34 B12 B34
constexpr int kTcDigitBuf = 2 * kTcKStepBytes;              // one chunk (two K-steps)
constexpr int kTcAccB = 256;     // TMEM column of the second accumulator (levels 4..6)

struct TcSmem {
    // offsets (bytes) inside the dynamic shared memory
    static constexpr int stage_x = 0;                                       // [4][64][kTcSX] f32
    static constexpr int stage_y = stage_x + kTcStages * kTcKC * kTcSX * 4;  // [4][64] f32
    static constexpr int digits = stage_y + kTcStages * kTcKC * 4;          // [2][kTcDigitBuf], 1024-aligned below
    static constexpr int digits_al = (digits + 1023) & ~1023;
    static constexpr int xchg = digits_al + 2 * kTcDigitBuf;                // [64][72] f64 partial exchange
    static constexpr int total = xchg + 64 * kTcLvl * 8;
};

__host__ __device__ constexpr uint32_t tc_mn_off(uint32_t mn, uint32_t k) {
    return (mn >> 4) * 512u + (k >> 3) * 128u + (k & 7u) * 16u + (mn & 15u);
}

// power-of-two scale alpha with |x| / alpha < 0.4962 for |x| <= amax (so the top
// digit of rint(x 2^32 / alpha) stays in [-128, 127]); returns the exponent E
__device__ __forceinline__ int tc_scale_exp(float amax) {
    if (!(amax > 0.f)) return 0;
    int e;
    frexpf(amax * 2.015625f, &e);  // amax * 2.015625 in [2^(e-1), 2^e)
    return e;
}

// low bytes of four words -> one word
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// per-column maxima of |source| (abs bits), the digit scales of the tensor-core Gram
__global__ void __launch_bounds__(256) col_absmax_kernel(const float* __restrict__ src, int64_t n_src, int ld, int nf,
                                                         unsigned int* __restrict__ out) {
    __shared__ unsigned int m[CALS_MAX_NF_DEV];
    for (int c = threadIdx.x; c < nf; c += blockDim.x) m[c] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < nf; c0 += 32) {
        const int c = c0 + lane;
        unsigned int v = 0u;
        if (c < nf)
            for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < n_src;
                 j += (int64_t)gridDim.x * (blockDim.x >> 5))
                v = max(v, abs_bits(__ldg(src + j * ld + c)));
        if (c < nf) atomicMax(&m[c], v);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nf; c += blockDim.x)
        if (m[c]) atomicMax(&out[c], m[c]);
}

struct TcCursor {
    int64_t t;   // work item index (batch-relative) or >= n_tiles when done
    int k0;      // first slice row of the chunk
    int kend;    // end of the work item
    int r, row;  // batch row, row id
    int64_t lo;  // first rating of the row
    int n;       // row length
    int kbeg;
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

// issue the gathered fp32 rows of chunk `c` into stage s (threads 0..63: one row each)
__device__ __forceinline__ void tc_issue_stage(const SweepArgs& A, const BigArgs& B, const TcCursor& c,
                                               uint32_t stage_x, uint32_t mbar) {
    if (c.t >= B.n_tiles) return;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // earlier generic reads of the stage
    const int kn = min(kTcKC, c.kend - c.k0);
    const uint32_t rowbytes = 16u * (uint32_t)xs_chunks(A.nf);
    if (threadIdx.x == 0) mbar_expect_tx(mbar, (uint32_t)kn * rowbytes);
    if (threadIdx.x < kn) {
        const int64_t j = __ldg(A.idx + c.lo + c.k0 + threadIdx.x);
        bulk_g2s(stage_x + (uint32_t)threadIdx.x * (kTcSX * 4u), A.src + j * A.ld_src, rowbytes, mbar);
    }
}

__global__ void __launch_bounds__(kTcThreads, 1) big_gram_tc_kernel(SweepArgs A, BigArgs B,
                                                                    const unsigned int* __restrict__ colmax) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t s_Ta[64], s_Tk[64];
    __shared__ float s_scale[64];       // 2^(32 - E_c): x -> fixed point
    __shared__ double s_alpha[65];      // 2^E_c (and alpha_y at 64)
    __shared__ float s_wold[64];
    __shared__ float s_red[32];
    __shared__ float s_ypre[2][kTcKC];  // residual: per-row partial dots of the two column halves
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_mbar_stage[kTcStages];
    __shared__ __align__(8) unsigned long long s_mbar_mma[2];
    __shared__ float s_yscale;
    __shared__ double s_rss[16];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nf = A.nf, gs = nf + 1;
    const uint32_t sbase = tc::smem_addr(smem);
    const uint32_t s_stage_x = sbase + TcSmem::stage_x;
    float* stage_y = reinterpret_cast<float*>(smem + TcSmem::stage_y);
    const uint32_t s_digits = sbase + TcSmem::digits_al;
    unsigned char* digits = smem + TcSmem::digits_al;
    double* xchg = reinterpret_cast<double*>(smem + TcSmem::xchg);

    // zero both digit tile sets once: padding bytes (N columns 65..71 of each level) are never written
    for (int e = tid; e < 2 * kTcDigitBuf / 16; e += blockDim.x)
        reinterpret_cast<uint4*>(digits)[e] = make_uint4(0u, 0u, 0u, 0u);
    if (warp == 0) tc::tmem_alloc<512>(&s_tmem);
    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) mbar_init(smem_u32(&s_mbar_stage[s]), 1);
        for (int s = 0; s < 2; ++s) mbar_init(smem_u32(&s_mbar_mma[s]), 1);
    }
    if (tid < 64) {
        const int E = tid < nf ? tc_scale_exp(__uint_as_float(colmax[tid])) : 0;
        s_scale[tid] = ldexpf(1.0f, 32 - E);
        s_alpha[tid] = ldexp(1.0, E);
    }
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t idesc = tc::idesc_i8(128, kTcN) | (1u << 15) | (1u << 16);  // MN-major A and B

    // producer cursor runs kTcStages - 1 chunks ahead of the consumer
    TcCursor cons{}, prod{};
    cons.t = blockIdx.x;
    tc_cursor_item(A, B, cons);
    prod = cons;
    uint32_t stage_phase = 0u, mma_phase = 0u;  // bit s: parity of the next completion of barrier s
    uint32_t mma_pending = 0u;                  // bit b: a commit on s_mbar_mma[b] not yet waited for
    float ypf = 0.f;                            // y of row `tid` of the chunk kTcStages - 1 ahead
    int ypf_stage = -1;
    for (int s = 0; s < kTcStages - 1; ++s) {
        tc_issue_stage(A, B, prod, s_stage_x + (uint32_t)s * (kTcKC * kTcSX * 4u), smem_u32(&s_mbar_stage[s]));
        if (prod.t < B.n_tiles && tid < min(kTcKC, prod.kend - prod.k0))
            stage_y[s * kTcKC + tid] = __ldg(A.val + prod.lo + prod.k0 + tid);
        if (prod.t < B.n_tiles) tc_cursor_next(A, B, prod);
    }
    int64_t chunk = 0;
    double racc = 0.0;
    bool item_first = true;
    const bool want_rss = A.rss_rows != nullptr;

    while (cons.t < B.n_tiles) {
        const int st = (int)(chunk % kTcStages);
        const int db = (int)(chunk & 1);
        // ---- prefetch: the chunk kTcStages - 1 ahead into the stage freed by the previous chunk
        {
            const int ps = (int)((chunk + kTcStages - 1) % kTcStages);
            if (ypf_stage >= 0 && tid < kTcKC) stage_y[ypf_stage * kTcKC + tid] = ypf;
            ypf_stage = -1;
            if (prod.t < B.n_tiles) {
                tc_issue_stage(A, B, prod, s_stage_x + (uint32_t)ps * (kTcKC * kTcSX * 4u),
                               smem_u32(&s_mbar_stage[ps]));
                if (tid < min(kTcKC, prod.kend - prod.k0)) {
                    ypf = __ldg(A.val + prod.lo + prod.k0 + tid);
                    ypf_stage = ps;
                }
                tc_cursor_next(A, B, prod);
            }
        }
        // ---- per work item setup
        if (item_first) {
            if (tid < 64) {
                const uint64_t T = tid < nf ? B.thr[(size_t)cons.r * nf + tid] : ~0ull;
                s_Ta[tid] = (uint32_t)(T >> 32);
                s_Tk[tid] = 0xFFFFFFFFu - (uint32_t)T;
                s_wold[tid] = (want_rss && tid < nf) ? A.tgt_old[(int64_t)cons.row * A.ld_old + tid] : 0.f;
            }
            // y scale of this work item
            float ym = 0.f;
            for (int k = cons.kbeg + tid; k < cons.kend; k += blockDim.x) ym = fmaxf(ym, fabsf(__ldg(A.val + cons.lo + k)));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ym = fmaxf(ym, __shfl_xor_sync(CALS_FULL_MASK, ym, o));
            if (lane == 0) s_red[warp] = ym;
            racc = 0.0;
            __syncthreads();
            if (tid == 0) {
                float m = 0.f;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, s_red[w]);
                const int E = tc_scale_exp(m);
                s_yscale = ldexpf(1.0f, 32 - E);
                s_alpha[64] = ldexp(1.0, E);
            }
        }
        // ---- wait for the chunk's rows and for the MMAs that last read tile set db
        mbar_wait(smem_u32(&s_mbar_stage[st]), (stage_phase >> st) & 1u);
        stage_phase ^= 1u << st;
        if (mma_pending & (1u << db)) {  // the MMAs that last read tile set db
            mbar_wait(smem_u32(&s_mbar_mma[db]), (mma_phase >> db) & 1u);
            mma_phase ^= 1u << db;
            mma_pending &= ~(1u << db);
        }
        __syncthreads();  // per-item setup visible; stage_y of this chunk written (previous iterations)
        const int kn = min(kTcKC, cons.kend - cons.k0);
        // ---- digit pass: warp w -> rows 8 (w >> 1) .. +7, column quads 8 (w & 1) .. +7
        {
            const float* Xs = reinterpret_cast<const float*>(smem + TcSmem::stage_x) + st * kTcKC * kTcSX;
            const float* ys = stage_y + st * kTcKC;
            const int kl = lane >> 2, fql = lane & 3;
            const int k = 8 * (warp >> 1) + kl;
            const bool krow = k < kn;
            const uint32_t kg = (uint32_t)(cons.k0 + k);
            unsigned char* dbuf = digits + db * kTcDigitBuf + (k >> 5) * kTcKStepBytes;
            const uint32_t kk = (uint32_t)(k & 31);
            float pdot = 0.f;
#pragma unroll
            for (int it = 0; it < 2; ++it) {
                const int fq = 4 * (2 * (warp & 1) + it) + fql;  // column quad 0..15
                const int c0 = 4 * fq;
                float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                if (krow && c0 < nf) x = *reinterpret_cast<const float4*>(Xs + k * kTcSX + c0);
                const float xv[4] = {x.x, x.y, x.z, x.w};
                uint32_t Y[4][4];   // [element][level 4..1]: Y0 = X, Y_{i+1} = (Y_i + 128) >> 8
                uint32_t keepm = 0u;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int c = c0 + j;
                    const float v = (c < nf) ? xv[j] : 0.f;
                    if (want_rss) pdot = fmaf(v, s_wold[c & 63], pdot);
                    const int X = __float2int_rn(v * s_scale[c & 63]);
                    Y[j][0] = (uint32_t)X;
                    Y[j][1] = (uint32_t)((X + 128) >> 8);
                    Y[j][2] = (uint32_t)(((int)Y[j][1] + 128) >> 8);
                    Y[j][3] = (uint32_t)(((int)Y[j][2] + 128) >> 8);
                    const uint32_t a = abs_bits(v);
                    const bool keep = krow && c < nf && (a > s_Ta[c & 63] || (a == s_Ta[c & 63] && kg <= s_Tk[c & 63]));
                    keepm |= keep ? (0xFFu << (8 * j)) : 0u;
                }
                // level L (1..4) word of the quad = bytes of Y[.][4 - L]
#pragma unroll
                for (int L = 1; L <= 4; ++L) {
                    const uint32_t w = pack4(Y[0][4 - L], Y[1][4 - L], Y[2][4 - L], Y[3][4 - L]);
                    const int pair = (L - 1) >> 1, half = (L - 1) & 1;
                    // N side (unmasked): tile B(pair), column half * 72 + c0
                    *reinterpret_cast<uint32_t*>(dbuf + 2 * kTcATile + pair * kTcBTile +
                                                 tc_mn_off((uint32_t)(half * kTcLvl + c0), kk)) = w;
                    // M side (masked): tile A(pair), row half * 64 + c0
                    *reinterpret_cast<uint32_t*>(dbuf + pair * kTcATile + tc_mn_off((uint32_t)(half * 64 + c0), kk)) =
                        w & keepm;
                }
            }
            // y digits: one lane per row (column 64 of each level, zero-padded word)
            if (fql == 0 && (warp & 1) == 0) {
                const float yv = krow ? ys[k] : 0.f;
                const int X = __float2int_rn(yv * s_yscale);
                uint32_t y4[4];
                y4[0] = (uint32_t)X;
                y4[1] = (uint32_t)((X + 128) >> 8);
                y4[2] = (uint32_t)(((int)y4[1] + 128) >> 8);
                y4[3] = (uint32_t)(((int)y4[2] + 128) >> 8);
#pragma unroll
                for (int L = 1; L <= 4; ++L) {
                    const int pair = (L - 1) >> 1, half = (L - 1) & 1;
                    *reinterpret_cast<uint32_t*>(dbuf + 2 * kTcATile + pair * kTcBTile +
                                                 tc_mn_off((uint32_t)(half * kTcLvl + 64), kk)) = y4[4 - L] & 0xFFu;
                }
            }
            if (want_rss) {
                // row dot = sum over the 4 lanes of the quad group and the two column halves (fixed order)
                pdot += __shfl_xor_sync(CALS_FULL_MASK, pdot, 1);
                pdot += __shfl_xor_sync(CALS_FULL_MASK, pdot, 2);
                if (fql == 0) s_ypre[warp & 1][k] = pdot;
            }
        }
        tc::fence_smem_async();
        __syncthreads();
        // ---- MMAs of this chunk (thread 0), completion -> s_mbar_mma[db]
        if (tid == 0) {
            tc::fence_after();
            const int nks = (kn + 31) >> 5;
            for (int ks = 0; ks < nks; ++ks) {
                const uint32_t base = s_digits + (uint32_t)(db * kTcDigitBuf + ks * kTcKStepBytes);
                const uint64_t a12 = tc::sdesc(base, 128, 512), a34 = tc::sdesc(base + kTcATile, 128, 512);
                const uint64_t b12 = tc::sdesc(base + 2 * kTcATile, 128, 512);
                const uint64_t b34 = tc::sdesc(base + 2 * kTcATile + kTcBTile, 128, 512);
                const uint32_t acc = (item_first && ks == 0) ? 0u : 1u;
                tc::mma_i8_ss(tmem, a12, b12, idesc, acc);
                tc::mma_i8_ss(tmem + kTcAccB, a12, b34, idesc, acc);
                tc::mma_i8_ss(tmem + kTcAccB, a34, b12, idesc, 1u);
            }
            tc::commit(smem_u32(&s_mbar_mma[db]));
        }
        mma_pending |= 1u << db;
        // ---- residual of the previous rows (fp64 from the fp32 dot)
        if (want_rss && tid < kn) {
            const double d = (double)stage_y[st * kTcKC + tid] - ((double)s_ypre[0][tid] + (double)s_ypre[1][tid]);
            racc = fma(d, d, racc);
        }
        const bool item_last = cons.k0 + kTcKC >= cons.kend;
        if (item_last) {
            // all MMAs of the item done -> recombine G and b in float64
            // (a commit tracks every earlier MMA of the thread, so this one covers the whole item)
            mbar_wait(smem_u32(&s_mbar_mma[db]), (mma_phase >> db) & 1u);
            mma_phase ^= 1u << db;
            mma_pending &= ~(1u << db);
            tc::fence_after();
            const int row = cons.row, r = cons.r;
            const bool direct = r >= B.n_multi;
            double* out = direct ? A.gbuf + (size_t)r * nf * gs : B.part + (size_t)cons.t * nf * gs;
            if (warp == 2 || warp == 3) {
                // rows of the second stacked level (ra = 1): partials into the exchange buffer
                const int c = 32 * (warp - 2) + lane;
                const uint32_t lrow = (uint32_t)(32 * warp) << 16;
                const double wA0 = ldexp(1.0, -24), wA1 = ldexp(1.0, -32), wB0 = ldexp(1.0, -40), wB1 = ldexp(1.0, -48);
                for (int f0 = 0; f0 < kTcLvl; f0 += 8) {
                    uint32_t a0[8], a1[8], b0[8], b1[8];
                    tc::ld_32x32b_x8(tmem + lrow + f0, a0);
                    tc::ld_32x32b_x8(tmem + lrow + kTcLvl + f0, a1);
                    tc::ld_32x32b_x8(tmem + lrow + kTcAccB + f0, b0);
                    tc::ld_32x32b_x8(tmem + lrow + kTcAccB + kTcLvl + f0, b1);
                    tc::ld_wait();
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        xchg[c * kTcLvl + f0 + j] = wA0 * (double)(int)a0[j] + wA1 * (double)(int)a1[j] +
                                                    wB0 * (double)(int)b0[j] + wB1 * (double)(int)b1[j];
                }
            }
            __syncthreads();
            if (warp < 2) {
                // ra == 0 rows: own partial + the exchanged ra == 1 partial, scaled
                const int c = 32 * warp + lane;
                const uint32_t lrow = (uint32_t)(32 * warp) << 16;
                const double wA0 = ldexp(1.0, -16), wA1 = ldexp(1.0, -24), wB0 = ldexp(1.0, -32), wB1 = ldexp(1.0, -40);
                for (int f0 = 0; f0 < kTcLvl; f0 += 8) {
                    uint32_t a0[8], a1[8], b0[8], b1[8];
                    tc::ld_32x32b_x8(tmem + lrow + f0, a0);
                    tc::ld_32x32b_x8(tmem + lrow + kTcLvl + f0, a1);
                    tc::ld_32x32b_x8(tmem + lrow + kTcAccB + f0, b0);
                    tc::ld_32x32b_x8(tmem + lrow + kTcAccB + kTcLvl + f0, b1);
                    tc::ld_wait();
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int f = f0 + j;
                        if (c < nf && f <= 64 && (f < nf || f == 64)) {
                            const double p = wA0 * (double)(int)a0[j] + wA1 * (double)(int)a1[j] +
                                             wB0 * (double)(int)b0[j] + wB1 * (double)(int)b1[j];
                            const double g = s_alpha[c] * s_alpha[f] * (p + xchg[c * kTcLvl + f]);
                            if (f == 64) {
                                out[(size_t)c * gs + nf] = g;
                            } else {
                                out[(size_t)c * gs + f] = g + ((direct && f == c) ? A.lam * (double)cons.n : 0.0);
                            }
                        }
                    }
                }
            }
            if (want_rss) {
                double v = racc;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CALS_FULL_MASK, v, o);
                if (lane == 0) s_rss[warp] = v;
            }
            tc::fence_before();
            __syncthreads();
            if (want_rss && tid == 0) {
                double v = 0.0;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += s_rss[w];
                if (direct) A.rss_rows[row] = v;
                else B.rss_part[cons.t] = v;
            }
        }
        item_first = item_last;
        tc_cursor_next(A, B, cons);
        ++chunk;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

}  // namespace cals
