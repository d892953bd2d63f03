// gram.cuh -- sketched normal equations from a staged slice.
//
// G[c][f] = sum_{k kept for c} X[k][c] * X[k][f]   (f < nf)
// G[c][nf] = sum_{k kept for c} X[k][c] * y[k]     (the RHS b[c])
// This is the reference's gram_rhs_global (_kernels.py:123-146): G row c
// sums over column c's kept rows only, so G is generally non-symmetric.  The
// sum runs over the kept rows only (algorithmic flops): a few lanes own one
// column and walk its kept-row list or bitmap, each lane accumulating a
// 16-byte-chunk slice of [X | y] with packed FFMA2; partials over q-groups
// are reduced in a fixed order, so results are deterministic.
#pragma once
#include "sweep_common.cuh"

namespace cals {

// ---------------------------------------------------------------------------
// Warp-owned variant: the calling warp owns columns c = c_first + j * c_step
// (j < n_cols) and has already built their kept-row lists.  Columns are
// processed in rounds of CT (power of two, CT * LPC <= 32); q-groups QG split
// each list round-robin and are reduced with shuffles in a fixed order.
// ---------------------------------------------------------------------------
template <int CPL, typename OT>
__device__ __forceinline__ void sparse_gram_owned(uint32_t xs, int sx, uint32_t ys, int nf, int len, bool full,
                                                  uint32_t lists, int Smax, int c_first, int c_step, int n_cols,
                                                  float lam_n, OT* __restrict__ Gout, int lane,
                                                  bool accumulate = false) {
    const int nq = xs_chunks(nf);
    const int LPC = nq < 4 ? nq : 4;
    const int maxct = 32 / LPC;
    const int gs = nf + 1;
    const uint32_t rowb = 4u * (uint32_t)sx;
    for (int j0 = 0; j0 < n_cols; j0 += maxct) {
        const int cnt = min(maxct, n_cols - j0);
        int CT = 1;
        while (CT < cnt) CT <<= 1;
        const int QG = 32 / (CT * LPC);
        const int cs = lane / (QG * LPC);
        const int qg = (lane / LPC) % QG;
        const int fl = lane % LPC;
        const bool cvalid = cs < cnt;
        const int c = c_first + (j0 + (cvalid ? cs : 0)) * c_step;
        const uint32_t L = lists + 2u * (uint32_t)(c * Smax);
        const uint32_t xcol = xs + 4u * (uint32_t)c;
        float acc[4 * CPL];
#pragma unroll
        for (int i = 0; i < 4 * CPL; ++i) acc[i] = 0.f;
        float accb = 0.f;
        const bool chunk_ok_last = (fl + (CPL - 1) * LPC) < nq;
        for (int q = qg; q < len; q += QG) {
            const uint32_t k = full ? (uint32_t)q : lds_u16(L + 2u * (uint32_t)q);
            const uint32_t rb = k * rowb;
            const float xc = cvalid ? lds_f32(xcol + rb) : 0.f;
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                if (i < CPL - 1 || chunk_ok_last) {
                    const float4 v = lds_f128(xs + rb + 16u * (uint32_t)(fl + i * LPC));
                    ffma2_bcast(acc[4 * i + 0], acc[4 * i + 1], v.x, v.y, xc);
                    ffma2_bcast(acc[4 * i + 2], acc[4 * i + 3], v.z, v.w, xc);
                }
            }
            if (fl == 0) accb = fmaf(xc, lds_f32(ys + 4u * k), accb);
        }
        for (int o = LPC; o < LPC * QG; o <<= 1) {
#pragma unroll
            for (int i = 0; i < 4 * CPL; ++i) acc[i] += __shfl_xor_sync(CALS_FULL_MASK, acc[i], o);
            accb += __shfl_xor_sync(CALS_FULL_MASK, accb, o);
        }
        if (cvalid && qg == 0) {
            OT* grow = Gout + (size_t)c * gs;
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                const int ch = fl + i * LPC;
                if (ch < nq) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int f = 4 * ch + t;
                        if (f < nf)
                            grow[f] = (accumulate ? grow[f] : (OT)0) + (OT)acc[4 * i + t] + ((f == c) ? (OT)lam_n : (OT)0);
                    }
                }
            }
            if (fl == 0) grow[nf] = (accumulate ? grow[nf] : (OT)0) + (OT)accb;
        }
        __syncwarp();
    }
}

// Register-resident variant for a warp owning n_cols <= 32/LPC columns: the
// accumulators persist across staged chunks (OwnedAcc), so the reduction and
// the write-out happen once per work item (owned_flush) instead of per chunk.
__host__ __device__ inline bool owned_single_round(int nf, int nwarps) {
    const int nq = xs_chunks(nf);
    const int lpc = nq < 4 ? nq : 4;
    return (nf + nwarps - 1) / nwarps <= 32 / lpc;
}

struct OwnedMap {
    int LPC, QG, cs, qg, fl, c;
    bool cvalid;
    __device__ __forceinline__ OwnedMap(int nf, int c_first, int c_step, int n_cols, int lane) {
        const int nq = xs_chunks(nf);
        LPC = nq < 4 ? nq : 4;
        int CT = 1;
        while (CT < n_cols) CT <<= 1;
        QG = 32 / (CT * LPC);
        cs = lane / (QG * LPC);
        qg = (lane / LPC) % QG;
        fl = lane % LPC;
        cvalid = cs < n_cols;
        c = c_first + (cvalid ? cs : 0) * c_step;
    }
};

template <int CPL, typename AT = float>
struct OwnedAcc {
    AT acc[4 * CPL];
    AT accb;
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < 4 * CPL; ++i) acc[i] = (AT)0;
        accb = (AT)0;
    }
};

// Float64 accumulation of one staged chunk (exact fp32 products, float64 sums):
// the same walk as owned_accumulate with DFMA instead of packed FFMA2.
template <int CPL>
__device__ __forceinline__ void owned_accumulate_f64(OwnedAcc<CPL, double>& S, const OwnedMap& M, uint32_t xs, int sx,
                                                     uint32_t ys, int nf, int kn, bool full, uint32_t bits, int nw) {
    const int nq = xs_chunks(nf);
    const uint32_t rowb = 4u * (uint32_t)sx;
    const uint32_t W = bits + 4u * (uint32_t)(M.c * nw);
    const uint32_t xcol = xs + 4u * (uint32_t)M.c;
    const bool chunk_ok_last = (M.fl + (CPL - 1) * M.LPC) < nq;
    const int nwk = M.cvalid ? (kn + 31) >> 5 : 0;
    for (int wd = M.qg; wd < nwk; wd += M.QG) {
        uint32_t word;
        if (full) {
            const int rem = kn - 32 * wd;
            word = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
        } else {
            word = lds_u32(W + 4u * (uint32_t)wd);
        }
        while (word) {
            const uint32_t k = 32u * (uint32_t)wd + (uint32_t)(__ffs(word) - 1);
            word &= word - 1u;
            const uint32_t rb = k * rowb;
            const double xc = (double)lds_f32(xcol + rb);
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                if (i < CPL - 1 || chunk_ok_last) {
                    const float4 v = lds_f128(xs + rb + 16u * (uint32_t)(M.fl + i * M.LPC));
                    S.acc[4 * i + 0] = fma((double)v.x, xc, S.acc[4 * i + 0]);
                    S.acc[4 * i + 1] = fma((double)v.y, xc, S.acc[4 * i + 1]);
                    S.acc[4 * i + 2] = fma((double)v.z, xc, S.acc[4 * i + 2]);
                    S.acc[4 * i + 3] = fma((double)v.w, xc, S.acc[4 * i + 3]);
                }
            }
            if (M.fl == 0) S.accb = fma(xc, (double)lds_f32(ys + 4u * k), S.accb);
        }
    }
}

// Row M.c of float64 normal equations straight from float64 register sums.
template <int CPL>
__device__ __forceinline__ void owned_flush_f64(OwnedAcc<CPL, double>& S, const OwnedMap& M, int nf,
                                                double* __restrict__ out, double lam_n) {
    const int nq = xs_chunks(nf);
    const int gs = nf + 1;
    for (int o = M.LPC; o < M.LPC * M.QG; o <<= 1) {
#pragma unroll
        for (int i = 0; i < 4 * CPL; ++i) S.acc[i] += __shfl_xor_sync(CALS_FULL_MASK, S.acc[i], o);
        S.accb += __shfl_xor_sync(CALS_FULL_MASK, S.accb, o);
    }
    if (M.cvalid && M.qg == 0) {
        double* grow = out + (size_t)M.c * gs;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int ch = M.fl + i * M.LPC;
            if (ch < nq) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int f = 4 * ch + t;
                    if (f < nf) grow[f] = S.acc[4 * i + t] + ((f == M.c) ? lam_n : 0.0);
                }
            }
        }
        if (M.fl == 0) grow[nf] = S.accb;
    }
}



// Accumulate one staged chunk of kn rows: column M.c over the set bits of its
// kept-row bitmap words (bits[c][w], nw words per column), or over all rows
// when full.  q-group g takes words g, g + QG, ...
template <int CPL>
__device__ __forceinline__ void owned_accumulate(OwnedAcc<CPL>& S, const OwnedMap& M, uint32_t xs, int sx,
                                                 uint32_t ys, int nf, int kn, bool full, uint32_t bits, int nw) {
    const int nq = xs_chunks(nf);
    const uint32_t rowb = 4u * (uint32_t)sx;
    const uint32_t W = bits + 4u * (uint32_t)(M.c * nw);
    const uint32_t xcol = xs + 4u * (uint32_t)M.c;
    const bool chunk_ok_last = (M.fl + (CPL - 1) * M.LPC) < nq;
    const int nwk = M.cvalid ? (kn + 31) >> 5 : 0;
    for (int wd = M.qg; wd < nwk; wd += M.QG) {
      uint32_t word;
      if (full) {
          const int rem = kn - 32 * wd;
          word = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
      } else {
          word = lds_u32(W + 4u * (uint32_t)wd);
      }
      while (word) {
        const uint32_t k = 32u * (uint32_t)wd + (uint32_t)(__ffs(word) - 1);
        word &= word - 1u;
        const uint32_t rb = k * rowb;
        const float xc = lds_f32(xcol + rb);
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            if (i < CPL - 1 || chunk_ok_last) {
                const float4 v = lds_f128(xs + rb + 16u * (uint32_t)(M.fl + i * M.LPC));
                ffma2_bcast(S.acc[4 * i + 0], S.acc[4 * i + 1], v.x, v.y, xc);
                ffma2_bcast(S.acc[4 * i + 2], S.acc[4 * i + 3], v.z, v.w, xc);
            }
        }
        if (M.fl == 0) S.accb = fmaf(xc, lds_f32(ys + 4u * k), S.accb);
      }
    }
}

// Fixed-order reduction over the q-groups; row M.c of out (stride nf+1).
template <int CPL>
__device__ __forceinline__ void owned_flush(OwnedAcc<CPL>& S, const OwnedMap& M, int nf, float* __restrict__ out,
                                            float lam_n = 0.f) {
    const int nq = xs_chunks(nf);
    const int gs = nf + 1;
    for (int o = M.LPC; o < M.LPC * M.QG; o <<= 1) {
#pragma unroll
        for (int i = 0; i < 4 * CPL; ++i) S.acc[i] += __shfl_xor_sync(CALS_FULL_MASK, S.acc[i], o);
        S.accb += __shfl_xor_sync(CALS_FULL_MASK, S.accb, o);
    }
    if (M.cvalid && M.qg == 0) {
        float* grow = out + (size_t)M.c * gs;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int ch = M.fl + i * M.LPC;
            if (ch < nq) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int f = 4 * ch + t;
                    if (f < nf) grow[f] = S.acc[4 * i + t] + ((f == M.c) ? lam_n : 0.f);
                }
            }
        }
        if (M.fl == 0) grow[nf] = S.accb;
    }
}

// Fold the chunk's fp32 sums into float64 shared-memory accumulators G64
// ([nf][nf+1] doubles) and restart them at zero: fp32 only ever sums one staged
// chunk's kept rows (tens of terms), so the Gram of a long row carries float64
// accumulation error instead of the fp32 error of a 16384-row sequential sum
// (measured on the 500M config: that error dominated the factor error of
// ill-conditioned long rows).  q-groups are reduced first (fixed order).
template <int CPL>
__device__ __forceinline__ void owned_fold(OwnedAcc<CPL>& S, const OwnedMap& M, int nf, double* __restrict__ G64) {
    const int nq = xs_chunks(nf);
    const int gs = nf + 1;
    for (int o = M.LPC; o < M.LPC * M.QG; o <<= 1) {
#pragma unroll
        for (int i = 0; i < 4 * CPL; ++i) S.acc[i] += __shfl_xor_sync(CALS_FULL_MASK, S.acc[i], o);
        S.accb += __shfl_xor_sync(CALS_FULL_MASK, S.accb, o);
    }
    if (M.cvalid && M.qg == 0) {
        double* grow = G64 + (size_t)M.c * gs;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int ch = M.fl + i * M.LPC;
            if (ch < nq) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int f = 4 * ch + t;
                    if (f < nf) grow[f] += (double)S.acc[4 * i + t];
                }
            }
        }
        if (M.fl == 0) grow[nf] += (double)S.accb;
    }
    S.zero();
}

// Write row M.c of the normal equations from G64 (+ lam_n on the diagonal, in float64).
template <int CPL>
__device__ __forceinline__ void owned_flush64(const OwnedMap& M, int nf, const double* __restrict__ G64,
                                              double* __restrict__ out, double lam_n) {
    const int nq = xs_chunks(nf);
    const int gs = nf + 1;
    if (M.cvalid && M.qg == 0) {
        const double* grow = G64 + (size_t)M.c * gs;
        double* orow = out + (size_t)M.c * gs;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int ch = M.fl + i * M.LPC;
            if (ch < nq) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int f = 4 * ch + t;
                    if (f < nf) orow[f] = grow[f] + ((f == M.c) ? lam_n : 0.0);
                }
            }
        }
        if (M.fl == 0) orow[nf] = grow[nf];
    }
}

// Kept-row list of one column from its column-major bitmap words (ascending k).
__device__ __forceinline__ void bitmap_to_list(uint32_t words, int nwords, uint32_t list, int lane) {
    int base = 0;
    for (int w0 = 0; w0 < nwords; w0 += 32) {
        const int w = w0 + lane;
        uint32_t word = w < nwords ? lds_u32(words + 4u * (uint32_t)w) : 0u;
        const int cnt = __popc(word);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(CALS_FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        int pos = base + incl - cnt;
        while (word) {
            const int b = __ffs(word) - 1;
            word &= word - 1;
            sts_u16(list + 2u * (uint32_t)pos, (uint32_t)(32 * w + b));
            ++pos;
        }
        base += __shfl_sync(CALS_FULL_MASK, incl, 31);
    }
    __syncwarp();
}

}  // namespace cals
