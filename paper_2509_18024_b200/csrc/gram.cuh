// gram.cuh -- sketched normal equations from a staged slice.
//
// G[c][f] = sum_k P[k][c] * X[k][c] * X[k][f]   (f < nf)
// G[c][nf] = sum_k P[k][c] * X[k][c] * y[k]      (the RHS b[c])
// with P the selection mask (bit c of mb[k]).  This is the reference's
// gram_rhs_global (_kernels.py:123-146) -- G row c sums over column c's
// kept rows only, so G is generally non-symmetric -- written as a masked
// dense contraction (P . X)^T [X | y] so that every thread runs a 4x4
// register tile with vector shared-memory loads.  Partials over k-groups
// are reduced in a fixed order, so results are deterministic.
#pragma once
#include "sweep_common.cuh"

namespace cals {

// One 4x4 tile (rows c0..c0+3, columns f0..f0+3 of [X | y]) over k = kbeg, kbeg+kstep, ...
__device__ __forceinline__ void gram_tile(const float* __restrict__ Xs, int sx, const float* __restrict__ ys,
                                          const uint32_t* __restrict__ mb, int mw, int n, int nf, int c0, int f0,
                                          int kbeg, int kstep, float (&acc)[4][4]) {
    const int wsel = c0 >> 5, sh = c0 & 31;
    const int yslot = nf - f0;  // component of the B tile that is the response (if in [0, 4))
    const bool bx = f0 < 4 * xs_chunks(nf);  // staged data chunks only (padding beyond is not staged)
    (void)sx;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 4
    for (int k = kbeg; k < n; k += kstep) {
        const float4 av = *reinterpret_cast<const float4*>(Xs + (size_t)k * sx + c0);
        float4 bv = bx ? *reinterpret_cast<const float4*>(Xs + (size_t)k * sx + f0) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (yslot >= 0 && yslot < 4) {
            const float yk = ys[k];
            bv.x = yslot == 0 ? yk : bv.x;
            bv.y = yslot == 1 ? yk : bv.y;
            bv.z = yslot == 2 ? yk : bv.z;
            bv.w = yslot == 3 ? yk : bv.w;
        }
        const uint32_t m = mb[k * mw + wsel] >> sh;
        const float a[4] = {(m & 1u) ? av.x : 0.f, (m & 2u) ? av.y : 0.f, (m & 4u) ? av.z : 0.f,
                            (m & 8u) ? av.w : 0.f};
        const float b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
}

// Must be called by all threads of the block.  Xs: n rows, stride sx (zero
// padding beyond nf), ys: n responses, mb: n * mw mask words.
// Writes (or adds into) G (nf x (nf+1), row stride nf+1).  scratch: >= blockDim*16 floats.
__device__ void tile_gram(const float* __restrict__ Xs, int sx, const float* __restrict__ ys,
                          const uint32_t* __restrict__ mb, int mw, int n, int nf, float* __restrict__ G,
                          float* __restrict__ scratch, bool accumulate = false) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int gs = nf + 1;
    const int RB = (nf + 3) >> 2, CB = (gs + 3) >> 2, NB = RB * CB;
    if (NB <= nt) {
        const int KG = nt / NB;
        if (tid < NB * KG) {
            const int bid = tid % NB, kg = tid / NB;
            float acc[4][4];
            gram_tile(Xs, sx, ys, mb, mw, n, nf, (bid / CB) * 4, (bid % CB) * 4, kg, KG, acc);
            float* out = scratch + (size_t)(kg * NB + bid) * 16;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) out[i * 4 + j] = acc[i][j];
        }
        __syncthreads();
        for (int e = tid; e < nf * gs; e += nt) {
            const int c = e / gs, f = e - c * gs;
            const int bid = (c >> 2) * CB + (f >> 2);
            const int slot = (c & 3) * 4 + (f & 3);
            float v = 0.f;
            for (int g = 0; g < KG; ++g) v += scratch[(size_t)(g * NB + bid) * 16 + slot];
            G[c * gs + f] = accumulate ? G[c * gs + f] + v : v;
        }
        __syncthreads();
    } else {
        for (int bid = tid; bid < NB; bid += nt) {
            const int c0 = (bid / CB) * 4, f0 = (bid % CB) * 4;
            float acc[4][4];
            gram_tile(Xs, sx, ys, mb, mw, n, nf, c0, f0, 0, 1, acc);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int c = c0 + i, f = f0 + j;
                    if (c < nf && f < gs) G[c * gs + f] = accumulate ? G[c * gs + f] + acc[i][j] : acc[i][j];
                }
        }
        __syncthreads();
    }
}

// Selection bitmap: bit c of mb[k*mw + c/32] = (key(k0 + k, c) >= thr[c]).
// Lanes run along columns (conflict-free row reads), ballots form the words;
// for nf <= 16 several rows share a warp.
__device__ void build_mask(const float* __restrict__ Xs, int sx, int n, int nf, const uint64_t* thr, bool full,
                           uint32_t* __restrict__ mb, int mw, int k0 = 0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    int P = 32;
    if (nf <= 16) P = nf <= 1 ? 1 : (nf <= 2 ? 2 : (nf <= 4 ? 4 : (nf <= 8 ? 8 : 16)));
    const int rpw = 32 / P, sub = lane / P, cl = lane - sub * P;
    const uint32_t fieldmask = P == 32 ? 0xffffffffu : ((1u << P) - 1u);
    for (int base = warp * rpw; base < n; base += nwarps * rpw) {
        const int k = base + sub;
        for (int w = 0; w < mw; ++w) {
            const int c = w * 32 + cl;
            bool bit = false;
            if (k < n && c < nf)
                bit = full || make_key(Xs[(size_t)k * sx + c], (uint32_t)(k0 + k)) >= thr[c];
            const uint32_t bal = __ballot_sync(CALS_FULL_MASK, bit);
            if (cl == 0 && k < n) mb[k * mw + w] = (bal >> (sub * P)) & fieldmask;
        }
    }
}

// ---------------------------------------------------------------------------
// Sparse sketched normal equations (algorithmic flop count): for every column
// c, G[c][:] = sum_{k in S_c} X[k][c] * [X[k][:] | y[k]] over the kept rows
// S_c only (_kernels.py:132-145).  A warp task owns CT columns; its lanes are
// (column slot, q-group, chunk lane): LPC lanes per column each own CPL
// 16-byte chunks of the row (interleaved, so the lanes of one column read one
// contiguous row segment), QG q-groups split the kept-row list round-robin and
// are reduced with shuffles in a fixed order; lane (fl == 0) also owns b[c].
// Kept-row lists (ascending k) are built from the selection bitmap by the
// same warp.  Writes rows of G (+lam_n on the diagonal) to Gout (row stride nf+1).
// ---------------------------------------------------------------------------
template <int CPL>
__device__ __forceinline__ void sparse_gram_warp(uint32_t xs, int sx, uint32_t ys, uint32_t mb, int mw, int n, int nf,
                                                 int s, bool full, uint32_t lists, int Smax, float lam_n,
                                                 float* __restrict__ Gout, int warp, int nwarps, int lane) {
    const int nq = xs_chunks(nf);
    const int LPC = nq < 4 ? nq : 4;
    int CT = (nf + nwarps - 1) / nwarps;    // columns per task: power of two, CT * LPC <= 32
    CT = CT <= 1 ? 1 : (CT <= 2 ? 2 : (CT <= 4 ? 4 : (CT <= 8 ? 8 : (CT <= 16 ? 16 : 32))));
    while (CT * LPC > 32) CT >>= 1;
    const int QG = 32 / (CT * LPC);         // power of two
    const int cs = lane / (QG * LPC);
    const int qg = (lane / LPC) % QG;
    const int fl = lane % LPC;
    const int gs = nf + 1;
    const int ntask = (nf + CT - 1) / CT;
    const uint32_t rowb = 4u * (uint32_t)sx;
    for (int task = warp; task < ntask; task += nwarps) {
        const int cbase = task * CT;
        const int c = cbase + cs;
        const bool cvalid = c < nf;
        if (!full) {
            // lists of the task's columns from the bitmap (CT columns share one word)
            int cnt = 0;  // lane cc keeps column cbase+cc's running count
            const int wsel = cbase >> 5, sh = cbase & 31;
            for (int k0 = 0; k0 < n; k0 += 32) {
                const int k = k0 + lane;
                const uint32_t word = k < n ? (lds_u32(mb + 4u * (uint32_t)(k * mw + wsel)) >> sh) : 0u;
                for (int cc = 0; cc < CT && cbase + cc < nf; ++cc) {
                    const bool bit = (word >> cc) & 1u;
                    const uint32_t bal = __ballot_sync(CALS_FULL_MASK, bit);
                    const int base = __shfl_sync(CALS_FULL_MASK, cnt, cc);
                    if (bit)
                        sts_u16(lists + 2u * (uint32_t)((cbase + cc) * Smax + base + __popc(bal & lanemask_lt())), k);
                    if (lane == cc) cnt += __popc(bal);
                }
            }
            __syncwarp();
        }
        const int len = full ? n : s;
        const uint32_t L = lists + 2u * (uint32_t)((cvalid ? c : cbase) * Smax);
        const uint32_t xcol = xs + 4u * (uint32_t)(cvalid ? c : 0);
        float acc[4 * CPL];
#pragma unroll
        for (int i = 0; i < 4 * CPL; ++i) acc[i] = 0.f;
        float accb = 0.f;
        const bool chunk_ok_last = (fl + (CPL - 1) * LPC) < nq;
        for (int q = qg; q < len; q += QG) {
            const uint32_t k = full ? (uint32_t)q : lds_u16(L + 2u * (uint32_t)q);
            const uint32_t rb = k * rowb;
            const float xc = lds_f32(xcol + rb);
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                const int ch = fl + i * LPC;
                if (i < CPL - 1 || chunk_ok_last) {
                    const float4 v = lds_f128(xs + rb + 16u * (uint32_t)ch);
                    ffma2_bcast(acc[4 * i + 0], acc[4 * i + 1], v.x, v.y, xc);
                    ffma2_bcast(acc[4 * i + 2], acc[4 * i + 3], v.z, v.w, xc);
                }
            }
            if (fl == 0) accb = fmaf(xc, lds_f32(ys + 4u * k), accb);
        }
        // fixed-order reduction over the q-groups (lane bits LPC .. LPC*QG)
        for (int o = LPC; o < LPC * QG; o <<= 1) {
#pragma unroll
            for (int i = 0; i < 4 * CPL; ++i) acc[i] += __shfl_xor_sync(CALS_FULL_MASK, acc[i], o);
            accb += __shfl_xor_sync(CALS_FULL_MASK, accb, o);
        }
        if (cvalid && qg == 0) {
            float* grow = Gout + (size_t)c * gs;
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                const int ch = fl + i * LPC;
                if (ch < nq) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int f = 4 * ch + t;
                        if (f < nf) grow[f] = acc[4 * i + t] + ((f == c) ? lam_n : 0.f);
                    }
                }
            }
            if (fl == 0) grow[nf] = accb;
        }
        __syncwarp();
    }
}

// CPL (16-byte chunks per lane) dispatch: nq <= 4 -> 1, <= 8 -> 2, <= 16 -> 4, else 8.
__device__ __forceinline__ void sparse_gram(uint32_t xs, int sx, uint32_t ys, uint32_t mb, int mw, int n, int nf, int s,
                                            bool full, uint32_t lists, int Smax, float lam_n, float* Gout, int warp,
                                            int nwarps, int lane) {
    const int nq = xs_chunks(nf);
    if (nq <= 4) sparse_gram_warp<1>(xs, sx, ys, mb, mw, n, nf, s, full, lists, Smax, lam_n, Gout, warp, nwarps, lane);
    else if (nq <= 8) sparse_gram_warp<2>(xs, sx, ys, mb, mw, n, nf, s, full, lists, Smax, lam_n, Gout, warp, nwarps, lane);
    else if (nq <= 16) sparse_gram_warp<4>(xs, sx, ys, mb, mw, n, nf, s, full, lists, Smax, lam_n, Gout, warp, nwarps, lane);
    else sparse_gram_warp<8>(xs, sx, ys, mb, mw, n, nf, s, full, lists, Smax, lam_n, Gout, warp, nwarps, lane);
}

// ---------------------------------------------------------------------------
// Warp-owned variant: the calling warp owns columns c = c_first + j * c_step
// (j < n_cols) and has already built their kept-row lists.  Columns are
// processed in rounds of CT (power of two, CT * LPC <= 32); q-groups QG split
// each list round-robin and are reduced with shuffles in a fixed order.
// ---------------------------------------------------------------------------
template <int CPL>
__device__ __forceinline__ void sparse_gram_owned(uint32_t xs, int sx, uint32_t ys, int nf, int len, bool full,
                                                  uint32_t lists, int Smax, int c_first, int c_step, int n_cols,
                                                  float lam_n, float* __restrict__ Gout, int lane,
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
            float* grow = Gout + (size_t)c * gs;
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                const int ch = fl + i * LPC;
                if (ch < nq) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int f = 4 * ch + t;
                        if (f < nf) grow[f] = (accumulate ? grow[f] : 0.f) + acc[4 * i + t] + ((f == c) ? lam_n : 0.f);
                    }
                }
            }
            if (fl == 0) grow[nf] = (accumulate ? grow[nf] : 0.f) + accb;
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

template <int CPL>
struct OwnedAcc {
    float acc[4 * CPL];
    float accb;
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < 4 * CPL; ++i) acc[i] = 0.f;
        accb = 0.f;
    }
};

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

__device__ __forceinline__ void sparse_gram_owned_any(uint32_t xs, int sx, uint32_t ys, int nf, int len, bool full,
                                                      uint32_t lists, int Smax, int c_first, int c_step, int n_cols,
                                                      float lam_n, float* Gout, int lane) {
    const int nq = xs_chunks(nf);
    if (nq <= 4) sparse_gram_owned<1>(xs, sx, ys, nf, len, full, lists, Smax, c_first, c_step, n_cols, lam_n, Gout, lane);
    else if (nq <= 8) sparse_gram_owned<2>(xs, sx, ys, nf, len, full, lists, Smax, c_first, c_step, n_cols, lam_n, Gout, lane);
    else if (nq <= 16) sparse_gram_owned<4>(xs, sx, ys, nf, len, full, lists, Smax, c_first, c_step, n_cols, lam_n, Gout, lane);
    else sparse_gram_owned<8>(xs, sx, ys, nf, len, full, lists, Smax, c_first, c_step, n_cols, lam_n, Gout, lane);
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
