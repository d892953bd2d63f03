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

// Must be called by all threads of the block.  Xs: n rows, stride sx
// (y in column nf, zero padding up to sx).  mb: n * mw mask words.
// Writes (or adds into) G (nf x (nf+1), row stride nf+1).  scratch: >= blockDim*16 floats.
__device__ void tile_gram(const float* __restrict__ Xs, int sx, const uint32_t* __restrict__ mb, int mw,
                          int n, int nf, float* __restrict__ G, float* __restrict__ scratch,
                          bool accumulate = false) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int RB = (nf + 3) >> 2, CB = sx >> 2, NB = RB * CB;
    const int gs = nf + 1;
    if (NB <= nt) {
        const int KG = nt / NB;
        if (tid < NB * KG) {
            const int bid = tid % NB, kg = tid / NB;
            const int c0 = (bid / CB) * 4, f0 = (bid % CB) * 4;
            const int wsel = c0 >> 5, sh = c0 & 31;
            float acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 4
            for (int k = kg; k < n; k += KG) {
                const float4 av = *reinterpret_cast<const float4*>(Xs + (size_t)k * sx + c0);
                const float4 bv = *reinterpret_cast<const float4*>(Xs + (size_t)k * sx + f0);
                const uint32_t m = mb[k * mw + wsel] >> sh;
                const float a0 = (m & 1u) ? av.x : 0.f;
                const float a1 = (m & 2u) ? av.y : 0.f;
                const float a2 = (m & 4u) ? av.z : 0.f;
                const float a3 = (m & 8u) ? av.w : 0.f;
                const float a[4] = {a0, a1, a2, a3};
                const float b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
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
            const int wsel = c0 >> 5, sh = c0 & 31;
            float acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
            for (int k = 0; k < n; ++k) {
                const float4 av = *reinterpret_cast<const float4*>(Xs + (size_t)k * sx + c0);
                const float4 bv = *reinterpret_cast<const float4*>(Xs + (size_t)k * sx + f0);
                const uint32_t m = mb[k * mw + wsel] >> sh;
                const float a[4] = {(m & 1u) ? av.x : 0.f, (m & 2u) ? av.y : 0.f, (m & 4u) ? av.z : 0.f,
                                    (m & 8u) ? av.w : 0.f};
                const float b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
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

// Selection bitmap: bit c of mb[k*mw + c/32] = (key(k, c) >= thr[c]).
__device__ void build_mask(const float* __restrict__ Xs, int sx, int n, int nf, const uint64_t* thr,
                           bool full, uint32_t* __restrict__ mb, int mw) {
    for (int e = threadIdx.x; e < n * mw; e += blockDim.x) {
        const int k = e / mw, w = e - k * mw;
        const int cbeg = w * 32, cend = min(nf, cbeg + 32);
        uint32_t bits = 0;
        if (full) {
            bits = (cend - cbeg == 32) ? 0xffffffffu : ((1u << (cend - cbeg)) - 1u);
        } else {
            for (int c = cbeg; c < cend; ++c)
                if (make_key(Xs[(size_t)k * sx + c], (uint32_t)k) >= thr[c]) bits |= 1u << (c - cbeg);
        }
        mb[e] = bits;
    }
}

}  // namespace cals
