// solve.cuh -- small dense solves for the sketched normal equations.
//
// The sketched Gram X*^T X + lam*n*I is NOT symmetric (only one factor is
// sketched, core.py:7-14), so it is solved by LU with partial pivoting, as
// the reference does with LAPACK gesv (_kernels.py:233-236).  Rows whose
// sketch is complete (s == n) take the exact SPD ridge path (core.py:206-207,
// als.py:184-205): elimination without pivoting, failing on a non-positive
// pivot exactly where Cholesky fails.  A failure (or an ill-conditioned
// system) is re-solved in float64 with the reference's single jitter retry
// (+1e-10 * tr(G)/n_f on the diagonal, core.py:126-131) by sweep_refine.cu;
// block_lu_solve below serves the public single-row update (misc.cu).
//
// Input: augmented matrix G[r * gs + j], j < nf the Gram, j == nf the RHS.
#pragma once
#include <utility>

#include "common.cuh"

namespace cals {

// Block-wide LU (nf <= 128) in shared memory, in place on W (stride nf+1),
// working copy of G (cals_update_core).  All threads of the block must call it.  Returns 0/1.
template <typename T>
__device__ int block_lu_solve(T* W, int nf, bool spd, T* x_out, int* s_piv) {
    const int gs = nf + 1;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5;
    for (int k = 0; k < nf; ++k) {
        if (warp == 0) {
            int p = k;
            T best = (T)-1;
            if (!spd) {
                for (int r = k + lane; r < nf; r += 32) {
                    T v = W[r * gs + k];
                    v = v < 0 ? -v : v;
                    if (v > best) { best = v; p = r; }
                }
                int bi = (best >= 0) ? p : 0x7fffffff;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    T ob = __shfl_xor_sync(CALS_FULL_MASK, best, o);
                    int oi = __shfl_xor_sync(CALS_FULL_MASK, bi, o);
                    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
                }
                p = bi;
                if (lane == 0) s_piv[0] = (best > (T)0) ? p : -1;
            } else {
                T d = W[k * gs + k];
                if (lane == 0) s_piv[0] = (d > (T)0) ? k : -1;
            }
        }
        __syncthreads();
        int p = s_piv[0];
        if (p < 0) return 1;
        if (p != k) {
            for (int j = tid; j < gs; j += nt) {
                T t = W[k * gs + j];
                W[k * gs + j] = W[p * gs + j];
                W[p * gs + j] = t;
            }
            __syncthreads();
        }
        T d = W[k * gs + k];
        int rows = nf - k - 1, cols = nf - k;  // trailing rows, columns k+1..nf (incl. RHS)
        for (int e = tid; e < rows * cols; e += nt) {
            int r = k + 1 + e / cols;
            int j = k + 1 + e % cols;
            W[r * gs + j] -= (W[r * gs + k] / d) * W[k * gs + j];
        }
        __syncthreads();
    }
    if (warp == 0) {
        for (int r = nf - 1; r >= 0; --r) {
            T acc = 0;
            for (int j = r + 1 + lane; j < nf; j += 32) acc += W[r * gs + j] * x_out[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(CALS_FULL_MASK, acc, o);
            if (lane == 0) x_out[r] = (W[r * gs + nf] - acc) / W[r * gs + r];
            __syncwarp();
        }
    }
    __syncthreads();
    int bad = 0;
    for (int j = tid; j < nf; j += nt) {
        T v = x_out[j];
        if (!(v == v) || (v - v != 0)) bad = 1;
    }
    return __syncthreads_or(bad);
}

// Segmented warp LU: 32/NFP systems per warp, NFP lanes per system (lane r of
// a segment owns row r).  Partial pivoting without physical row swaps: the
// pivot row of step k is broadcast once and every unused row is eliminated
// against it; back substitution walks the pivot order.  Same arithmetic as
// row-swapping LU (first max |a| wins ties, like LAPACK idamax).
// fp32 elimination accuracy guard: the fp32 LU's error grows like the system's
// condition number (measured: ~6e-9 * cond), and the factor contract is 1e-4
// relative to the reference's float64 solve.  A spread of pivot magnitudes
// beyond the rank's ratio (a lower bound on cond) sends the system to the float64
// refinement (sweep_refine.cu: plain float64 first, the reference's jitter
// only if that is singular too), exactly like an fp32 breakdown.
// Ratio by rank (the fp32 elimination's error also grows with n_f): 100 up to
// n_f = 20, then 2000 / n_f (31 at 64); set per half-sweep (ill_ratio_for).
// Measured on the 500M config at a later iteration (tools/ill_diag.py).  Above
// n_f = 64 the fp32 LU is skipped (defer_all_kernel): 97 % of the wide config's
// systems exceeded any useful ratio.
__host__ inline float ill_ratio_for(int nf) {
    return nf <= 20 ? 100.0f : (nf <= 64 ? 2000.0f / (float)nf : 1000.0f / (float)nf);
}
__device__ __forceinline__ bool ill_conditioned(float dmin, float dmax, float ratio) { return dmax > ratio * dmin; }

// Returns, per lane, whether ITS system failed (uniform within a segment);
// x: the lane's unknown (variable r of its system).
template <int NFP>
__device__ __forceinline__ bool seg_lu_solve(const double* __restrict__ Grow, int nf, bool spd, float ill_ratio, bool seg_valid,
                                             float& x, int lane) {
    const int r = lane & (NFP - 1);
    const bool rv = seg_valid && r < nf;
    float a[NFP];
    float rhs = 0.f;
#pragma unroll
    for (int j = 0; j < NFP; ++j) a[j] = (rv && j < nf) ? (float)Grow[j] : 0.f;
    if (rv) rhs = (float)Grow[nf];
    bool used = !rv;
    int ord = -1;
    bool fail = !seg_valid;
    float dmin = INFINITY, dmax = 0.f;  // pivot magnitudes: their spread flags ill-conditioning
#pragma unroll
    for (int k = 0; k < NFP; ++k) {
        if (k < nf) {
            // argmax over the segment's unused rows (all lanes shuffle: spd differs per segment)
            float best = used ? -1.f : fabsf(a[k]);
            int bi = r;
#pragma unroll
            for (int o = NFP / 2; o > 0; o >>= 1) {
                const float ob = __shfl_xor_sync(CALS_FULL_MASK, best, o, NFP);
                const int oi = __shfl_xor_sync(CALS_FULL_MASK, bi, o, NFP);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            const int p = spd ? k : bi;
            if (!spd) fail |= !(best > 0.f);
            const float d = __shfl_sync(CALS_FULL_MASK, a[k], p, NFP);
            fail |= spd ? !(d > 0.f) : !(d == d);
            dmin = fminf(dmin, fabsf(d));
            dmax = fmaxf(dmax, fabsf(d));
            const bool me = (r == p);
            if (me) { used = true; ord = k; }
            const float f = (!used && !fail) ? a[k] / d : 0.f;
#pragma unroll
            for (int j = 0; j < NFP; ++j) {
                if (j > k && j < nf) {
                    const float vp = __shfl_sync(CALS_FULL_MASK, a[j], p, NFP);
                    a[j] = fmaf(-f, vp, a[j]);
                }
            }
            const float bp = __shfl_sync(CALS_FULL_MASK, rhs, p, NFP);
            rhs = fmaf(-f, bp, rhs);
        }
    }
    x = 0.f;
    const int seg_base = lane & ~(NFP - 1);
#pragma unroll
    for (int k = NFP - 1; k >= 0; --k) {
        if (k < nf) {
            const uint32_t bal = __ballot_sync(CALS_FULL_MASK, ord == k);
            const uint32_t segbits = (NFP == 32) ? bal : ((bal >> seg_base) & ((1u << NFP) - 1u));
            const int pk = segbits ? (__ffs(segbits) - 1) : 0;
            float xk = (ord == k) ? rhs / a[k] : 0.f;
            xk = __shfl_sync(CALS_FULL_MASK, xk, pk, NFP);
            if (r == k) x = xk;
            if (ord >= 0 && ord < k) rhs = fmaf(-a[k], xk, rhs);
        }
    }
    const bool bad = rv && (!(x == x) || (x - x != 0.f));
    const uint32_t anybad = __ballot_sync(CALS_FULL_MASK, bad);
    const uint32_t segm = (NFP == 32) ? 0xffffffffu : (((1u << NFP) - 1u) << seg_base);
    return fail || ill_conditioned(dmin, dmax, ill_ratio) || (anybad & segm) != 0;
}

// Wide warp LU (32 < nf <= NF <= 64): lane owns rows `lane` and `lane + 32`
// of ONE system in registers; same no-swap partial pivoting and pivot-order
// back substitution as seg_lu_solve.  W: the augmented system (stride nf+1,
// any memory space).  Returns whether the system failed (warp-uniform); lane
// l ends with x0 = unknown l and x1 = unknown l + 32.
// Register select that keeps both operands in registers (a plain ?: between
// two register arrays can be rewritten as a pointer select into local memory).
__device__ __forceinline__ float sel_f32(bool hi, float b, float a) {
    float r;
    asm("{\n .reg .pred p;\n setp.ne.u32 p, %3, 0;\n selp.f32 %0, %1, %2, p;\n}\n"
        : "=f"(r) : "f"(b), "f"(a), "r"((unsigned)hi));
    return r;
}

template <int NF>
struct WideLU {
    float a[NF], b[NF];
    float ra, rb;
    bool ua, ub, fail;
    int oa, ob;
    float dmin, dmax;
    int nf;
};

// Elimination steps K in [B0, B0 + 16) (a runtime loop: the fully unrolled
// elimination is ~20k instructions and thrashes the instruction cache).  The
// column-K entries come from a 16-way register select; the update sweeps
// columns j >= B0 (compile-time), which also rewrites the block's columns
// left of K in still-unused rows -- entries no later step or the back
// substitution reads -- and leaves used rows alone (zero multiplier).
template <int NF, int B0>
__device__ __forceinline__ void wide_block(WideLU<NF>& S, bool spd, int lane) {
    constexpr int BE = (B0 + 16 < NF) ? B0 + 16 : NF;
    const int r0 = lane, r1 = lane + 32;
#pragma unroll 1
    for (int K = B0; K < BE; ++K) {
        float ca = S.a[B0], cb = S.b[B0];
#pragma unroll
        for (int i = 1; i < BE - B0; ++i) {
            if (K == B0 + i) {
                ca = S.a[B0 + i];
                cb = S.b[B0 + i];
            }
        }
        int p = K;
        if (!spd) {
            // one warp max-reduction of (|pivot| bits with the low 6 mantissa bits
            // replaced by 63 - row): largest magnitude, ties (to 2^-17 relative)
            // to the smallest row -- partial pivoting needs a large pivot, not the
            // exact maximum
            const uint32_t ka = S.ua ? (uint32_t)(63 - r0) : ((__float_as_uint(ca) & 0x7FFFFFC0u) | (uint32_t)(63 - r0));
            const uint32_t kb = S.ub ? (uint32_t)(63 - r1) : ((__float_as_uint(cb) & 0x7FFFFFC0u) | (uint32_t)(63 - r1));
            const uint32_t best = __reduce_max_sync(CALS_FULL_MASK, ka > kb ? ka : kb);
            S.fail |= (best >> 6) == 0u;
            p = 63 - (int)(best & 63u);
        }
        const bool hi = p >= 32;
        const int pl = p & 31;
        const float d = __shfl_sync(CALS_FULL_MASK, sel_f32(hi, cb, ca), pl);
        S.fail |= spd ? !(d > 0.f) : !(d == d);
        if (K < S.nf) {  // identity padding rows (K >= nf) pivot at 1.0: not a real pivot
            S.dmin = fminf(S.dmin, fabsf(d));
            S.dmax = fmaxf(S.dmax, fabsf(d));
        }
        if (lane == pl) {
            if (hi) { S.ub = true; S.ob = K; } else { S.ua = true; S.oa = K; }
        }
        const float inv = __frcp_rn(d);
        const float fa = S.ua ? 0.f : ca * inv;
        const float fb = S.ub ? 0.f : cb * inv;
#pragma unroll
        for (int j = B0; j < NF; ++j) {
            const float vp = __shfl_sync(CALS_FULL_MASK, sel_f32(hi, S.b[j], S.a[j]), pl);
            ffma2_bcast(S.a[j], S.b[j], -fa, -fb, vp);  // both rows in one FFMA2
        }
        const float bp = __shfl_sync(CALS_FULL_MASK, sel_f32(hi, S.rb, S.ra), pl);
        ffma2_bcast(S.ra, S.rb, -fa, -fb, bp);
    }
}

// Back-substitution step K (pivot order): unknown K from the row pivoted at step K.
template <int NF, int K>
__device__ __forceinline__ void wide_back(WideLU<NF>& S, float& x0, float& x1, int lane) {
    const uint32_t ba = __ballot_sync(CALS_FULL_MASK, S.oa == K);
    const uint32_t bb = __ballot_sync(CALS_FULL_MASK, S.ob == K);
    const int pl = ba ? __ffs(ba) - 1 : (bb ? __ffs(bb) - 1 : 0);
    float xk = (S.oa == K) ? S.ra / S.a[K] : 0.f;
    if (S.ob == K) xk = S.rb / S.b[K];
    xk = __shfl_sync(CALS_FULL_MASK, xk, pl);
    if (lane == (K & 31)) {
        if (K < 32) x0 = xk; else x1 = xk;
    }
    if (S.oa >= 0 && S.oa < K) S.ra = fmaf(-S.a[K], xk, S.ra);
    if (S.ob >= 0 && S.ob < K) S.rb = fmaf(-S.b[K], xk, S.rb);
}

template <int NF, int... Q>
__device__ __forceinline__ void wide_eliminate(WideLU<NF>& S, bool spd, int lane,
                                               std::integer_sequence<int, Q...>) {
    (wide_block<NF, 16 * Q>(S, spd, lane), ...);
}
template <int NF, int... K>
__device__ __forceinline__ void wide_substitute(WideLU<NF>& S, float& x0, float& x1, int lane,
                                                std::integer_sequence<int, K...>) {
    (wide_back<NF, NF - 1 - K>(S, x0, x1, lane), ...);
}

template <int NF>
__device__ __forceinline__ bool wide_lu_solve(const float* __restrict__ W, int nf, bool spd, float ill_ratio, float& x0, float& x1,
                                              int lane) {
    static_assert(NF > 32 && NF <= 64, "two rows per lane");
    const int gs = nf + 1;
    const int r0 = lane, r1 = lane + 32;
    const bool v0 = r0 < nf, v1 = r1 < nf;
    WideLU<NF> S;
    // rows >= nf are identity rows with a zero right-hand side: their steps
    // pivot on themselves and leave x = 0, so no step needs a bound check
#pragma unroll
    for (int j = 0; j < NF; ++j) {
        S.a[j] = (v0 && j < nf) ? W[r0 * gs + j] : (j == r0 ? 1.f : 0.f);
        S.b[j] = (v1 && j < nf) ? W[r1 * gs + j] : (j == r1 ? 1.f : 0.f);
    }
    S.ra = v0 ? W[r0 * gs + nf] : 0.f;
    S.rb = v1 ? W[r1 * gs + nf] : 0.f;
    S.ua = false;
    S.ub = false;
    S.oa = -1;
    S.ob = -1;
    S.fail = false;
    S.dmin = INFINITY;
    S.dmax = 0.f;
    S.nf = nf;
    wide_eliminate<NF>(S, spd, lane, std::make_integer_sequence<int, (NF + 15) / 16>{});
    x0 = 0.f;
    x1 = 0.f;
    wide_substitute<NF>(S, x0, x1, lane, std::make_integer_sequence<int, NF>{});
    const bool bad = (v0 && (!(x0 == x0) || (x0 - x0 != 0.f))) || (v1 && (!(x1 == x1) || (x1 - x1 != 0.f)));
    return S.fail || ill_conditioned(S.dmin, S.dmax, ill_ratio) || __any_sync(CALS_FULL_MASK, bad);
}

}  // namespace cals
