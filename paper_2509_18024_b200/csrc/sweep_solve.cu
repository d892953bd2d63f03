// sweep_solve.cu -- phase B of a half-sweep: solve a batch of sketched normal
// equations written by phase A in fp32 registers (LU with partial pivoting for
// sketched rows, SPD elimination for complete sketches; core.py:120-131,
// als.py:184-205), write the new factor rows (als.py:286) and their penalty
// terms n_i*|w_i|^2 (als.py:162-167).  A breakdown or an ill-conditioned system
// is deferred to the float64 refinement (sweep_refine.cu), which owns the
// reference's plain-then-jittered retry semantics.
#include "solve.cuh"
#include "sweep_common.cuh"

namespace cals {

// 32/NFP systems per warp (nf <= 32): segmented register LU.
template <int NFP>
__global__ void __launch_bounds__(256, 3) solve_warp_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                         int64_t n_list) {
    const int lane = threadIdx.x & 31;
    const int nf = A.nf, gs = nf + 1;
    constexpr int SPW = 32 / NFP;  // systems per warp
    const int seg = lane / NFP, r = lane % NFP;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b0 = gw * SPW; b0 < n_list; b0 += stride * SPW) {
        const int64_t li = b0 + seg;
        const bool sv = li < n_list;
        const int row = sv ? rows[li] : 0;
        const int n = sv ? (int)(A.ptr[row + 1] - A.ptr[row]) : 1;
        const bool spd = sv && A.budget[row] >= n;
        const double* G = A.gbuf + (size_t)(sv ? li : 0) * nf * gs;
        float x;
        const bool bad = seg_lu_solve<NFP>(G + (size_t)(r < nf ? r : 0) * gs, nf, spd, A.ill_ratio, sv, x, lane);
        // fp32 breakdown or ill-conditioning: the float64 refinement owns the row
        const bool deferred = bad && sv;
        if (deferred && r == 0) defer_refine(A, row, li);
        const int st = CALS_ROW_OK;
        if (sv && !deferred && r < nf) A.tgt[(int64_t)row * A.ld_tgt + r] = x;
        if (A.pen_rows != nullptr) {
            double p = (sv && r < nf) ? (double)x * (double)x : 0.0;
#pragma unroll
            for (int o = NFP / 2; o > 0; o >>= 1) p += __shfl_xor_sync(CALS_FULL_MASK, p, o, NFP);
            if (sv && !deferred && r == 0) A.pen_rows[row] = (double)n * p;
        }
        if (sv && !deferred && r == 0) {
            A.status[row] = st;
            report_status(A, row, st);
        }
    }
}

// One warp per system (32 < nf <= NF <= 64): wide register LU on a copy of
// the system staged (coalesced) into the warp's shared-memory slot.
template <int NF>
__global__ void __launch_bounds__(128, 3) solve_wide_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                          int64_t n_list) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nf = A.nf, gs = nf + 1, nout = nf * gs;
    float* W = reinterpret_cast<float*>(smem) + (size_t)warp * NF * (NF + 1);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t li = gw; li < n_list; li += stride) {
        const int row = rows[li];
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const bool spd = A.budget[row] >= n;
        const double* G = A.gbuf + (size_t)li * nout;
        __syncwarp();
        for (int e = lane; e < nout; e += 32) W[e] = (float)__ldcs(G + e);
        __syncwarp();
        float x0, x1;
        const int st = CALS_ROW_OK;
        if (wide_lu_solve<NF>(W, nf, spd, A.ill_ratio, x0, x1, lane)) {  // the float64 refinement owns the row
            if (lane == 0) defer_refine(A, row, li);
            continue;
        }
        float* out = A.tgt + (int64_t)row * A.ld_tgt;
        if (st != CALS_ROW_SINGULAR) {
            if (lane < nf) out[lane] = x0;
            if (lane + 32 < nf) out[lane + 32] = x1;
        }
        if (A.pen_rows != nullptr) {
            double p = (lane < nf ? (double)x0 * (double)x0 : 0.0) + (lane + 32 < nf ? (double)x1 * (double)x1 : 0.0);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(CALS_FULL_MASK, p, o);
            if (lane == 0) A.pen_rows[row] = (st == CALS_ROW_SINGULAR) ? 0.0 : (double)n * p;
        }
        if (lane == 0) {
            A.status[row] = st;
            report_status(A, row, st);
        }
    }
}

template __global__ void solve_wide_kernel<48>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_wide_kernel<64>(SweepArgs, const int32_t*, int64_t);

// One CTA of NF threads per system (64 < nf <= NF <= 128): thread r owns row r
// in registers (rows >= nf are identity rows with a zero right-hand side).
// Elimination in 16-column blocks with a runtime step inside each block (the
// column-K entry by a 16-way register select, as wide_block); per step the
// pivot is a CTA max-reduction of (|a[K]| bits | 127 - row) (ties to the
// smaller row, within 2^-17 relative, as wide_block), the pivot row is
// broadcast through shared memory, and every unused row is eliminated
// against it (no row swaps; back substitution walks the pivot order).
template <int NF, int B0>
__device__ __forceinline__ void rows_block(float (&a)[NF], float& rhs, bool& used, int& ord, float& mydiag,
                                           bool& fail, float& dmin, float& dmax, bool spd, int r, float* piv,
                                           uint32_t* wbest) {
    constexpr int BE = (B0 + 16 < NF) ? B0 + 16 : NF;
    const int lane = r & 31, warp = r >> 5;
#pragma unroll 1
    for (int K = B0; K < BE; ++K) {
        float ck = a[B0];
#pragma unroll
        for (int i = 1; i < BE - B0; ++i)
            if (K == B0 + i) ck = a[B0 + i];
        int p = K;
        if (!spd) {
            const uint32_t key = used ? (uint32_t)(127 - r) : ((__float_as_uint(ck) & 0x7FFFFF80u) | (uint32_t)(127 - r));
            const uint32_t wb = __reduce_max_sync(0xffffffffu, key);
            if (lane == 0) wbest[warp] = wb;
            __syncthreads();
            uint32_t best = wbest[0];
#pragma unroll
            for (int w = 1; w < NF / 32; ++w) best = wbest[w] > best ? wbest[w] : best;
            fail |= (best >> 7) == 0u;
            p = 127 - (int)(best & 127u);
        }
        if (r == p) {
            used = true;
            ord = K;
            mydiag = ck;
#pragma unroll
            for (int q = B0 / 4; q < NF / 4; ++q)
                *reinterpret_cast<float4*>(piv + 4 * q) = make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
            piv[NF] = rhs;
            piv[NF + 1] = ck;
        }
        __syncthreads();
        const float d = piv[NF + 1];
        fail |= spd ? !(d > 0.f) : !(d == d);
        dmin = fminf(dmin, fabsf(d));
        dmax = fmaxf(dmax, fabsf(d));
        const float f = used ? 0.f : ck * __frcp_rn(d);
#pragma unroll
        for (int q = B0 / 4; q < NF / 4; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(piv + 4 * q);
            ffma2_bcast(a[4 * q + 0], a[4 * q + 1], v.x, v.y, -f);
            ffma2_bcast(a[4 * q + 2], a[4 * q + 3], v.z, v.w, -f);
        }
        rhs = fmaf(-f, piv[NF], rhs);
        __syncthreads();  // piv is rewritten by the next step's owner
    }
}

// Back substitution for unknowns K in [B0, B0 + 16), descending.
template <int NF, int B0>
__device__ __forceinline__ void rows_back(const float (&a)[NF], float& rhs, int ord, float mydiag, int r, float* xs) {
    constexpr int BE = (B0 + 16 < NF) ? B0 + 16 : NF;
#pragma unroll 1
    for (int K = BE - 1; K >= B0; --K) {
        if (ord == K) xs[K] = rhs / mydiag;
        __syncthreads();
        const float xk = xs[K];
        float ak = a[B0];
#pragma unroll
        for (int i = 1; i < BE - B0; ++i)
            if (K == B0 + i) ak = a[B0 + i];
        if (ord >= 0 && ord < K) rhs = fmaf(-ak, xk, rhs);
    }
}

template <int NF, int... Q>
__device__ __forceinline__ void rows_eliminate(float (&a)[NF], float& rhs, bool& used, int& ord, float& mydiag,
                                               bool& fail, float& dmin, float& dmax, bool spd, int r, float* piv,
                                               uint32_t* wbest, std::integer_sequence<int, Q...>) {
    (rows_block<NF, 16 * Q>(a, rhs, used, ord, mydiag, fail, dmin, dmax, spd, r, piv, wbest), ...);
}
template <int NF, int... Q>
__device__ __forceinline__ void rows_substitute(const float (&a)[NF], float& rhs, int ord, float mydiag, int r,
                                                float* xs, std::integer_sequence<int, Q...>) {
    (rows_back<NF, NF - 16 - 16 * Q>(a, rhs, ord, mydiag, r, xs), ...);
}

template <int NF>
__global__ void __launch_bounds__(NF, 3) solve_rows_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                          int64_t n_list) {
    __shared__ __align__(16) float piv[NF + 4];
    __shared__ float xs[NF];
    __shared__ uint32_t wbest[NF / 32];
    __shared__ double red[32];
    __shared__ int s_bad;
    const int r = threadIdx.x;
    const int nf = A.nf, gs = nf + 1;
    for (int64_t li = blockIdx.x; li < n_list; li += gridDim.x) {
        const int row = rows[li];
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const bool spd = A.budget[row] >= n;
        const double* G = A.gbuf + (size_t)li * nf * gs;
        float a[NF];
#pragma unroll
        for (int j = 0; j < NF; ++j) a[j] = (r < nf && j < nf) ? (float)__ldcs(G + (size_t)r * gs + j) : (j == r ? 1.f : 0.f);
        float rhs = r < nf ? (float)__ldcs(G + (size_t)r * gs + nf) : 0.f;
        bool used = false, fail = false;
        int ord = -1;
        float mydiag = 1.f, dmin = INFINITY, dmax = 0.f;
        if (r == 0) s_bad = 0;
        rows_eliminate<NF>(a, rhs, used, ord, mydiag, fail, dmin, dmax, spd, r, piv, wbest,
                           std::make_integer_sequence<int, NF / 16>{});
        rows_substitute<NF>(a, rhs, ord, mydiag, r, xs, std::make_integer_sequence<int, NF / 16>{});
        __syncthreads();
        // unknown r (solved from the row pivoted at step r)
        float x = r < nf ? xs[r] : 0.f;
        const bool bad = fail || ill_conditioned(dmin, dmax, A.ill_ratio) || (r < nf && (!(x == x) || (x - x != 0.f)));
        if (bad) atomicOr(&s_bad, 1);
        __syncthreads();
        const int st = CALS_ROW_OK;
        if (s_bad) {  // the float64 refinement owns the row
            if (r == 0) defer_refine(A, row, li);
            __syncthreads();
            continue;
        }
        if (st != CALS_ROW_SINGULAR && r < nf) A.tgt[(int64_t)row * A.ld_tgt + r] = x;
        if (A.pen_rows != nullptr) {
            double p = (r < nf) ? (double)x * (double)x : 0.0;
            p = block_sum_d(p, red);
            if (r == 0) A.pen_rows[row] = (st == CALS_ROW_SINGULAR) ? 0.0 : (double)n * p;
        }
        if (r == 0) {
            A.status[row] = st;
            report_status(A, row, st);
        }
        __syncthreads();
    }
}

template __global__ void solve_rows_kernel<96>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_rows_kernel<128>(SweepArgs, const int32_t*, int64_t);

template __global__ void solve_warp_kernel<8>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_warp_kernel<16>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_warp_kernel<32>(SweepArgs, const int32_t*, int64_t);

}  // namespace cals
