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
        {
            // nf (nf + 1) is even and every slot starts 16-byte aligned: 16-byte streaming loads,
            // eight per lane in flight (the copy is latency-bound at 12 warps per SM otherwise)
            const double2* G2 = reinterpret_cast<const double2*>(G);
            float2* W2 = reinterpret_cast<float2*>(W);
            const int n2 = nout >> 1;
            int e = lane;
            for (; e + 32 * 7 < n2; e += 32 * 8) {
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldcs(G2 + e + 32 * u);
#pragma unroll
                for (int u = 0; u < 8; ++u) W2[e + 32 * u] = make_float2((float)v[u].x, (float)v[u].y);
            }
            for (; e < n2; e += 32) {
                const double2 v = __ldcs(G2 + e);
                W2[e] = make_float2((float)v.x, (float)v.y);
            }
        }
        __syncwarp();
        float x0, x1;
        const int st = CALS_ROW_OK;
        if (wide_lu_solve<NF>(W, nf, spd, A.ill_ratio, x0, x1, lane)) {  // the float64 refinement owns the row
            if (lane == 0) {
                if (A.ir_list != nullptr) defer_ir(A, row, li);  // mixed-precision solve first (sweep_solve_ir.cu)
                else defer_refine(A, row, li);
            }
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

template __global__ void solve_warp_kernel<8>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_warp_kernel<16>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_warp_kernel<32>(SweepArgs, const int32_t*, int64_t);

}  // namespace cals
