// sweep_solve.cu -- phase B of a half-sweep: solve a batch of sketched normal
// equations written by phase A, with the reference's failure semantics
// (LU with partial pivoting for sketched rows, SPD for complete sketches,
// one float64 jitter retry; core.py:120-131, als.py:184-205), write the new
// factor rows (als.py:286) and their penalty terms n_i*|w_i|^2 (als.py:162-167).
#include "solve.cuh"
#include "sweep_common.cuh"

namespace cals {

// One warp per system (nf <= 32).
template <int NFP>
__global__ void __launch_bounds__(256) solve_warp_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                         int64_t n_list) {
    __shared__ float xs[8][32];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int nf = A.nf, gs = nf + 1;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t li = gw; li < n_list; li += stride) {
        const int row = rows[li];
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const bool spd = A.budget[row] >= n;
        const float* G = A.gbuf + (size_t)li * nf * gs;
        float* x = xs[wl];
        int st = CALS_ROW_OK;
        if (warp_lu_solve<NFP>(G, gs, nf, spd, x, lane)) {
            double* W = A.retry_ws + (size_t)gw * A.retry_stride;
            double* xd = W + nf * gs;
            const int bad = warp_retry_f64(G, nf, spd, W, xd, lane);
            __syncwarp();
            if (lane < nf) x[lane] = (float)xd[lane];
            st = bad ? CALS_ROW_SINGULAR : CALS_ROW_JITTERED;
        }
        __syncwarp();
        const float w = lane < nf ? x[lane] : 0.f;
        if (st != CALS_ROW_SINGULAR && lane < nf) A.tgt[(int64_t)row * A.ld_tgt + lane] = w;
        if (A.pen_rows != nullptr) {
            double p = (double)w * (double)w;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(CALS_FULL_MASK, p, o);
            if (lane == 0) A.pen_rows[row] = (st == CALS_ROW_SINGULAR) ? 0.0 : (double)n * p;
        }
        if (lane == 0) {
            A.status[row] = st;
            report_status(A, row, st);
        }
        __syncwarp();
    }
}

// One CTA per system (nf > 32): LU in shared memory.
__global__ void __launch_bounds__(128) solve_block_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                          int64_t n_list) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ float wv[CALS_MAX_NF_DEV];
    __shared__ double red[32];
    __shared__ int s_piv[1], s_flag[1];
    const int nf = A.nf, gs = nf + 1, nout = nf * gs, tid = threadIdx.x;
    float* W = reinterpret_cast<float*>(smem);
    for (int64_t li = blockIdx.x; li < n_list; li += gridDim.x) {
        const int row = rows[li];
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const bool spd = A.budget[row] >= n;
        const float* G = A.gbuf + (size_t)li * nout;
        __syncthreads();
        for (int e = tid; e < nout; e += blockDim.x) W[e] = G[e];
        __syncthreads();
        int st = CALS_ROW_OK;
        if (block_lu_solve<float>(W, nf, spd, wv, s_piv)) {
            if (tid < 32) {
                double* Wd = A.retry_ws + (size_t)blockIdx.x * A.retry_stride;
                double* xd = Wd + nout;
                const int bad = warp_retry_f64(G, nf, spd, Wd, xd, tid);
                if (tid < 32) {
                    for (int f = tid; f < nf; f += 32) wv[f] = (float)xd[f];
                    if (tid == 0) s_flag[0] = bad ? CALS_ROW_SINGULAR : CALS_ROW_JITTERED;
                }
            }
            __syncthreads();
            st = s_flag[0];
        }
        if (st != CALS_ROW_SINGULAR)
            for (int f = tid; f < nf; f += blockDim.x) A.tgt[(int64_t)row * A.ld_tgt + f] = wv[f];
        if (A.pen_rows != nullptr) {
            double p = 0.0;
            for (int f = tid; f < nf; f += blockDim.x) p += (double)wv[f] * (double)wv[f];
            p = block_sum_d(p, red);
            if (tid == 0) A.pen_rows[row] = (st == CALS_ROW_SINGULAR) ? 0.0 : (double)n * p;
        }
        if (tid == 0) {
            A.status[row] = st;
            report_status(A, row, st);
        }
    }
}

template __global__ void solve_warp_kernel<8>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_warp_kernel<16>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_warp_kernel<32>(SweepArgs, const int32_t*, int64_t);

}  // namespace cals
