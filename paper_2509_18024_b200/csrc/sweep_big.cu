// sweep_big.cu -- the tiled tier of the half-sweep: regressions whose slice
// does not fit in shared memory (the reference's long rows, which it handles
// with the presort walk, core.py:167-170,209-213).
//
// A big row is cut into work items of `item_rows` slice rows, processed in
// shared-memory chunks.  Per half-sweep:
//   big_scan     counts per column above / inside the table bracket and
//                appends the bracket's keys to a per-(row, column) list
//   big_resolve  one warp per (row, column): exact s-th key from the list
//                (warp sample-select), or from the whole column if the
//                bracket missed (fallback, always correct)
//   big_gram     masked partial Gram per item (fixed-order partials)
//   big_solve    fixed-order fp64 sum of the partials, + lam*n*I, LU / SPD
//   big_rss      fused residual of the new row (item side)
#include "gram.cuh"
#include "select.cuh"
#include "solve.cuh"
#include "sweep_common.cuh"

namespace cals {


__device__ __forceinline__ int find_row(const int64_t* tile_ptr, int64_t n_big, int64_t t) {
    int64_t lo = 0, hi = n_big - 1;  // largest r with tile_ptr[r] <= t
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (tile_ptr[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return (int)lo;
}

// Stage slice rows [k0, k0+kn) of the row starting at rating `lo` into Xs.
__device__ __forceinline__ void stage_chunk(const SweepArgs& A, int64_t lo, int k0, int kn, float* Xs, int sx,
                                            const FastDiv& fdiv, bool with_y) {
    const int nf = A.nf, nt = blockDim.x;
    const int nel = kn * nf;
#pragma unroll 4
    for (int e = threadIdx.x; e < nel; e += nt) {
        const int k = (int)fdiv.div((uint32_t)e);
        const int c = e - k * nf;
        Xs[k * sx + c] = __ldg(A.src + (int64_t)__ldg(A.idx + lo + k0 + k) * A.ld_src + c);
    }
    if (with_y) {
        for (int k = threadIdx.x; k < kn; k += nt) {
            Xs[k * sx + nf] = __ldg(A.val + lo + k0 + k);
            for (int c = nf + 1; c < sx; ++c) Xs[k * sx + c] = 0.f;
        }
    }
}

__global__ void __launch_bounds__(kThreads) big_scan_kernel(SweepArgs A, BigArgs B) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_above[CALS_MAX_NF_DEV], s_in[CALS_MAX_NF_DEV], s_base[CALS_MAX_NF_DEV],
        s_slot[CALS_MAX_NF_DEV];
    __shared__ uint32_t s_hib[CALS_MAX_NF_DEV], s_lob[CALS_MAX_NF_DEV];
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x;
    const int sx = xs_stride(nf);
    float* Xs = reinterpret_cast<float*>(smem);
    const FastDiv fdiv((uint32_t)nf);
    for (int64_t t = blockIdx.x; t < B.n_tiles; t += gridDim.x) {
        const int r = find_row(B.tile_ptr, B.n_big, t);
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        if (s >= n) continue;  // complete sketch: nothing to select (uniform per block)
        const int kbeg = (int)(t - B.tile_ptr[r]) * B.item_rows;
        const int kend = min(n, kbeg + B.item_rows);
        if (tid < nf) {
            uint32_t hib, lob;
            table_bracket(A.qtab + (size_t)tid * (kQ + 1), n, s, A.delta_tab, hib, lob);
            s_hib[tid] = hib;
            s_lob[tid] = lob;
            s_above[tid] = 0;
            s_in[tid] = 0;
        }
        const int64_t cbase = B.cand_ptr[r];
        const int capB = (int)((B.cand_ptr[r + 1] - cbase) / nf);
        for (int k0 = kbeg; k0 < kend; k0 += B.chunk) {
            const int kn = min(B.chunk, kend - k0);
            __syncthreads();
            stage_chunk(A, lo, k0, kn, Xs, sx, fdiv, false);
            if (tid < nf) s_slot[tid] = 0;
            __syncthreads();
            const int per = nt / nf;
            int my_in = 0, my_above = 0;
            const int c = tid % nf, j = tid / nf;
            if (tid < per * nf) {
                const uint32_t hib = s_hib[c], lob = s_lob[c];
                for (int k = j; k < kn; k += per) {
                    const uint32_t a = abs_bits(Xs[k * sx + c]);
                    my_above += (a >= hib);
                    my_in += (a >= lob && a < hib);
                }
                atomicAdd(&s_above[c], my_above);
                if (my_in) atomicAdd(&s_slot[c], my_in);
            }
            __syncthreads();
            if (tid < nf) {
                const int cnt_c = s_slot[tid];
                s_base[tid] = cnt_c ? atomicAdd(&B.cnt[((size_t)r * nf + tid) * 2 + 1], cnt_c) : 0;
                s_slot[tid] = 0;
            }
            __syncthreads();
            if (tid < per * nf && my_in) {
                const uint32_t hib = s_hib[c], lob = s_lob[c];
                uint64_t* cl = B.cand + cbase + (int64_t)c * capB;
                for (int k = j; k < kn; k += per) {
                    const float x = Xs[k * sx + c];
                    const uint32_t a = abs_bits(x);
                    if (a >= lob && a < hib) {
                        const int pos = s_base[c] + atomicAdd(&s_slot[c], 1);
                        if (pos < capB) cl[pos] = make_key(x, (uint32_t)(k0 + k));
                    }
                }
            }
        }
        __syncthreads();
        if (tid < nf && s_above[tid]) atomicAdd(&B.cnt[((size_t)r * nf + tid) * 2], s_above[tid]);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) big_resolve_kernel(SweepArgs A, BigArgs B) {
    const int nf = A.nf;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwork = B.n_big * nf;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = gw; w < nwork; w += wstride) {
        const int r = (int)(w / nf), c = (int)(w % nf);
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int s = A.budget[row];
        const float* src = A.src;
        const int32_t* idx = A.idx + lo;
        const int ld = A.ld_src;
        auto keyat = [src, idx, ld, c](int k) {
            return make_key(__ldg(src + (int64_t)__ldg(idx + k) * ld + c), (uint32_t)k);
        };
        uint64_t T;
        if (s >= n) {
            uint64_t mn = ~0ull;
            if (A.thr_keys != nullptr) {
                for (int k = lane; k < n; k += 32) {
                    uint64_t kk = keyat(k);
                    mn = kk < mn ? kk : mn;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    uint64_t t2 = __shfl_xor_sync(CALS_FULL_MASK, mn, o);
                    mn = t2 < mn ? t2 : mn;
                }
            }
            T = (A.thr_keys != nullptr) ? mn : 0ull;
        } else {
            const int above = B.cnt[((size_t)r * nf + c) * 2];
            const int in = B.cnt[((size_t)r * nf + c) * 2 + 1];
            const int64_t cbase = B.cand_ptr[r];
            const int capB = (int)((B.cand_ptr[r + 1] - cbase) / nf);
            uint64_t* cl = B.cand + cbase + (int64_t)c * capB;
            uint32_t hib, lob;
            table_bracket(A.qtab + (size_t)c * (kQ + 1), n, s, A.delta_tab, hib, lob);
            const uint64_t hik = hi_key_of(hib), lok = (uint64_t)lob << 32;
            if (above < s && s <= above + in && in <= capB && lok < hik) {
                T = warp_select_keys(KeyList{cl}, in, s - above, lok, hik, lane);
            } else {
                uint64_t rlo, rhi;
                int m, need;
                if (above >= s) { rlo = hik; rhi = ~0ull; m = above; need = s; }
                else if (above + in < s) { rlo = 0ull; rhi = lok; m = n - above - in; need = s - above - in; }
                else { rlo = lok; rhi = hik; m = in; need = s - above; }
                T = warp_select_column(keyat, n, m, need, rlo, rhi, cl, capB, lane);
            }
        }
        if (lane == 0) {
            B.thr[(size_t)r * nf + c] = T;
            if (A.thr_keys != nullptr) A.thr_keys[(int64_t)row * nf + c] = T;
        }
    }
}

__global__ void __launch_bounds__(kThreads) big_gram_kernel(SweepArgs A, BigArgs B) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t s_thr[CALS_MAX_NF_DEV];
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x;
    const int sx = xs_stride(nf), mw = (nf + 31) / 32, gs = nf + 1;
    float* Xs = reinterpret_cast<float*>(smem);
    uint32_t* mb = reinterpret_cast<uint32_t*>(smem + align16((size_t)B.chunk * sx * 4));
    float* G = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(mb) + align16((size_t)B.chunk * mw * 4));
    float* scratch = G + align16((size_t)nf * gs * 4) / 4;
    const FastDiv fdiv((uint32_t)nf);
    for (int64_t t = blockIdx.x; t < B.n_tiles; t += gridDim.x) {
        const int r = find_row(B.tile_ptr, B.n_big, t);
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const bool full = A.budget[row] >= n;
        const int kbeg = (int)(t - B.tile_ptr[r]) * B.item_rows;
        const int kend = min(n, kbeg + B.item_rows);
        __syncthreads();
        if (tid < nf) s_thr[tid] = B.thr[(size_t)r * nf + tid];
        const int nout = nf * gs;
        bool first = true;
        for (int k0 = kbeg; k0 < kend; k0 += B.chunk) {
            const int kn = min(B.chunk, kend - k0);
            __syncthreads();
            stage_chunk(A, lo, k0, kn, Xs, sx, fdiv, true);
            __syncthreads();
            // mask with slice-row ids relative to the whole row (keys carry them)
            for (int e = tid; e < kn * mw; e += nt) {
                const int k = e / mw, w = e - k * mw;
                const int cb = w * 32, ce = min(nf, cb + 32);
                uint32_t bits = 0;
                if (full) bits = (ce - cb == 32) ? 0xffffffffu : ((1u << (ce - cb)) - 1u);
                else
                    for (int c = cb; c < ce; ++c)
                        if (make_key(Xs[k * sx + c], (uint32_t)(k0 + k)) >= s_thr[c]) bits |= 1u << (c - cb);
                mb[e] = bits;
            }
            __syncthreads();
            tile_gram(Xs, sx, mb, mw, kn, nf, G, scratch, !first);
            first = false;
        }
        float* out = B.part + (size_t)t * nout;
        for (int e = tid; e < nout; e += nt) out[e] = G[e];
    }
}

template <int NFP>
__global__ void __launch_bounds__(kThreads) big_solve_kernel(SweepArgs A, BigArgs B) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ float wv[CALS_MAX_NF_DEV];
    __shared__ int s_piv[1], s_stat[1];
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int gs = nf + 1, nout = nf * gs;
    float* G = reinterpret_cast<float*>(smem);
    float* W = G + align16((size_t)nout * 4) / 4;
    for (int64_t r = blockIdx.x; r < B.n_big; r += gridDim.x) {
        const int row = B.rows[r];
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const bool full = A.budget[row] >= n;
        const int64_t t0 = B.tile_ptr[r], t1 = B.tile_ptr[r + 1];
        const float lam_n = (float)(A.lam * (double)n);
        __syncthreads();
        for (int e = tid; e < nout; e += nt) {
            double v = 0.0;
            for (int64_t t = t0; t < t1; ++t) v += (double)B.part[(size_t)t * nout + e];
            const int c = e / gs, f = e - c * gs;
            G[e] = (float)v + ((c == f) ? lam_n : 0.f);
        }
        __syncthreads();
        const int st = solve_row<NFP>(G, nf, full, wv, W, A.retry_ws + (size_t)blockIdx.x * A.retry_stride, s_piv,
                                      s_stat);
        for (int f = tid; f < nf; f += nt) {
            if (st != CALS_ROW_SINGULAR) A.tgt[(int64_t)row * A.ld_tgt + f] = wv[f];
            B.wbig[(size_t)r * nf + f] = wv[f];
        }
        if (tid == 0) { A.status[row] = st; report_status(A, row, st); }
    }
}

__global__ void __launch_bounds__(kThreads) big_rss_kernel(SweepArgs A, BigArgs B) {
    __shared__ double red[32];
    __shared__ float w[CALS_MAX_NF_DEV];
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x;
    for (int64_t t = blockIdx.x; t < B.n_tiles; t += gridDim.x) {
        const int r = find_row(B.tile_ptr, B.n_big, t);
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const int kbeg = (int)(t - B.tile_ptr[r]) * B.item_rows;
        const int kend = min(n, kbeg + B.item_rows);
        __syncthreads();
        for (int f = tid; f < nf; f += nt) w[f] = B.wbig[(size_t)r * nf + f];
        __syncthreads();
        double acc = 0.0;
        for (int k = kbeg + tid; k < kend; k += nt) {
            const float* xr = A.src + (int64_t)__ldg(A.idx + lo + k) * A.ld_src;
            double pred = 0.0;
            for (int f = 0; f < nf; ++f) pred = fma((double)__ldg(xr + f), (double)w[f], pred);
            const double d = (double)__ldg(A.val + lo + k) - pred;
            acc = fma(d, d, acc);
        }
        acc = block_sum_d(acc, red);
        if (tid == 0) B.rss_part[t] = acc;
    }
}

__global__ void big_rss_reduce_kernel(SweepArgs A, BigArgs B) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < B.n_big; r += (int64_t)gridDim.x * blockDim.x) {
        const int row = B.rows[r];
        double v = 0.0;
        for (int64_t t = B.tile_ptr[r]; t < B.tile_ptr[r + 1]; ++t) v += B.rss_part[t];
        A.rss_rows[row] = (A.status[row] == CALS_ROW_SINGULAR) ? 0.0 : v;
    }
}

template __global__ void big_solve_kernel<8>(SweepArgs, BigArgs);
template __global__ void big_solve_kernel<16>(SweepArgs, BigArgs);
template __global__ void big_solve_kernel<32>(SweepArgs, BigArgs);
template __global__ void big_solve_kernel<0>(SweepArgs, BigArgs);

}  // namespace cals
