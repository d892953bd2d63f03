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
//   big_gram     masked partial Gram per item (fixed-order partials), plus the
//                item's share of the fused residual of the previous row
//   big_reduce   fixed-order fp64 sum of the partials, + lam*n*I -> normal
//                equations for the batched solve (sweep_solve.cu)
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

__global__ void __launch_bounds__(kThreads) big_scan_kernel(SweepArgs A, BigArgs B) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_above[CALS_MAX_NF_DEV], s_in[CALS_MAX_NF_DEV], s_base[CALS_MAX_NF_DEV],
        s_slot[CALS_MAX_NF_DEV];
    __shared__ uint32_t s_hib[CALS_MAX_NF_DEV], s_lob[CALS_MAX_NF_DEV];
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x;
    const int sx = xs_stride(nf);
    float* Xs = reinterpret_cast<float*>(smem);
    const FastDiv fq((uint32_t)xs_chunks(nf));
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
            stage_slice(A, lo, k0, kn, Xs, nullptr, fq);
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
    __shared__ float wold[CALS_MAX_NF_DEV];
    __shared__ double red[32];
    const int nf = A.nf, tid = threadIdx.x, nt = blockDim.x;
    const int sx = xs_stride(nf), mw = (nf + 31) / 32, gs = nf + 1;
    float* Xs = reinterpret_cast<float*>(smem);
    float* ys = reinterpret_cast<float*>(smem + align16((size_t)B.chunk * sx * 4));
    uint32_t* mb = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(ys) + align16((size_t)B.chunk * 4));
    float* G = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(mb) + align16((size_t)B.chunk * mw * 4));
    float* scratch = G + align16((size_t)nf * gs * 4) / 4;
    const FastDiv fq((uint32_t)xs_chunks(nf));
    for (int64_t t = blockIdx.x; t < B.n_tiles; t += gridDim.x) {
        const int r = find_row(B.tile_ptr, B.n_big, t);
        const int row = B.rows[r];
        const int64_t lo = A.ptr[row];
        const int n = (int)(A.ptr[row + 1] - lo);
        const bool full = A.budget[row] >= n;
        const int kbeg = (int)(t - B.tile_ptr[r]) * B.item_rows;
        const int kend = min(n, kbeg + B.item_rows);
        __syncthreads();
        if (tid < nf) {
            s_thr[tid] = B.thr[(size_t)r * nf + tid];
            if (A.tgt_old != nullptr) wold[tid] = A.tgt_old[(int64_t)row * A.ld_old + tid];
        }
        const int nout = nf * gs;
        bool first = true;
        double racc = 0.0;
        for (int k0 = kbeg; k0 < kend; k0 += B.chunk) {
            const int kn = min(B.chunk, kend - k0);
            __syncthreads();
            stage_slice(A, lo, k0, kn, Xs, ys, fq);
            __syncthreads();
            if (A.rss_rows != nullptr) {
                for (int k = tid; k < kn; k += nt) {
                    double pred = 0.0;
                    for (int f = 0; f < nf; ++f) pred = fma((double)Xs[k * sx + f], (double)wold[f], pred);
                    const double d = (double)ys[k] - pred;
                    racc = fma(d, d, racc);
                }
            }
            build_mask(Xs, sx, kn, nf, s_thr, full, mb, mw, k0);
            __syncthreads();
            tile_gram(Xs, sx, ys, mb, mw, kn, nf, G, scratch, !first);
            first = false;
        }
        float* out = B.part + (size_t)t * nout;
        for (int e = tid; e < nout; e += nt) out[e] = G[e];
        if (A.rss_rows != nullptr) {
            racc = block_sum_d(racc, red);
            if (tid == 0) B.rss_part[t] = racc;
        }
    }
}

// Big rows [r0, r0 + count): fixed-order float64 sum of the item partials,
// + lam*n*I on the diagonal -> A.gbuf slot (r - r0); residual partial sums.
__global__ void __launch_bounds__(kThreads) big_reduce_kernel(SweepArgs A, BigArgs B, int64_t r0, int64_t count) {
    const int nf = A.nf, gs = nf + 1, nout = nf * gs;
    for (int64_t q = blockIdx.x; q < count; q += gridDim.x) {
        const int64_t r = r0 + q;
        const int row = B.rows[r];
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const int64_t t0 = B.tile_ptr[r], t1 = B.tile_ptr[r + 1];
        const float lam_n = (float)(A.lam * (double)n);
        float* G = A.gbuf + (size_t)q * nout;
        for (int e = threadIdx.x; e < nout; e += blockDim.x) {
            double v = 0.0;
            for (int64_t t = t0; t < t1; ++t) v += (double)B.part[(size_t)t * nout + e];
            const int c = e / gs, f = e - c * gs;
            G[e] = (float)v + ((c == f) ? lam_n : 0.f);
        }
        if (A.rss_rows != nullptr && threadIdx.x == 0) {
            double v = 0.0;
            for (int64_t t = t0; t < t1; ++t) v += B.rss_part[t];
            A.rss_rows[row] = v;
        }
    }
}

}  // namespace cals
