// sweep_refine.cu -- float64 solve of the normal equations the fp32 solve
// kernels cannot hold to the reference's float64 answer.
//
// The fp32 solve kernels defer a system here when its elimination breaks down
// (zero / non-finite pivot) or when the spread of its pivot magnitudes says it
// is ill-conditioned (ill_ratio_for, solve.cuh): the fp32 LU's error grows like
// cond * 6e-9 (measured), beyond the 1e-4 factor contract for cond >~ 1e4,
// while a float64 solve of the same (fp32-stored) normal equations stays at
// ~cond * 1e-9.  Like the reference (core.py:120-131, als.py:184-205): LU with
// partial pivoting (first largest pivot, as LAPACK's idamax) or, for a
// complete sketch, elimination without pivoting failing on a non-positive
// pivot (Cholesky's condition); on a breakdown the reference's jitter
// 1e-10 * tr(G) / n_f and one retry.  One CTA per deferred system, the
// system in shared memory as float64.
#include "solve.cuh"
#include "sweep_common.cuh"

namespace cals {

constexpr int kRfChunk = 64;       // slice rows staged per pass of the float64 Gram
constexpr int kRfSliceMax = 4096;  // rows up to this length rebuild their Gram in float64 from the slice

__host__ __device__ inline int refine_threads(int nf) { return 256; }
__host__ __device__ inline size_t refine_smem(int nf) {
    const size_t g = align16((size_t)nf * (nf + 1) * 8), bits = align16((size_t)nf * (kRfChunk / 32) * 4);
    const size_t simt = g + align16((size_t)kRfChunk * round_up4(nf) * 4) + align16(kRfChunk * 4) + bits;
    const size_t rb = g + align16((size_t)kRfChunk * (nf + 1) * 8) + bits;  // refine_rb_kernel (nf > 32)
    return nf > 32 ? rb : simt;
}

// Float64 Gram of one row from its slice: column c keeps the rows whose key
// reaches the row's selection threshold (all rows for a complete sketch);
// thread (c, fl) accumulates G[c][fl + j lpc] (f = nf: the right-hand side).
// Products of two fp32 values are exact in float64.
template <int NT>
__device__ __forceinline__ void refine_slice_gram(const SweepArgs& A, int row, int64_t lo, int n, bool full,
                                                  const uint64_t* s_thr, double* G, float* Xs, float* ys,
                                                  uint32_t* bits) {
    constexpr int kMaxAcc = NT == 256 ? 17 : 33;  // ceil((nf + 1) / lanes per column), lanes >= 4
    const int nf = A.nf, gs = nf + 1, tid = threadIdx.x;
    const int ldx = round_up4(nf), nq = xs_chunks(nf);
    const int lpc = NT / nf;
    const int c = tid / lpc, fl = tid - c * lpc;
    double acc[kMaxAcc];
#pragma unroll
    for (int j = 0; j < kMaxAcc; ++j) acc[j] = 0.0;
    for (int k0 = 0; k0 < n; k0 += kRfChunk) {
        const int kn = min(kRfChunk, n - k0);
        __syncthreads();  // previous chunk consumed
        for (int q = tid; q < kn * nq; q += NT) {
            const int k = q / nq, h = q - k * nq;
            *reinterpret_cast<float4*>(Xs + k * ldx + 4 * h) = __ldg(
                reinterpret_cast<const float4*>(A.src + (int64_t)__ldg(A.idx + lo + k0 + k) * A.ld_src + 4 * h));
        }
        for (int k = tid; k < kn; k += NT) ys[k] = __ldg(A.val + lo + k0 + k);
        __syncthreads();
        for (int q = tid; q < nf * (kRfChunk / 32); q += NT) {
            const int cc = q % nf, w = q / nf;
            uint32_t word = 0u;
            for (int b = 0; b < 32; ++b) {
                const int k = 32 * w + b;
                if (k < kn && (full || make_key(Xs[k * ldx + cc], (uint32_t)(k0 + k)) >= s_thr[cc])) word |= 1u << b;
            }
            bits[cc * (kRfChunk / 32) + w] = word;
        }
        __syncthreads();
        if (c < nf) {
            for (int w = 0; w < kRfChunk / 32; ++w) {
                uint32_t word = bits[c * (kRfChunk / 32) + w];
                while (word) {
                    const int k = 32 * w + __ffs(word) - 1;
                    word &= word - 1u;
                    const double xc = (double)Xs[k * ldx + c];
#pragma unroll
                    for (int j = 0; j < kMaxAcc; ++j) {
                        const int f = fl + j * lpc;
                        if (f < nf) acc[j] = fma(xc, (double)Xs[k * ldx + f], acc[j]);
                        else if (f == nf) acc[j] = fma(xc, (double)ys[k], acc[j]);
                    }
                }
            }
        }
    }
    if (c < nf) {
#pragma unroll
        for (int j = 0; j < kMaxAcc; ++j) {
            const int f = fl + j * lpc;
            if (f <= nf) G[c * gs + f] = acc[j] + ((f == c) ? A.lam * (double)n : 0.0);
        }
    }
}

// slice_ok: the rows' kept sets are per-row thresholds (method 'core'; fast_core
// rows use the stored normal equations, which hold its whole-source sketch).
// from_slice: the list holds rows (int32) that rebuild their Gram from the slice
// (method 'core', per-row thresholds); else (row << 32 | slot) entries solved
// from the stored normal equations.
template <int NT>
__global__ void __launch_bounds__(NT) refine_kernel(SweepArgs A, const int* __restrict__ count,
                                                   const void* __restrict__ list, int from_slice) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_x[CALS_MAX_NF_DEV];
    __shared__ double s_red[32];
    __shared__ int s_piv, s_bad;
    const int nf = A.nf, gs = nf + 1, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* G = reinterpret_cast<double*>(smem);
    float* Xs = reinterpret_cast<float*>(smem + align16((size_t)nf * gs * 8));
    float* ys = Xs + kRfChunk * round_up4(nf);
    uint32_t* bits = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(ys) + align16(kRfChunk * 4));
    __shared__ uint64_t s_thr[CALS_MAX_NF_DEV];
    const int n_list = *count;
    for (int64_t e = blockIdx.x; e < n_list; e += gridDim.x) {
        const int64_t ent = from_slice ? (int64_t)static_cast<const int32_t*>(list)[e] << 32
                                       : static_cast<const int64_t*>(list)[e];
        const int row = (int)(ent >> 32);
        const int64_t slot = (int64_t)(uint32_t)ent;
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const bool full = A.budget[row] >= n;
        const double* Gf = A.gbuf + (size_t)slot * nf * gs;
        // short rows rebuild their Gram in float64 (their fp32 sums are the error floor of an
        // ill-conditioned system); long rows' stored equations are float64-folded already
        __syncthreads();
        if (from_slice && tid < nf) s_thr[tid] = A.thr_keys[(int64_t)row * nf + tid];
        int st = CALS_ROW_SINGULAR;
        for (int attempt = 0; attempt < 2 && st == CALS_ROW_SINGULAR; ++attempt) {
            __syncthreads();
            if (from_slice) refine_slice_gram<NT>(A, row, A.ptr[row], n, full, s_thr, G, Xs, ys, bits);
            else
                for (int q = tid; q < nf * gs; q += NT) G[q] = Gf[q];
            __syncthreads();
            if (attempt == 1) {  // the reference's retry: G += 1e-10 * tr(G) / n_f * I (core.py:126-131)
                if (warp == 0) {
                    double tr = 0.0;
                    for (int i = lane; i < nf; i += 32) tr += G[i * gs + i];
                    tr = warp_sum_d(tr);
                    if (lane == 0) s_red[0] = 1e-10 * tr / (double)nf;
                }
                __syncthreads();
                for (int i = tid; i < nf; i += NT) G[i * gs + i] += s_red[0];
                __syncthreads();
            }
            if (tid == 0) s_bad = 0;
            // ---- float64 elimination on [G | b] ----
            for (int k = 0; k < nf; ++k) {
                if (warp == 0) {
                    int p = k;
                    if (!full) {
                        // first row of the largest |G[i][k]|, i >= k (idamax)
                        double best = -1.0;
                        int bi = nf;
                        for (int i = k + lane; i < nf; i += 32) {
                            const double v = fabs(G[i * gs + k]);
                            if (v > best) { best = v; bi = i; }
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const double ob = __shfl_xor_sync(CALS_FULL_MASK, best, o);
                            const int oi = __shfl_xor_sync(CALS_FULL_MASK, bi, o);
                            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
                        }
                        p = bi;
                        if (lane == 0 && !(best > 0.0)) s_bad = 1;
                    } else if (lane == 0 && !(G[k * gs + k] > 0.0)) {
                        s_bad = 1;
                    }
                    if (lane == 0) s_piv = p;
                }
                __syncthreads();
                if (s_bad) break;
                const int p = s_piv;
                if (p != k)
                    for (int j = tid; j < gs; j += NT) {
                        const double t = G[k * gs + j];
                        G[k * gs + j] = G[p * gs + j];
                        G[p * gs + j] = t;
                    }
                __syncthreads();
                const double d = G[k * gs + k];
                for (int i = k + 1 + tid; i < nf; i += NT) G[i * gs + k] /= d;  // multipliers
                __syncthreads();
                // rank-1 update of the trailing block: warps over rows, lanes over columns
                // (consecutive doubles per warp, the pivot-row value kept per column)
                for (int j = k + 1 + lane; j < gs; j += 32) {
                    const double pj = G[k * gs + j];
                    for (int i = k + 1 + warp; i < nf; i += NT / 32)
                        G[i * gs + j] = fma(-G[i * gs + k], pj, G[i * gs + j]);
                }
                __syncthreads();
            }
            if (s_bad) continue;  // singular: jittered retry (attempt 1) or give up
            // back substitution (one warp): x_i = (b_i - sum_{j > i} U_ij x_j) / U_ii
            if (warp == 0) {
                for (int i = nf - 1; i >= 0; --i) {
                    double t = 0.0;
                    for (int j = i + 1 + lane; j < nf; j += 32) t += G[i * gs + j] * s_x[j];
                    t = warp_sum_d(t);
                    if (lane == 0) s_x[i] = (G[i * gs + nf] - t) / G[i * gs + i];
                    __syncwarp();
                }
            }
            __syncthreads();
            st = attempt == 0 ? CALS_ROW_OK : CALS_ROW_JITTERED;
        }
        // write-out as the fp32 solve kernels do (als.py:286, penalty als.py:162-167)
        if (st != CALS_ROW_SINGULAR)
            for (int f = tid; f < nf; f += NT) A.tgt[(int64_t)row * A.ld_tgt + f] = (float)s_x[f];
        if (A.pen_rows != nullptr && warp == 0) {
            double p = 0.0;
            for (int f = lane; f < nf; f += 32) {
                const double xf = (double)(float)s_x[f];
                p += xf * xf;
            }
            p = warp_sum_d(p);
            if (lane == 0) A.pen_rows[row] = (st == CALS_ROW_SINGULAR) ? 0.0 : (double)n * p;
        }
        if (tid == 0) {
            A.status[row] = st;
            report_status(A, row, st);
            stat_add(A, kStRefined, 1);
        }
    }
}

// Float64 Gram of one row from its slice, straight into the register blocks of
// refine_rb_kernel: thread (tr, tc) accumulates G[i][j] for its rows i = tr + 16 a
// over the slice rows kept for column i, and its columns j = tc + 16 b (j = n_f: the
// right-hand side), products of two fp32 values exact in float64; + lam n on the diagonal.
template <int R, int C>
__device__ __forceinline__ void rb_slice_gram(const SweepArgs& A, int64_t lo, int n, bool full,
                                              const uint64_t* s_thr, double (&M)[R][C], double* Xd, double* yd,
                                              uint32_t* bits, int tr, int tc) {
    const int nf = A.nf, tid = threadIdx.x, NT = blockDim.x;
    const int ldx = nf + 1;  // the rating as column nf: [x_k | y_k] per staged row, float64 (exact)
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < C; ++b) M[a][b] = 0.0;
    (void)yd;
    for (int k0 = 0; k0 < n; k0 += kRfChunk) {
        const int kn = min(kRfChunk, n - k0);
        __syncthreads();  // previous chunk consumed
        for (int q = tid; q < kn * ldx; q += NT) {
            const int k = q / ldx, f = q - k * ldx;
            Xd[q] = f < nf ? (double)__ldg(A.src + (int64_t)__ldg(A.idx + lo + k0 + k) * A.ld_src + f)
                           : (double)__ldg(A.val + lo + k0 + k);
        }
        __syncthreads();
        for (int q = tid; q < nf * (kRfChunk / 32); q += NT) {
            const int cc = q % nf, w = q / nf;
            uint32_t word = 0u;
            for (int b = 0; b < 32; ++b) {
                const int k = 32 * w + b;
                if (k < kn && (full || make_key((float)Xd[k * ldx + cc], (uint32_t)(k0 + k)) >= s_thr[cc]))
                    word |= 1u << b;
            }
            bits[cc * (kRfChunk / 32) + w] = word;
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < R; ++a) {
            const int i = tr + 16 * a;
            if (i >= nf) continue;
            for (int w = 0; w < kRfChunk / 32; ++w) {
                uint32_t word = bits[i * (kRfChunk / 32) + w];
                while (word) {
                    const int k = 32 * w + __ffs(word) - 1;
                    word &= word - 1u;
                    const double* xr = Xd + k * ldx;
                    const double xi = xr[i];
#pragma unroll
                    for (int b = 0; b < C; ++b) {
                        const int j = tc + 16 * b;
                        if (j <= nf) M[a][b] = fma(xi, xr[j], M[a][b]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < C; ++b)
            if (tr + 16 * a == tc + 16 * b && tr + 16 * a < nf) M[a][b] += A.lam * (double)n;
}

// Register-blocked float64 elimination for 32 < n_f <= NF (the path every system takes
// above n_f = 64): 256 threads as a 16 x 16 grid, thread (tr, tc) holding rows
// tr + 16 a and columns tc + 16 b of the augmented system [G | b] in registers, so a
// step's rank-1 update is register FMAs (the pivot row and the multipliers come from
// shared memory) instead of a shared-memory read-modify-write per element.  Same
// arithmetic as refine_kernel: partial pivoting without row swaps (first largest
// |G[i][k]| among the unused rows, LAPACK's idamax; every row sees the same pivot
// rows in the same order, so the results equal a swapping LU), elimination without
// pivoting failing on a non-positive pivot for a complete sketch, the reference's
// jitter and one retry, back substitution in pivot order.
template <int NF>
__global__ void __launch_bounds__(256, 1) refine_rb_kernel(SweepArgs A, const int* __restrict__ count,
                                                           const void* __restrict__ list, int from_slice) {
    constexpr int NT = 256, R = NF / 16, C = NF / 16 + 1;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_x[CALS_MAX_NF_DEV];
    __shared__ double s_red[32];
    __shared__ double s_prow[2][16 * C], s_l[2][NF];
    __shared__ double s_cv[2][16], s_ca[2][16];
    __shared__ int s_ci[2][16];
    __shared__ int s_ord[NF];
    __shared__ uint64_t s_thr[CALS_MAX_NF_DEV];
    const int nf = A.nf, gs = nf + 1, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // tc = tid / 16: the 16 owners of a column are one half-warp (pivot search by shuffles)
    const int tr = tid & 15, tc = tid >> 4;
    double* G = reinterpret_cast<double*>(smem);  // [nf][nf+1]: U rows for the back substitution
    double* Xd = reinterpret_cast<double*>(smem + align16((size_t)nf * gs * 8));  // [kRfChunk][nf+1]
    uint32_t* bits_rb = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(Xd) +
                                                    align16((size_t)kRfChunk * gs * 8));
    const int n_list = *count;
    for (int64_t e = blockIdx.x; e < n_list; e += gridDim.x) {
        const int64_t ent = from_slice ? (int64_t)static_cast<const int32_t*>(list)[e] << 32
                                       : static_cast<const int64_t*>(list)[e];
        const int row = (int)(ent >> 32);
        const int64_t slot = (int64_t)(uint32_t)ent;
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const bool full = A.budget[row] >= n;
        const double* Gf = A.gbuf + (size_t)slot * nf * gs;
        __syncthreads();
        if (from_slice && tid < nf) s_thr[tid] = A.thr_keys[(int64_t)row * nf + tid];
        int st = CALS_ROW_SINGULAR;
        for (int attempt = 0; attempt < 2 && st == CALS_ROW_SINGULAR; ++attempt) {
            __syncthreads();
            // ---- the system into registers; padding rows (i >= nf) never pivot ----
            double M[R][C];
            uint32_t used = 0u;
            if (from_slice) {
                rb_slice_gram<R, C>(A, A.ptr[row], n, full, s_thr, M, Xd, nullptr, bits_rb, tr, tc);
            } else {
#pragma unroll
                for (int a = 0; a < R; ++a) {
                    const int i = tr + 16 * a;
#pragma unroll
                    for (int b = 0; b < C; ++b) {
                        const int j = tc + 16 * b;
                        M[a][b] = (i < nf && j <= nf) ? Gf[(size_t)i * gs + j] : 0.0;
                    }
                }
            }
#pragma unroll
            for (int a = 0; a < R; ++a)
                if (tr + 16 * a >= nf) used |= 1u << a;
            if (attempt == 1) {  // the reference's retry: G += 1e-10 * tr(G) / n_f * I (core.py:126-131)
                double t = 0.0;
#pragma unroll
                for (int a = 0; a < R; ++a)
#pragma unroll
                    for (int b = 0; b < C; ++b)
                        if (tr + 16 * a == tc + 16 * b && tr + 16 * a < nf) t += M[a][b];
                t = warp_sum_d(t);
                if (lane == 0) s_red[warp] = t;
                __syncthreads();
                double tt = 0.0;
                for (int w2 = 0; w2 < NT / 32; ++w2) tt += s_red[w2];
                const double jit = 1e-10 * tt / (double)nf;
#pragma unroll
                for (int a = 0; a < R; ++a)
#pragma unroll
                    for (int b = 0; b < C; ++b)
                        if (tr + 16 * a == tc + 16 * b && tr + 16 * a < nf) M[a][b] += jit;
            }
            bool bad = false;
            // steps k = 16 kb + kt: the outer loop is unrolled so column k's register block kb is static
#pragma unroll
            for (int kb = 0; kb < C; ++kb) {
                for (int kt = 0; kt < 16; ++kt) {
                    const int k = 16 * kb + kt;
                    if (k >= nf || bad) break;
                    const int par = k & 1;
                    if (tc == kt) {
                        // the column's owners (one half-warp): first largest |G[i][k]| over the unused rows
                        // (idamax), or row k itself for a complete sketch (elimination without pivoting)
                        double best = -1.0, bv = 0.0;
                        int bi = NF;
#pragma unroll
                        for (int a = 0; a < R; ++a) {
                            const int i = tr + 16 * a;
                            const double v = M[a][kb];
                            const bool cand = !((used >> a) & 1u) && (full ? i == k : true);
                            if (cand && fabs(v) > best) { best = fabs(v); bi = i; bv = v; }
                        }
                        const unsigned hm = 0xFFFFu << (16 * (kt & 1));  // this half-warp
#pragma unroll
                        for (int o = 8; o > 0; o >>= 1) {
                            const double ob = __shfl_xor_sync(hm, best, o, 16);
                            const int oi = __shfl_xor_sync(hm, bi, o, 16);
                            const double ov = __shfl_xor_sync(hm, bv, o, 16);
                            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; bv = ov; }
                        }
                        const bool fail = full ? !(bv > 0.0) : (!(best > 0.0) || bi >= nf);
                        // multipliers scaled by the correctly rounded reciprocal of the pivot, as
                        // LAPACK's dgetf2 / dgetrf2 do (dscal by one / A(j,j))
                        const double inv = fail ? 0.0 : __drcp_rn(bv);
#pragma unroll
                        for (int a = 0; a < R; ++a) {
                            const int i = tr + 16 * a;
                            s_l[par][i] = (((used >> a) & 1u) || i == bi) ? 0.0 : M[a][kb] * inv;
                        }
                        if (tr == 0) {
                            s_ci[par][0] = fail ? -1 : bi;
                            s_ord[k] = bi;
                        }
                    }
                    __syncthreads();
                    const int p = s_ci[par][0];
                    if (p < 0) { bad = true; break; }
                    if (tr == (p & 15)) {  // the pivot row's owners: its entries, and it is used from now on
                        const int ap = p >> 4;
#pragma unroll
                        for (int a = 0; a < R; ++a)
                            if (a == ap) {
                                used |= 1u << a;
#pragma unroll
                                for (int b = kb; b < C; ++b) s_prow[par][tc + 16 * b] = M[a][b];
                            }
                    }
                    __syncthreads();
                    double pr[C];
#pragma unroll
                    for (int b = kb; b < C; ++b) {
                        const int j = tc + 16 * b;
                        pr[b] = (j > k && j <= nf) ? s_prow[par][j] : 0.0;
                    }
#pragma unroll
                    for (int a = 0; a < R; ++a) {
                        if ((used >> a) & 1u) continue;
                        const double l = s_l[par][tr + 16 * a];
#pragma unroll
                        for (int b = kb; b < C; ++b) M[a][b] = fma(-l, pr[b], M[a][b]);
                    }
                }
            }
            if (bad) continue;  // singular: jittered retry (attempt 1) or give up
            // U rows to shared memory, then back substitution in pivot order (one warp)
            __syncthreads();
#pragma unroll
            for (int a = 0; a < R; ++a) {
                const int i = tr + 16 * a;
#pragma unroll
                for (int b = 0; b < C; ++b) {
                    const int j = tc + 16 * b;
                    if (i < nf && j <= nf) G[i * gs + j] = M[a][b];
                }
            }
            __syncthreads();
            if (warp == 0) {
                for (int k = nf - 1; k >= 0; --k) {
                    const int p = s_ord[k];
                    double t = 0.0;
                    for (int j = k + 1 + lane; j < nf; j += 32) t += G[p * gs + j] * s_x[j];
                    t = warp_sum_d(t);
                    if (lane == 0) s_x[k] = (G[p * gs + nf] - t) / G[p * gs + k];
                    __syncwarp();
                }
            }
            __syncthreads();
            st = attempt == 0 ? CALS_ROW_OK : CALS_ROW_JITTERED;
        }
        if (st != CALS_ROW_SINGULAR)
            for (int f = tid; f < nf; f += NT) A.tgt[(int64_t)row * A.ld_tgt + f] = (float)s_x[f];
        if (A.pen_rows != nullptr && warp == 0) {
            double pp = 0.0;
            for (int f = lane; f < nf; f += 32) {
                const double xf = (double)(float)s_x[f];
                pp += xf * xf;
            }
            pp = warp_sum_d(pp);
            if (lane == 0) A.pen_rows[row] = (st == CALS_ROW_SINGULAR) ? 0.0 : (double)n * pp;
        }
        if (tid == 0) {
            A.status[row] = st;
            report_status(A, row, st);
            stat_add(A, kStRefined, 1);
        }
    }
}
template __global__ void refine_rb_kernel<64>(SweepArgs, const int*, const void*, int);
template __global__ void refine_rb_kernel<128>(SweepArgs, const int*, const void*, int);

// Above n_f = 64 nearly every sketched system exceeds the pivot-spread ratio
// (measured on the wide config: 97 %), so the fp32 LU is skipped and every
// system goes to the float64 pass directly.
__global__ void __launch_bounds__(256) defer_all_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                        int64_t n_list) {
    for (int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; li < n_list; li += (int64_t)gridDim.x * blockDim.x)
        defer_refine(A, rows[li], li);
}

template __global__ void refine_kernel<256>(SweepArgs, const int*, const void*, int);

}  // namespace cals
