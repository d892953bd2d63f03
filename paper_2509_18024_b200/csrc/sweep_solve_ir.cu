// sweep_solve_ir.cu -- mixed-precision solve of the sketched normal equations:
// every system above n_f = 64, and at 32 < n_f <= 64 the systems the fp32 warp
// LU (solve_wide_kernel) found ill-conditioned (core.py:120-131, _kernels.py:233-236: LAPACK gesv
// on the float64 system).
//
// The float64 system stays in the batch buffer; a CTA of N = 64 / 128 threads factors
// its fp32 rounding with a register-resident LU (thread r owns row r, N
// columns in registers, partial pivoting without row swaps: the pivot row of a
// step is published through shared memory and every unused row eliminates
// against it), then refines the solution against the float64 system:
//     r = b - G x   (float64)
//     L U d = r     (fp32 triangular solves from the packed factors)
//     x += d        (float64)
// The residual decides what the iteration converges to.  A tiled row's stored
// equations were accumulated in float64, so its residual reads them back.  A
// short row's equations (staged / tiny tier) were summed in fp32 -- measured on
// the wide config at a later iteration that rounding alone moves most solutions
// by more than 1e-4 -- so its residual is formed from the slice itself, exactly:
//     t_k = y_k - x_k . x          (float64 dot per slice row)
//     r_c = sum_{k kept for c} X[k][c] t_k - lam n x_c
// (the kept sets from the row's selection thresholds), i.e. the residual of the
// float64 normal equations without ever forming them; the fp32 factors only
// precondition.
// until the corrections say the float64 answer is reached: with rho the ratio
// of successive correction norms, it stops when |d| <= 1e-6 |x| or, from the
// second correction on, rho / (1 - rho) * |d| <= 1e-6 |x| (max norms; the
// factor contract is 1e-4 per row), and hands the system to the
// float64 elimination (sweep_refine.cu) when the fp32 factorisation breaks
// down or the refinement contracts slower than 0.7 per step or has not
// converged after kIrMaxIt = 12 corrections (cond * 1e-6 >~ 0.7; a correction costs ~1/12 of
// the float64 elimination, so the budget is where the two break even).  That float64
// pass owns the reference's singular / jitter semantics, so this kernel only
// ever reports CALS_ROW_OK.  A complete sketch (s == n, als.py:184-205)
// eliminates without pivoting and defers on a non-positive pivot.
//
// N = 128: three CTAs per SM (66 KB of shared memory each: the fp32 copy of the
// system, then the packed factors for the triangular solves); N = 64: eight.
#include "solve.cuh"
#include "sweep_common.cuh"

namespace cals {

constexpr int kIrN = 128;          // largest padded order (thread r owns row r); the kernel is built for 64 and 128
constexpr int kIrMaxIt = 12;       // corrections before the float64 pass takes over (N = 128; 6 at N = 64)
constexpr int kIrSliceN = 448;     // rows up to this length (and rf_slice_max) take the slice residual; the staged
                                   // tier holds no longer row above n_f = 64 (cals_plan_build)
constexpr float kIrTol = 1e-6f;    // rho * |d| <= kIrTol * |x|
constexpr float kIrRhoMax = 0.7f;  // slowest accepted contraction (N = 128; 0.5 at N = 64)

__host__ __device__ inline size_t solve_ir_smem(int N) { return (size_t)N * (N + 1) * sizeof(float); }

template <int N>
struct IrShared {
    float prow[2][N + 8];  // pivot row of the step: columns, [128] rhs, [129] the pivot itself
    uint32_t key[2][4];       // per-warp pivot candidates (N / 32 used)
    double xd[N];          // the solution, float64
    float rhs[N];          // right-hand side in pivot order
    float xs[N];           // solved block values of the triangular solves
    float dinv[N];         // 1 / U_tt
    int perm[N];           // equation e was the pivot row of step perm[e]
    int inv[N];            // ... and step t pivoted on equation inv[t]
    float red[4];
    double pen[4];
    double t[kIrSliceN];      // slice residual: y_k - x_k . x
    int idx[kIrSliceN];       // the row's source rows
};

// (d0, d1) += s2 * (b0, b1), s2 a packed pair: one FFMA2 (each half an IEEE fmaf)
__device__ __forceinline__ void ffma2_sv(float& d0, float& d1, unsigned long long s2, float b0, float b1) {
    unsigned long long acc, bv;
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(d0), "f"(d1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(s2), "l"(bv));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(acc));
}

// a[B0 + i] for a CTA-uniform runtime i in [0, 16): a jump table instead of a 16-way select chain
template <int N, int B0>
__device__ __forceinline__ float ir_pick(const float (&a)[N], int i) {
    switch (i) {
        case 0: return a[B0 + 0];
        case 1: return a[B0 + 1];
        case 2: return a[B0 + 2];
        case 3: return a[B0 + 3];
        case 4: return a[B0 + 4];
        case 5: return a[B0 + 5];
        case 6: return a[B0 + 6];
        case 7: return a[B0 + 7];
        case 8: return a[B0 + 8];
        case 9: return a[B0 + 9];
        case 10: return a[B0 + 10];
        case 11: return a[B0 + 11];
        case 12: return a[B0 + 12];
        case 13: return a[B0 + 13];
        case 14: return a[B0 + 14];
        default: return a[B0 + 15];
    }
}
// Elimination steps K in [B0, B0 + 16): a runtime loop inside a compile-time column
// block (the fully unrolled elimination thrashes the instruction cache).  Column K of
// the thread's row comes from a 16-way register select; the update sweeps columns
// j >= B0, the pivot row publishing zeros at j <= K so the multipliers stored left of
// K survive.
template <int N, int B0>
__device__ __forceinline__ bool ir_block(float (&a)[N], float& rhs, bool& used, int& ord, float& diag, IrShared<N>& S,
                                         float* __restrict__ Lrow, int nf, bool spd, int r, int lane, int warp) {
#pragma unroll 1
    for (int K = B0; K < B0 + 16; ++K) {
        if (K >= nf) return false;
        const int par = K & 1;
        const float ck = ir_pick<N, B0>(a, K - B0);
        int p = K;
        if (!spd) {
            // largest |a[r][K]| over the unused rows, ties (to 2^-16 relative) to the smallest row:
            // partial pivoting needs a large pivot, not the exact maximum
            const uint32_t mine = used ? 0u : ((__float_as_uint(ck) & 0x7FFFFF80u) | (uint32_t)(127 - r));
            const uint32_t wbest = __reduce_max_sync(CALS_FULL_MASK, mine);
            if (lane == 0) S.key[par][warp] = wbest;
            __syncthreads();
            uint32_t best = S.key[par][0];
#pragma unroll
            for (int w = 1; w < N / 32; ++w) best = max(best, S.key[par][w]);
            if ((best >> 7) == 0u) return true;  // no nonzero finite candidate (NaN keys are caught below)
            p = 127 - (int)(best & 127u);
        }
        if (r == p) {
            used = true;
            ord = K;
            diag = ck;
            float* pr = S.prow[par];
#pragma unroll
            for (int j = B0; j < B0 + 16; j += 4)
                *reinterpret_cast<float4*>(pr + j) = make_float4(j + 0 > K ? a[j + 0] : 0.f, j + 1 > K ? a[j + 1] : 0.f,
                                                                 j + 2 > K ? a[j + 2] : 0.f, j + 3 > K ? a[j + 3] : 0.f);
#pragma unroll
            for (int j = B0 + 16; j < N; j += 4)
                *reinterpret_cast<float4*>(pr + j) = make_float4(a[j], a[j + 1], a[j + 2], a[j + 3]);
            pr[N] = rhs;
            pr[N + 1] = ck;
        }
        __syncthreads();
        const float* pr = S.prow[par];
        const float d = pr[N + 1];
        if (spd ? !(d > 0.f) : !(fabsf(d) <= 3.0e38f)) return true;  // breakdown: uniform (every thread reads d)
        const float f = used ? 0.f : ck * __frcp_rn(d);
        if (!used) Lrow[K] = f;  // the multiplier (L entry) goes straight to the packed factors
        const float nf1 = -f;
        unsigned long long nf2;
        asm("mov.b64 %0, {%1, %1};" : "=l"(nf2) : "f"(nf1));
#pragma unroll
        for (int j = B0; j < N; j += 4) {
            const float4 v = *reinterpret_cast<const float4*>(pr + j);
            ffma2_sv(a[j + 0], a[j + 1], nf2, v.x, v.y);
            ffma2_sv(a[j + 2], a[j + 3], nf2, v.z, v.w);
        }
        rhs = fmaf(nf1, pr[N], rhs);
    }
    return false;
}

template <int N, int... Q>
__device__ __forceinline__ bool ir_eliminate(float (&a)[N], float& rhs, bool& used, int& ord, float& diag,
                                             IrShared<N>& S, float* __restrict__ Lrow, int nf, bool spd, int r, int lane,
                                             int warp, std::integer_sequence<int, Q...>) {
    bool fail = false;
    ((fail = fail || ir_block<N, 16 * Q>(a, rhs, used, ord, diag, S, Lrow, nf, spd, r, lane, warp)), ...);
    return fail;
}

// U x = rhs over the packed factors (pivot-order row t = stored row S.inv[t]: L left of column t, U
// from it); thread t owns pivot-order row t.  Blocks of 32: the owning warp solves its diagonal block by
// shuffles, the rows above subtract the block's contribution.
template <int N>
__device__ __forceinline__ float ir_solve_upper(const float* __restrict__ LU, IrShared<N>& S, float rhs, int t, int lane,
                                                int warp) {
    const float* row = LU + S.inv[t] * (N + 1);
    const float di = S.dinv[t];
    float x = 0.f;
#pragma unroll
    for (int B = N / 32 - 1; B >= 0; --B) {
        if (warp == B) {
#pragma unroll
            for (int k = 31; k >= 0; --k) {
                const float xk = __shfl_sync(CALS_FULL_MASK, rhs * di, k);
                if (lane == k) x = xk;
                if (lane < k) rhs = fmaf(-row[32 * B + k], xk, rhs);
            }
            S.xs[t] = x;
        }
        if (B > 0) {
            __syncthreads();
            if (warp < B) {
#pragma unroll
                for (int k = 0; k < 32; k += 4) {
                    const float4 xv = *reinterpret_cast<const float4*>(S.xs + 32 * B + k);
                    rhs = fmaf(-row[32 * B + k + 0], xv.x, rhs);
                    rhs = fmaf(-row[32 * B + k + 1], xv.y, rhs);
                    rhs = fmaf(-row[32 * B + k + 2], xv.z, rhs);
                    rhs = fmaf(-row[32 * B + k + 3], xv.w, rhs);
                }
            }
        }
    }
    return x;
}

// L y = rhs (unit diagonal), same blocking, forward.
template <int N>
__device__ __forceinline__ float ir_solve_lower(const float* __restrict__ LU, IrShared<N>& S, float rhs, int t, int lane,
                                                int warp) {
    const float* row = LU + S.inv[t] * (N + 1);
#pragma unroll
    for (int B = 0; B < N / 32; ++B) {
        if (warp == B) {
#pragma unroll
            for (int k = 0; k < 31; ++k) {
                const float yk = __shfl_sync(CALS_FULL_MASK, rhs, k);
                if (lane > k) rhs = fmaf(-row[32 * B + k], yk, rhs);
            }
            S.xs[t] = rhs;
        }
        if (B < N / 32 - 1) {
            __syncthreads();
            if (warp > B) {
#pragma unroll
                for (int k = 0; k < 32; k += 4) {
                    const float4 yv = *reinterpret_cast<const float4*>(S.xs + 32 * B + k);
                    rhs = fmaf(-row[32 * B + k + 0], yv.x, rhs);
                    rhs = fmaf(-row[32 * B + k + 1], yv.y, rhs);
                    rhs = fmaf(-row[32 * B + k + 2], yv.z, rhs);
                    rhs = fmaf(-row[32 * B + k + 3], yv.w, rhs);
                }
            }
        }
    }
    return rhs;
}

// max over the CTA of a non-negative float (uniform result)
template <int N>
__device__ __forceinline__ float ir_block_max(float v, IrShared<N>& S, int lane, int warp) {
    const uint32_t w = __reduce_max_sync(CALS_FULL_MASK, __float_as_uint(v));
    __syncthreads();
    if (lane == 0) S.red[warp] = __uint_as_float(w);
    __syncthreads();
    float m = S.red[0];
#pragma unroll
    for (int w = 1; w < N / 32; ++w) m = fmaxf(m, S.red[w]);
    return m;
}

// rows != nullptr: the batch's systems rows[li], equations in slot li (n_f > 64: every system).
// rows == nullptr: the systems the fp32 solve deferred, (row << 32 | slot) entries of A.ir_list
// (32 < n_f <= 64).
template <int N>
__global__ void __launch_bounds__(N, N == 128 ? 3 : 8) solve_ir_kernel(SweepArgs A, const int32_t* __restrict__ rows,
                                                                        int64_t n_rows) {
    constexpr int LD = N + 1;  // shared-memory row stride (conflict-free column walks)
    constexpr int NW = N / 32;
    constexpr int MC = N / 32 + 1;  // 32-column groups of an augmented row
    // the correction budget sits where a correction and the float64 elimination break even: the
    // 64-wide elimination is cheap (measured on the 500M config: 6 / 0.5 beats 12 / 0.7 by 1 ms)
    constexpr int max_it = N == 128 ? kIrMaxIt : 6;
    constexpr float rho_max = N == 128 ? kIrRhoMax : 0.5f;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(16) IrShared<N> S;
    float* LU = reinterpret_cast<float*>(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nf = A.nf, gs = nf + 1;
    const int64_t n_list = rows != nullptr ? n_rows : (int64_t)*A.ir_cnt;
    for (int64_t li = blockIdx.x; li < n_list; li += gridDim.x) {
        const int64_t ent = rows != nullptr ? (((int64_t)rows[li] << 32) | li) : A.ir_list[li];
        const int row = (int)(ent >> 32);
        const int64_t slot = (int64_t)(uint32_t)ent;
        const int n = (int)(A.ptr[row + 1] - A.ptr[row]);
        const bool spd = A.budget[row] >= n;
        const double* __restrict__ G = A.gbuf + (size_t)slot * nf * gs;
        const int64_t lo = A.ptr[row];
        // short rows (fp32-summed equations): the residual comes from the slice
        const bool slice = n <= kIrSliceN && n <= A.rf_slice_max;
        const uint64_t thr = (slice && tid < nf) ? A.thr_keys[(int64_t)row * nf + tid] : 0ull;
        __syncthreads();  // the previous system's factors are consumed
        if (slice)
            for (int k = tid; k < n; k += N) S.idx[k] = __ldg(A.idx + lo + k);
        // ---- the system, rounded to fp32, into shared memory (warp per row, coalesced) ----
        for (int i0 = warp; i0 < nf; i0 += 4 * NW) {
            double v[4][MC];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + NW * u;
#pragma unroll
                for (int m = 0; m < MC; ++m) {
                    const int j = lane + 32 * m;
                    v[u][m] = (i < nf && j < gs) ? __ldcs(G + (size_t)i * gs + j) : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + NW * u;
#pragma unroll
                for (int m = 0; m < MC; ++m) {
                    const int j = lane + 32 * m;
                    if (i < nf && j < gs) LU[i * LD + j] = (float)v[u][m];
                }
            }
        }
        __syncthreads();
        if (rows != nullptr && li + gridDim.x < n_list) {  // the CTA's next system on its way into L2 meanwhile
            const char* nx = reinterpret_cast<const char*>(A.gbuf + (size_t)(li + gridDim.x) * nf * gs);
            for (int off = tid * 128; off < nf * gs * 8; off += N * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + off));
        }
        // ---- thread r takes row r; rows / columns beyond nf are identity padding ----
        float a[N];
        float rhs = 0.f;
        const int r = tid;
        if (r < nf) {
#pragma unroll
            for (int j = 0; j < N; ++j) a[j] = j < nf ? LU[r * LD + j] : 0.f;
            rhs = LU[r * LD + nf];
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) a[j] = j == r ? 1.f : 0.f;
        }
        bool used = r >= nf;  // padding rows never pivot: they keep step r
        int ord = r;
        float diag = 1.f;
        bool fail = ir_eliminate<N>(a, rhs, used, ord, diag, S, LU + r * LD, nf, spd, r, lane, warp,
                                    std::make_integer_sequence<int, N / 16>{});
        fail = fail || __syncthreads_or(!used);  // every row pivoted (uniform)
        int st = -1;                            // -1: deferred to the float64 pass
        if (!fail) {
            // ---- the U part of the row joins its multipliers in shared memory (row r stays row r;
            // the triangular solves walk the rows in pivot order through S.inv) ----
#pragma unroll
            for (int j = 0; j < N; ++j)
                if (j >= ord) LU[r * LD + j] = a[j];
            S.dinv[ord] = __frcp_rn(diag);
            S.rhs[ord] = rhs;
            S.perm[r] = ord;
            S.inv[ord] = r;
            __syncthreads();
            const int t = tid;
            float x0 = ir_solve_upper<N>(LU, S, S.rhs[t], t, lane, warp);
            double x = (double)x0;
            float prev = ir_block_max<N>(fabsf(x0), S, lane, warp);  // |x0|: the "correction" before the first
            if (!(prev <= 3.0e38f)) fail = true;
            for (int it = 0; it < max_it && !fail && st < 0; ++it) {
                S.xd[t] = x;
                if (t >= nf) S.rhs[t] = 0.f;
                __syncthreads();
                if (slice) {
                    // t_k = y_k - x_k . x: warp per slice row, 4 columns per lane
                    double xq[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) xq[q] = 4 * lane + q < nf ? S.xd[4 * lane + q] : 0.0;
                    for (int k0 = warp; k0 < n; k0 += 4 * NW) {
                        float4 v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int k = k0 + NW * u;
                            v[u] = (k < n && 4 * lane < nf)
                                       ? __ldg(reinterpret_cast<const float4*>(A.src + (int64_t)S.idx[k] * A.ld_src) + lane)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int k = k0 + NW * u;
                            double p = (double)v[u].x * xq[0];
                            p = fma((double)v[u].y, xq[1], p);
                            p = fma((double)v[u].z, xq[2], p);
                            p = fma((double)v[u].w, xq[3], p);
                            p = warp_sum_d(p);
                            if (lane == 0 && k < n) S.t[k] = (double)__ldg(A.val + lo + k) - p;
                        }
                    }
                    __syncthreads();
                    // r_c = sum over column c's kept rows of X[k][c] t_k - lam n x_c: thread per column
                    if (t < nf) {
                        double acc = 0.0;
                        const float* col = A.src + t;
                        int k = 0;
                        for (; k + 8 <= n; k += 8) {
                            float xv[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) xv[u] = __ldg(col + (int64_t)S.idx[k + u] * A.ld_src);
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                if (spd || make_key(xv[u], (uint32_t)(k + u)) >= thr) acc = fma((double)xv[u], S.t[k + u], acc);
                        }
                        for (; k < n; ++k) {
                            const float xv = __ldg(col + (int64_t)S.idx[k] * A.ld_src);
                            if (spd || make_key(xv, (uint32_t)k) >= thr) acc = fma((double)xv, S.t[k], acc);
                        }
                        S.rhs[S.perm[t]] = (float)(acc - A.lam * (double)n * x);
                    }
                } else {
                    // r = b - G x in float64 from the stored equations: warp per equation, lanes over columns
                    for (int e0 = warp; e0 < nf; e0 += 4 * NW) {
                        double acc[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int e = e0 + NW * u;
                            acc[u] = 0.0;
                            if (e < nf) {
                                const double* g = G + (size_t)e * gs;
#pragma unroll
                                for (int m = 0; m < NW; ++m) {
                                    const int j = lane + 32 * m;
                                    if (j < nf) acc[u] = fma(__ldg(g + j), S.xd[j], acc[u]);
                                }
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int e = e0 + NW * u;
                            const double sm = warp_sum_d(acc[u]);
                            if (lane == 0 && e < nf) S.rhs[S.perm[e]] = (float)(__ldg(G + (size_t)e * gs + nf) - sm);
                        }
                    }
                }
                __syncthreads();
                const float y = ir_solve_lower<N>(LU, S, S.rhs[t], t, lane, warp);
                __syncthreads();  // the lower solve's last block values are read before the upper solve rewrites them
                const float d = ir_solve_upper<N>(LU, S, y, t, lane, warp);
                x += (double)d;
                const float dn = ir_block_max<N>(fabsf(d), S, lane, warp);
                const float xn = ir_block_max<N>(fabsf((float)x), S, lane, warp);
                if (!(dn <= 3.0e38f)) { fail = true; break; }
                // contraction measured between two corrections (the first one is compared with |x0|, which
                // only bounds it: x0 also carries the fp32 rounding of the equations, so the first
                // correction ends the iteration only when it is itself negligible)
                const float rho = prev > 0.f ? dn / prev : 0.f;
                if (dn <= kIrTol * xn || (it > 0 && rho <= rho_max && rho * dn <= (1.f - rho) * kIrTol * xn)) st = CALS_ROW_OK;
                else if (rho > rho_max) fail = true;
                prev = dn;
            }
            if (st == CALS_ROW_OK) {
                const float xf = (float)x;
                if (t < nf) A.tgt[(int64_t)row * A.ld_tgt + t] = xf;
                if (A.pen_rows != nullptr) {
                    const double p = warp_sum_d(t < nf ? (double)xf * (double)xf : 0.0);
                    if (lane == 0) S.pen[warp] = p;
                    __syncthreads();
                    if (tid == 0) {
                        double ps = S.pen[0];
#pragma unroll
                        for (int w = 1; w < NW; ++w) ps += S.pen[w];
                        A.pen_rows[row] = (double)n * ps;
                    }
                }
                if (tid == 0) {
                    A.status[row] = CALS_ROW_OK;
                    report_status(A, row, CALS_ROW_OK);
                }
            }
        }
        if (st < 0 && tid == 0) defer_refine(A, row, slot);  // the float64 elimination owns the row
    }
}
template __global__ void solve_ir_kernel<64>(SweepArgs, const int32_t*, int64_t);
template __global__ void solve_ir_kernel<128>(SweepArgs, const int32_t*, int64_t);

}  // namespace cals
