// common.cuh -- shared device helpers for the core-elements ALS kernels (sm_100a).
//
// Selection key (bit-exact with the reference's ordering, core.py:26-27,
// _kernels.py:84-96): |x| descending, then slice-local row ascending.
//   key(k) = (abs_bits(x) << 32) | (0xFFFFFFFF - k)
// abs_bits of an fp32 is monotone in |x| for every finite value including
// denormals (never compiled with -ftz / fast-math) and +-0 collapse to 0.
// Keys of one column are unique, so "top-s" is exactly {key >= T} for the
// s-th largest key T.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "coreals_b200.h"

#define CALS_FULL_MASK 0xffffffffu

namespace cals {

__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }

__device__ __forceinline__ uint64_t make_key(float x, uint32_t k) {
    return ((uint64_t)abs_bits(x) << 32) | (uint64_t)(0xFFFFFFFFu - k);
}

// ---- explicit shared-memory addressing ------------------------------------
// Hot loops address shared memory through 32-bit shared-window addresses so
// the generic->shared conversion (which ptxas otherwise rematerialises per
// access under register pressure) happens once per kernel.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Bitonic sort of one 64-bit key per lane; result descending (lane 0 = max).
// (d0, d1) += (a0, a1) * s as ONE packed FFMA2 (sm_100: fma.rn.f32x2; each
// lane is an IEEE fmaf, so results are bit-identical to two fmaf calls).
__device__ __forceinline__ void ffma2_bcast(float& d0, float& d1, float a0, float a1, float s) {
    unsigned long long acc, av, sv;
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(d0), "f"(d1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(av), "l"(sv));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(acc));
}

// need-th largest (1-based) of the unique keys held by lanes [0, m), m <= 32,
// by counting: each lane counts the keys above its own (m broadcast rounds;
// cheaper than a 32-wide bitonic sort for the small m of a final sub-bucket).
__device__ __forceinline__ uint64_t warp_kth_desc(uint64_t v, int m, int need, int lane) {
    int gt = 0;
    for (int j = 0; j < m; ++j) {
        const uint64_t o = __shfl_sync(0xffffffffu, v, j);
        gt += (o > v) ? 1 : 0;
    }
    const uint32_t hit = __ballot_sync(0xffffffffu, lane < m && gt == need - 1);
    return __shfl_sync(0xffffffffu, v, __ffs(hit) - 1);
}

__device__ __forceinline__ uint64_t warp_sort_desc(uint64_t v, int lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            uint64_t o = __shfl_xor_sync(CALS_FULL_MASK, v, stride);
            bool lower = (lane & stride) == 0;
            bool desc_block = (lane & size) == 0;
            bool keep_max = (lower == desc_block);
            v = keep_max ? (v > o ? v : o) : (v < o ? v : o);
        }
    }
    return v;
}


// Bitonic sort of 64 keys held two per lane (element e = lane + 32*h), descending
// by element index: after the call v0 = rank lane, v1 = rank lane + 32.
__device__ __forceinline__ void warp_sort64_desc(uint64_t& v0, uint64_t& v1, int lane) {
#pragma unroll
    for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride == 32) {
                // partner is the other register of the same lane (e and e + 32)
                const bool desc_block = (lane & size) == 0;  // size == 64: all descending
                const uint64_t hi = v0 > v1 ? v0 : v1, lo = v0 > v1 ? v1 : v0;
                v0 = desc_block ? hi : lo;
                v1 = desc_block ? lo : hi;
            } else {
                const uint64_t o0 = __shfl_xor_sync(CALS_FULL_MASK, v0, stride);
                const uint64_t o1 = __shfl_xor_sync(CALS_FULL_MASK, v1, stride);
                const bool lower = (lane & stride) == 0;
                const bool d0 = ((lane & size) == 0), d1 = (((lane + 32) & size) == 0);
                const bool k0 = (lower == d0), k1 = (lower == d1);
                v0 = k0 ? (v0 > o0 ? v0 : o0) : (v0 < o0 ? v0 : o0);
                v1 = k1 ? (v1 > o1 ? v1 : o1) : (v1 < o1 ? v1 : o1);
            }
        }
    }
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CALS_FULL_MASK, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CALS_FULL_MASK, v, o);
    return v;
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CALS_FULL_MASK, v, o);
    return v;
}

// Fixed-order block reduction of one double per thread (deterministic).
// scratch: >= blockDim.x/32 doubles.  Result valid in thread 0.
__device__ __forceinline__ double block_sum_d(double v, double* scratch) {
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum_d(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) {
        int nw = (blockDim.x + 31) >> 5;
        for (int w = 0; w < nw; ++w) r += scratch[w];
    }
    return r;
}

__device__ __forceinline__ int block_sum_i(int v, int* scratch) {
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum_i(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    int r = 0;
    int nw = (blockDim.x + 31) >> 5;
    for (int w = 0; w < nw; ++w) r += scratch[w];
    __syncthreads();
    return r;  // valid in every thread
}

// Exact floor division e / d for e < 2^24, d <= 256, via one multiply-high.
struct FastDiv {
    uint32_t d, magic;
    __host__ __device__ FastDiv() : d(1), magic(0) {}
    __host__ __device__ explicit FastDiv(uint32_t dd) : d(dd), magic((uint32_t)((0x100000000ull + dd - 1) / dd)) {}
    __device__ __forceinline__ uint32_t div(uint32_t e) const { return d == 1 ? e : __umulhi(e, magic); }
};

}  // namespace cals
