// peaks.cu -- compute-pipe peaks of the B200 for the roofline's compute term
// (SURVEY 8d asked for them: MEASURED_PEAKS.json has only HBM and cuBLAS bf16)
// plus a numerical check of the tcgen05 kind::i8 path used by the integer Gram.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_18024_b200/csrc \
//        -o tools/peaks tools/peaks.cu && tools/peaks > profiles/r02_peaks.json
//
// Every figure is whole-chip work / CUDA-event time of one launch (best of 5)
// over 148 x k CTAs, so it is at the clock the chip actually ran.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tc.cuh"

using namespace cals;

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess) {                                                              \
            fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                          \
        }                                                                                     \
    } while (0)

constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) k_ffma(float* out, float a, float b) {
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x + i;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_ffma2(float* out, float a, float b) {
    unsigned long long acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float2 v = make_float2(threadIdx.x + i, i);
        memcpy(&acc[i], &v, 8);
    }
    float2 av = make_float2(a, a), bv = make_float2(b, b);
    unsigned long long A, B;
    memcpy(&A, &av, 8);
    memcpy(&B, &bv, 8);
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float2 v;
        memcpy(&v, &acc[i], 8);
        s += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_dfma(double* out, double a, double b) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x + i;
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// float64 FMA of fp32 operands (what a float64 Gram of fp32 data issues): F2F.F64.F32 + DFMA
__global__ void __launch_bounds__(256) k_dfma_f32(double* out, float a, float step) {
    double acc[8];
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        acc[i] = 0.0;
        x[i] = threadIdx.x * 0.5f + i;
    }
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc[i] = fma((double)x[i], (double)a, acc[i]);
            x[i] += step;
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// shared-memory bandwidth: conflict-free LDS.128
__global__ void __launch_bounds__(256) k_lds(float* out) {
    __shared__ float4 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = threadIdx.x;
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float4 v = buf[(idx + u * 256) & 2047];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        idx = (idx + 32) & 2047;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// ---- tcgen05: one CTA per SM, thread 0 issues `rounds` x KSTEPS MMAs ---------
enum Kind { KI8_SS = 0, KI8_TS = 1, KTF32_SS = 2, KBF16_SS = 3 };
constexpr int KB = 128;  // K bytes staged per operand row (4 MMAs of 32 bytes)

template <int KIND>
__global__ void __launch_bounds__(128, 1)
    k_mma(const int8_t* __restrict__ Ag, const int8_t* __restrict__ Bg, int N, int rounds, int32_t* __restrict__ Dout,
          long long* __restrict__ cycles) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long mbar;
    unsigned char* As = smem;                // 128 x KB
    unsigned char* Bs = smem + 128 * KB;     // N x KB
    const int tid = threadIdx.x, warp = tid >> 5;
    // operands into the K-major interleaved layout
    for (int e = tid; e < 128 * KB; e += blockDim.x) {
        const int r = e / KB, kb = e % KB;
        As[tc::kmajor_off(r, kb, KB)] = (unsigned char)Ag[e];
    }
    for (int e = tid; e < N * KB; e += blockDim.x) {
        const int r = e / KB, kb = e % KB;
        Bs[tc::kmajor_off(r, kb, KB)] = (unsigned char)Bg[e];
    }
    if (warp == 0) tc::tmem_alloc<512>(&tslot);
    if (tid == 0) tc::mbar_init(tc::smem_addr(&mbar), 1);
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tslot;
    const uint32_t a_tmem = tbase + 256;  // A operand columns (TS mode): 128 lanes x KB/4 columns
    if (KIND == KI8_TS) {
        // row r = lane 32*warp + lane: its KB bytes packed 4 per column
        const int r = tid;
        for (int c0 = 0; c0 < KB / 4; c0 += 8) {
            uint32_t v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint32_t w = 0;
                for (int b = 0; b < 4; ++b) w |= (uint32_t)(uint8_t)Ag[r * KB + 4 * (c0 + j) + b] << (8 * b);
                v[j] = w;
            }
            tc::st_32x32b_x8(a_tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
        }
        tc::st_wait();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t sa = tc::smem_addr(As), sb = tc::smem_addr(Bs);
    const int elem = (KIND == KTF32_SS) ? 4 : (KIND == KBF16_SS ? 2 : 1);
    (void)elem;
    uint32_t idesc = KIND == KTF32_SS ? tc::idesc_tf32(128, N) : (KIND == KBF16_SS ? tc::idesc_bf16(128, N)
                                                                                    : tc::idesc_i8(128, N));
    long long t0 = 0, t1 = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const int R = pass == 0 ? 1 : rounds;
        if (tid == 0) {
            t0 = clock64();
            for (int it = 0; it < R; ++it) {
#pragma unroll
                for (int ks = 0; ks < KB / 32; ++ks) {
                    const uint64_t bd = tc::sdesc(sb + 256u * ks, 128, KB * 8);
                    const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
                    if (KIND == KI8_TS) {
                        tc::mma_i8_ts(tbase, a_tmem + 8u * ks, bd, idesc, acc);
                    } else {
                        const uint64_t ad = tc::sdesc(sa + 256u * ks, 128, KB * 8);
                        if (KIND == KI8_SS) tc::mma_i8_ss(tbase, ad, bd, idesc, acc);
                        else if (KIND == KTF32_SS) tc::mma_tf32_ss(tbase, ad, bd, idesc, acc);
                        else tc::mma_bf16_ss(tbase, ad, bd, idesc, acc);
                    }
                }
            }
            tc::commit(tc::smem_addr(&mbar));
            tc::mbar_wait(tc::smem_addr(&mbar), pass & 1);
            t1 = clock64();
        }
        __syncthreads();
        tc::fence_after();
        if (pass == 0 && blockIdx.x == 0) {
            // D (128 x N, s32) -> global; warp w reads lanes 32w..32w+31
            for (int c0 = 0; c0 < N; c0 += 8) {
                uint32_t v[8];
                tc::ld_32x32b_x8(tbase + ((uint32_t)(32 * warp) << 16) + c0, v);
                tc::ld_wait();
#pragma unroll
                for (int j = 0; j < 8; ++j) Dout[tid * N + c0 + j] = (int32_t)v[j];
            }
        }
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
    }
    if (tid == 0) cycles[blockIdx.x] = t1 - t0;
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tbase);
}


// MN-major (M / N contiguous) interleaved operands, as the integer Gram writes them:
// byte (mn, k) of a [R x 32] K-step tile at (mn/16)*512 + (k/8)*128 + (k%8)*16 + mn%16
__host__ __device__ constexpr uint32_t mn_off(uint32_t mn, uint32_t k) {
    return (mn >> 4) * 512u + (k >> 3) * 128u + (k & 7u) * 16u + (mn & 15u);
}
__global__ void __launch_bounds__(128, 1)
    k_mma_mn(const int8_t* __restrict__ Ag, const int8_t* __restrict__ Bg, int N, int ksteps, int32_t* __restrict__ Dout) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long mbar;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int KT = 32 * ksteps;
    unsigned char* As = smem;                       // ksteps tiles of 128 x 32
    unsigned char* Bs = smem + ksteps * 128 * 32;   // ksteps tiles of N x 32
    for (int e = tid; e < 128 * KT; e += blockDim.x) {
        const int m = e / KT, k = e % KT;
        As[(k / 32) * 4096 + mn_off(m, k % 32)] = (unsigned char)Ag[m * KT + k];
    }
    const int btile = (N + 15) / 16 * 512;
    for (int e = tid; e < N * KT; e += blockDim.x) {
        const int n = e / KT, k = e % KT;
        Bs[(k / 32) * btile + mn_off(n, k % 32)] = (unsigned char)Bg[n * KT + k];
    }
    if (warp == 0) tc::tmem_alloc<256>(&tslot);
    if (tid == 0) tc::mbar_init(tc::smem_addr(&mbar), 1);
    tc::fence_smem_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tslot;
    const uint32_t idesc = tc::idesc_i8(128, N) | (1u << 15) | (1u << 16);  // A and B MN-major
    if (tid == 0) {
        for (int ks = 0; ks < ksteps; ++ks)
            tc::mma_i8_ss(tbase, tc::sdesc(tc::smem_addr(As) + 4096u * ks, 128, 512),
                          tc::sdesc(tc::smem_addr(Bs) + (uint32_t)btile * ks, 128, 512), idesc, ks > 0);
        tc::commit(tc::smem_addr(&mbar));
        tc::mbar_wait(tc::smem_addr(&mbar), 0);
    }
    __syncthreads();
    tc::fence_after();
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        tc::ld_32x32b_x8(tbase + ((uint32_t)(32 * warp) << 16) + c0, v);
        tc::ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j) Dout[tid * N + c0 + j] = (int32_t)v[j];
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<256>(tbase);
}

static float time_launch(void (*launch)(void*), void* arg, int reps = 5) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    launch(arg);
    CK(cudaDeviceSynchronize());
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(a));
        launch(arg);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return best;
}

struct Ctx {
    int sms;
    void* out;
    int8_t *A, *B;
    int32_t* D;
    long long* cyc;
    int N, rounds;
};

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    Ctx c{};
    c.sms = p.multiProcessorCount;
    const int blocks = c.sms * 4, threads = 256;
    CK(cudaMalloc(&c.out, (size_t)blocks * threads * 8));
    std::string js = "{";
    char buf[512];
    snprintf(buf, sizeof buf, "\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d", p.name, c.sms, p.clockRate);
    js += buf;

    auto sim = [&](const char* name, void (*launch)(void*), double flops) {
        const float ms = time_launch(launch, &c);
        snprintf(buf, sizeof buf, ", \"%s_tflops\": %.2f", name, flops / (ms * 1e-3) / 1e12);
        js += buf;
    };
    const double nthr = (double)blocks * threads;
    sim("ffma", [](void* v) { auto* c = (Ctx*)v; k_ffma<<<c->sms * 4, 256>>>((float*)c->out, 0.999f, 0.001f); },
        nthr * kIters * 16 * 2);
    sim("ffma2", [](void* v) { auto* c = (Ctx*)v; k_ffma2<<<c->sms * 4, 256>>>((float*)c->out, 0.999f, 0.001f); },
        nthr * kIters * 8 * 4);
    sim("dfma", [](void* v) { auto* c = (Ctx*)v; k_dfma<<<c->sms * 4, 256>>>((double*)c->out, 0.999, 0.001); },
        nthr * (kIters / 4) * 16 * 2);
    sim("dfma_of_f32", [](void* v) { auto* c = (Ctx*)v; k_dfma_f32<<<c->sms * 4, 256>>>((double*)c->out, 0.999f, 1e-3f); },
        nthr * (kIters / 4) * 8 * 2);
    {
        const float ms = time_launch([](void* v) { auto* c = (Ctx*)v; k_lds<<<c->sms * 4, 256>>>((float*)c->out); }, &c);
        snprintf(buf, sizeof buf, ", \"lds128_tbs\": %.2f", nthr * (kIters / 4) * 8 * 16 / (ms * 1e-3) / 1e12);
        js += buf;
    }

    // ---- tcgen05 --------------------------------------------------------------
    const int NMAX = 256;
    std::vector<int8_t> hA(128 * KB), hB(NMAX * KB);
    srand(1);
    for (auto& x : hA) x = (int8_t)((rand() % 256) - 128);
    for (auto& x : hB) x = (int8_t)((rand() % 256) - 128);
    CK(cudaMalloc(&c.A, hA.size()));
    CK(cudaMalloc(&c.B, hB.size()));
    CK(cudaMalloc(&c.D, 128 * NMAX * 4));
    CK(cudaMalloc(&c.cyc, c.sms * 8));
    CK(cudaMemcpy(c.A, hA.data(), hA.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.B, hB.data(), hB.size(), cudaMemcpyHostToDevice));
    const size_t smem = (size_t)(128 + NMAX) * KB;
    CK(cudaFuncSetAttribute(k_mma<KI8_SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_mma<KI8_TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_mma<KTF32_SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_mma<KBF16_SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    std::vector<int32_t> hD(128 * NMAX);
    auto check_i8 = [&](int N) {
        CK(cudaMemcpy(hD.data(), c.D, 128 * N * 4, cudaMemcpyDeviceToHost));
        long bad = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < N; ++n) {
                int32_t ref = 0;
                for (int k = 0; k < KB; ++k) ref += (int32_t)hA[m * KB + k] * (int32_t)hB[n * KB + k];
                bad += hD[m * N + n] != ref;
            }
        return bad;
    };
    struct Case {
        const char* name;
        int kind, N;
        double k_per_round;  // MACs per MMA row-column pair per round (K elements)
    };
    const Case cases[] = {{"i8_ss", KI8_SS, 64, KB},   {"i8_ss", KI8_SS, 128, KB}, {"i8_ss", KI8_SS, 256, KB},
                          {"i8_ts", KI8_TS, 64, KB},   {"i8_ts", KI8_TS, 128, KB}, {"i8_ts", KI8_TS, 256, KB},
                          {"tf32_ss", KTF32_SS, 128, KB / 4}, {"tf32_ss", KTF32_SS, 256, KB / 4},
                          {"bf16_ss", KBF16_SS, 256, KB / 2}};
    for (const Case& cs : cases) {
        c.N = cs.N;
        c.rounds = 2048;
        void (*L)(void*) = nullptr;
        switch (cs.kind) {
            case KI8_SS: L = [](void* v) { auto* c = (Ctx*)v; k_mma<KI8_SS><<<c->sms, 128, (128 + 256) * KB>>>(c->A, c->B, c->N, c->rounds, c->D, c->cyc); }; break;
            case KI8_TS: L = [](void* v) { auto* c = (Ctx*)v; k_mma<KI8_TS><<<c->sms, 128, (128 + 256) * KB>>>(c->A, c->B, c->N, c->rounds, c->D, c->cyc); }; break;
            case KTF32_SS: L = [](void* v) { auto* c = (Ctx*)v; k_mma<KTF32_SS><<<c->sms, 128, (128 + 256) * KB>>>(c->A, c->B, c->N, c->rounds, c->D, c->cyc); }; break;
            default: L = [](void* v) { auto* c = (Ctx*)v; k_mma<KBF16_SS><<<c->sms, 128, (128 + 256) * KB>>>(c->A, c->B, c->N, c->rounds, c->D, c->cyc); }; break;
        }
        const float ms = time_launch(L, &c, 3);
        std::vector<long long> cyc(c.sms);
        CK(cudaMemcpy(cyc.data(), c.cyc, c.sms * 8, cudaMemcpyDeviceToHost));
        long long mx = 0;
        for (auto v : cyc) mx = v > mx ? v : mx;
        const double macs_per_cta = (double)c.rounds * 128.0 * cs.N * cs.k_per_round;
        const long bad = (cs.kind == KI8_SS || cs.kind == KI8_TS) ? check_i8(cs.N) : -1;
        snprintf(buf, sizeof buf,
                 ", \"%s_m128_n%d\": {\"tops\": %.1f, \"macs_per_clk_per_sm\": %.0f, \"cycles_per_mma\": %.1f, "
                 "\"check_mismatches\": %ld}",
                 cs.name, cs.N, 2.0 * macs_per_cta * c.sms / (ms * 1e-3) / 1e12, macs_per_cta / (double)mx,
                 (double)mx / (c.rounds * (KB / 32)), bad);
        js += buf;
        fprintf(stderr, "%s N=%d ms=%.3f cycles=%lld bad=%ld\n", cs.name, cs.N, ms, mx, bad);
    }

    {
        // MN-major layout check at N = 144 (64 + y + pad per level, two levels), 2 K-steps
        const int N = 144, KS = 2, KT = 64;
        std::vector<int8_t> a(128 * KT), b(N * KT);
        for (auto& x : a) x = (int8_t)((rand() % 256) - 128);
        for (auto& x : b) x = (int8_t)((rand() % 256) - 128);
        int8_t *da, *db;
        int32_t* dd;
        CK(cudaMalloc(&da, a.size()));
        CK(cudaMalloc(&db, b.size()));
        CK(cudaMalloc(&dd, 128 * N * 4));
        CK(cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice));
        const int sm = KS * 4096 + KS * 9 * 512;
        CK(cudaFuncSetAttribute(k_mma_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        k_mma_mn<<<1, 128, sm>>>(da, db, N, KS, dd);
        CK(cudaDeviceSynchronize());
        std::vector<int32_t> d(128 * N);
        CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
        long bad = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < N; ++n) {
                int32_t ref = 0;
                for (int k = 0; k < KT; ++k) ref += (int32_t)a[m * KT + k] * (int32_t)b[n * KT + k];
                bad += d[m * N + n] != ref;
            }
        snprintf(buf, sizeof buf, ", \"i8_mn_major_m128_n144_check_mismatches\": %ld", bad);
        js += buf;
        fprintf(stderr, "mn-major N=144 bad=%ld\n", bad);
    }
    js += "}";
    printf("%s\n", js.c_str());
    return 0;
}
