// abi.cu -- extern "C" boundary: host planner, workspace sizing, launchers.
// See include/coreals_b200.h for the contract of every entry point.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <utility>
#include <vector>

#include "coreals_b200.h"
#include "sweep_common.cuh"


using namespace cals;

namespace {

constexpr size_t kSmemBudget = 224 * 1024;  // dynamic shared memory per CTA (B200 opt-in max is 227 KB)
constexpr int kQSsmall = 4096, kQSbig = 8192;
constexpr int kItemRowsMin = 16384;  // slice rows per work item (sweep on the 500M config: 4096 -> 16384 = -2.4 %)

thread_local char g_err[256] = "";

// explicit tuning (cals_set_tuning); zero / negative fields select the built-in defaults
cals_tuning g_tuning = {0, -1.0f, -1, 0, 0, 0.0f, 0, 0, 0, 0, 0};
int64_t g_big_cand_budget = 0, g_big_tile_budget = 0;  // debug overrides, see cals_debug_big_batch
unsigned long long* g_stats = nullptr;  // debug counters (device), see cals_debug_stats

// ---- optional per-kernel timing (CUDA events on the launch stream) --------
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
struct Prof {
    bool on = false;
    std::vector<ProfRec> live;
    std::vector<cudaEvent_t> pool;
    std::mutex mu;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};
Prof& prof() {
    static Prof p;
    return p;
}
struct ProfScope {
    const char* name;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
        Prof& P = prof();
        if (!P.on) return;
        std::lock_guard<std::mutex> lk(P.mu);
        a = P.get();
        cudaEventRecord(a, st);
    }
    ~ProfScope() {
        if (!a) return;
        Prof& P = prof();
        std::lock_guard<std::mutex> lk(P.mu);
        cudaEvent_t b = P.get();
        cudaEventRecord(b, st);
        P.live.push_back({name, a, b});
    }
};

inline float delta_tab_for(int QS) { return 3.0f * 0.5f / std::sqrt((float)QS); }

constexpr size_t kSmallSmem = 150 * 1024;  // staged-tier CTA budget

inline int budget_of(int64_t n, double rate) {
    volatile double prod = (double)n * rate;
    int64_t s = (int64_t)std::floor(prod + 1e-9);
    return (int)std::max<int64_t>(1, std::min<int64_t>(s, n));
}

int small_nmax(int nf, double rate) {
    int lo = 1, hi = 1 << 15;
    while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (T1Layout(mid, budget_of(mid, rate), nf, kThreads).total <= kSmallSmem) lo = mid; else hi = mid - 1;
    }
    return std::min(lo, 65535);
}

int big_chunk(int nf) {
    // largest power of two whose staged chunk (+ y + kept-row lists) fits ~96 KB
    const size_t per = (size_t)xs_stride(nf) * 4 + 4 + (size_t)nf * 2;
    int ch = 1024;
    while (ch > 64 && (size_t)ch * per > 96 * 1024) ch >>= 1;
    // big_scan: a thread scans chunk / (kThreads / nf) rows, at most 32 (one mask bit each)
    while (ch > 32 && ch / std::max(1, kThreads / nf) > 32) ch >>= 1;
    return ch;
}

size_t big_gram_smem(int nf, int chunk, int gwords = 0) {
    const int sx = xs_stride(nf);
    const int nq = xs_chunks(nf);
    const int threads = big_gram_threads(nq <= 4 ? 1 : (nq <= 8 ? 2 : (nq <= 16 ? 4 : 8)));
    const bool persist = owned_single_round(nf, threads / 32);
    const size_t g = persist ? 0 : align16((size_t)nf * (nf + 1) * 4);
    const size_t lists = persist ? 0 : (size_t)nf * chunk * 2 + (size_t)nf * 4;
    const size_t g64 = persist ? (size_t)nf * (nf + 1) * 8 : 0;  // float64 Gram accumulators
    return align16((size_t)chunk * sx * 4) + align16((size_t)chunk * 4) + g +
           align16((size_t)nf * (chunk / 32) * 4 + lists + (size_t)chunk * gwords * 4) + g64;
}

// rows per staging buffer of the pipelined scan (two buffers; each thread counts <= 32 rows)
// (one row per thread and copy: at most kThreads rows)
int scan_chunk(int nf) {
    const int ch = big_chunk(nf);
    return std::min(kThreads, nf >= 32 ? std::max(32, ch / 2) : ch);
}

size_t big_scan_smem(int nf, int chunk) {
    return align16((size_t)chunk * xs_stride(nf) * 4) + align16((size_t)nf * kHB * 4);
}

int64_t cand_cap(int64_t n, float delta_tab) {
    // must cover the kernel's bracket (table_levels): 2 d n plus level rounding
    const double ks = n > 2048 ? 4.0 : 3.0, kt = n > 2048 ? 1.5 : 1.0;
    const double d = ks * std::sqrt(0.25 / (double)n) + kt * delta_tab + 1.5 / kQ;
    int64_t cap = (int64_t)std::ceil(3.0 * d * (double)n) + 64;
    cap = std::max<int64_t>(cap, 64);
    return std::min<int64_t>(cap, std::max<int64_t>(n, 64));
}

struct Carve {
    char* base;
    size_t off = 0;
    explicit Carve(void* b) : base((char*)b) {}
    template <typename T>
    T* take(size_t count) {
        off = (off + 255) & ~(size_t)255;
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

struct Device {
    int sms = 148;
    size_t smem_optin = 227 * 1024;
    bool init = false;
    cudaStream_t side = nullptr;  // second stream: the staged tier beside the tiled tier
    cudaEvent_t fork = nullptr, join = nullptr;
};
constexpr int kMaxDevices = 64;
// per-device state (SM count, the side stream and its fork/join events), keyed by the
// caller's current device; one host thread per device drives the half-sweeps
Device& dev() {
    static Device d[kMaxDevices];
    static std::mutex mu;
    int id = 0;
    cudaGetDevice(&id);
    if (id < 0 || id >= kMaxDevices) id = 0;
    std::lock_guard<std::mutex> lk(mu);
    Device& D = d[id];
    if (!D.init) {
        cudaDeviceGetAttribute(&D.sms, cudaDevAttrMultiProcessorCount, id);
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, id);
        if (optin > 0) D.smem_optin = (size_t)optin;
        cudaStreamCreateWithFlags(&D.side, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&D.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&D.join, cudaEventDisableTiming);
        D.init = true;
    }
    return D;
}

template <typename K>
void allow_smem(K kernel) {
    static std::mutex mu;
    static std::vector<std::pair<int, const void*>> done;  // the attribute is per device
    std::lock_guard<std::mutex> lk(mu);
    const void* k = reinterpret_cast<const void*>(kernel);
    int id = 0, optin = 0;
    cudaGetDevice(&id);
    if (std::find(done.begin(), done.end(), std::make_pair(id, k)) == done.end()) {
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, id);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
        cudaGetLastError();  // an attribute failure must not masquerade as a launch error
        done.push_back({id, k});
    }
}

template <typename K>
int grid_for(K kernel, size_t smem, int64_t work, int cap_per_sm = 8, int threads = kThreads) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    occ = std::max(1, std::min(occ, cap_per_sm));
    int64_t g = (int64_t)std::min(dev().sms, 160) * occ;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, work));
}

int cuda_status(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
        return CALS_ERR_CUDA;
    }
    return CALS_OK;
}

// Normal-equation batch: rows solved per phase-A/phase-B launch pair.  The budget
// counts 4 bytes per entry but the buffers hold float64: each is <= ~2 GiB.
int64_t gbuf_rows_for(int nf, int64_t rows) {
    const int64_t per = (int64_t)nf * (nf + 1) * 4;
    const int64_t cap = std::max<int64_t>(4096, ((int64_t)1 << 30) / per);
    return std::max<int64_t>(1, std::min<int64_t>(cap, rows));
}

// Tiled-tier batches: rows [r[i], r[i+1]) share one scan/resolve/gram pass,
// bounded so candidate keys and partial normal equations fit the workspace.
struct BigBatches {
    std::vector<int64_t> r;
    int64_t max_rows = 0, max_tiles = 0, max_cand = 0;
};
BigBatches big_batches(const cals_plan* P) {
    BigBatches b;
    b.r.push_back(0);
    if (P->n_big <= 0 || !P->big_tile_ptr_host || !P->big_cand_ptr_host) {
        b.max_rows = P->n_big;
        b.max_tiles = P->n_big_tiles;
        b.max_cand = P->big_cand_total;
        if (P->n_big > 0) b.r.push_back(P->n_big);
        return b;
    }
    const int nf = P->n_f;
    // 8 GiB of candidate keys per batch: fewer, larger batches (500M config: 46 -> ~8 batches per
    // half-sweep, 425 -> 362 ms per iteration, tools/batch_sweep.py); the workspace stays a
    // small share of the 180 GB of HBM (32 GB for both sides of the 500M config)
    const int64_t cand_budget = g_big_cand_budget > 0 ? g_big_cand_budget : (int64_t)1 << 30;
    const int64_t tile_budget = g_big_tile_budget > 0
                                    ? g_big_tile_budget
                                    : std::max<int64_t>(1, ((int64_t)1 << 30) / ((int64_t)nf * (nf + 1) * 4));
    const int64_t* tp = P->big_tile_ptr_host;
    const int64_t* cp = P->big_cand_ptr_host;
    // a batch's normal equations must fit one gbuf pass (single-item rows are written there directly)
    const int64_t row_budget = gbuf_rows_for(nf, P->n_small + P->n_big);
    int64_t start = 0;
    for (int64_t r = 0; r < P->n_big; ++r) {
        const bool over = (cp[r + 1] - cp[start] > cand_budget) || (tp[r + 1] - tp[start] > tile_budget) ||
                          (r + 1 - start > row_budget);
        if (over && r > start) {
            b.r.push_back(r);
            start = r;
        }
    }
    b.r.push_back(P->n_big);
    for (size_t i = 0; i + 1 < b.r.size(); ++i) {
        b.max_rows = std::max(b.max_rows, b.r[i + 1] - b.r[i]);
        b.max_tiles = std::max(b.max_tiles, tp[b.r[i + 1]] - tp[b.r[i]]);
        b.max_cand = std::max(b.max_cand, cp[b.r[i + 1]] - cp[b.r[i]]);
    }
    return b;
}

struct Work {
    uint32_t* qtab;
    int* cnt;
    uint64_t* cand;
    uint64_t* thr;
    double* part;
    double* rss_part;
    int* hist;
    uint32_t* brk;
    int* fcnt;
    unsigned long long* famax;
    double* gbuf;
    int64_t gbuf_rows;
    double* gbuf2;    // staged tier's own normal-equation buffer when both tiers run concurrently
    uint64_t* thr_all;  // [n_rows][nf] selection thresholds (when the caller asks for none)
    float* tc_scale;    // [65] tensor-core Gram digit scales 2^(32 - E) (64 columns + ratings)
    double* tc_alpha;   // [65] 2^E
    int* item_ctr;      // big_gram_tc / big_scan2 work-item counter
    int* icnt;          // [tiles][nf] per-item in-bracket counts (big_scan2)
    int* rf_cnt;        // [4]: per stream, rows deferred to the float64 refinement from the stored
    int64_t* rf_list;   // equations [2][gbuf_rows] (row << 32 | slot), and from the slice:
    int64_t* ir_list;   // [2][gbuf_rows]: systems handed to the mixed-precision solve (counters rf_cnt[4..5])
    int32_t* rs_list;   // [2][n_rows] rows
};

constexpr int kMaxGrid = 160 * 16;  // grid_for never exceeds min(SMs, 160) * 16 CTAs
constexpr int64_t kMaxSolveWarps = 160 * 64;  // solve_warp_kernel grid cap (64 warps per SM)

Work carve(const cals_plan* P, void* ws, size_t* total) {
    Carve c(ws);
    Work w{};
    const int nf = P->n_f;
    w.qtab = c.take<uint32_t>((size_t)nf * (kQ + 1));
    const BigBatches bb = big_batches(P);
    w.cnt = c.take<int>((size_t)bb.max_rows * nf * 2);
    w.cand = c.take<uint64_t>((size_t)bb.max_cand);
    w.thr = c.take<uint64_t>((size_t)bb.max_rows * nf);
    w.part = c.take<double>((size_t)bb.max_tiles * nf * (nf + 1));
    w.rss_part = c.take<double>((size_t)bb.max_tiles);
    w.hist = c.take<int>((size_t)bb.max_rows * nf * kHB);
    w.icnt = c.take<int>((size_t)std::max<int64_t>(bb.max_tiles, 1) * nf);
    w.brk = c.take<uint32_t>((size_t)std::max<int64_t>(P->n_big, 1) * nf);  // all big rows (one calibration pass)
    w.fcnt = c.take<int>((size_t)bb.max_rows * nf);                      // fast_core: kept counts (multi-item rows)
    w.famax = c.take<unsigned long long>((size_t)bb.max_rows * nf);      // fast_core: fallback keys
    w.gbuf_rows = gbuf_rows_for(nf, P->n_small + P->n_big);
    w.gbuf = c.take<double>((size_t)w.gbuf_rows * nf * (nf + 1));
    if (P->n_small > 0 && P->n_big > 0) {  // the two tiers run on two streams
        w.gbuf2 = c.take<double>((size_t)w.gbuf_rows * nf * (nf + 1));
    }
    w.thr_all = c.take<uint64_t>((size_t)std::max<int64_t>(P->n_rows, 1) * nf);
    w.tc_scale = c.take<float>(65);
    w.tc_alpha = c.take<double>(65);
    w.item_ctr = c.take<int>(1);
    w.rf_cnt = c.take<int>(8);
    w.rf_list = c.take<int64_t>((size_t)2 * w.gbuf_rows);
    w.ir_list = c.take<int64_t>((size_t)2 * w.gbuf_rows);
    w.rs_list = c.take<int32_t>((size_t)2 * std::max<int64_t>(P->n_rows, 1));
    *total = c.off + 256;
    return w;
}

template <int NFP>
void launch_solve_fp32(const SweepArgs& A, const int32_t* rows, int64_t count, cudaStream_t st);

// float64 recomputation of the systems the fp32 solve deferred (the count stays
// on the device; one CTA per SM walks the list), then the list is reset
void launch_refine(const SweepArgs& A, cudaStream_t st, bool from_slice) {
    ProfScope ps("refine_kernel", st);
    const size_t sm = refine_smem(A.nf);
    const int* cnt = from_slice ? A.rs_cnt : A.rf_cnt;
    const void* list = from_slice ? static_cast<const void*>(A.rs_list) : static_cast<const void*>(A.rf_list);
    // the per-batch list is usually empty (long rows rarely defer): one CTA per SM keeps that launch cheap
    const int fs = from_slice ? 1 : 0;
    if (A.nf > 64) {  // every system: register-blocked elimination (one 256-thread CTA per SM)
        allow_smem(refine_rb_kernel<128>);
        refine_rb_kernel<128><<<dev().sms, 256, sm, st>>>(A, cnt, list, fs);
    } else if (A.nf > 32) {
        allow_smem(refine_rb_kernel<64>);
        refine_rb_kernel<64><<<dev().sms * (from_slice ? 2 : 1), 256, sm, st>>>(A, cnt, list, fs);
    } else {
        const int per_sm = from_slice ? 4 : 1;
        allow_smem(refine_kernel<256>);
        refine_kernel<256><<<dev().sms * per_sm, 256, sm, st>>>(A, cnt, list, fs);
    }
    cudaMemsetAsync(const_cast<int*>(cnt), 0, sizeof(int), st);
}

template <int NFP>
void launch_solve(const SweepArgs& A, const int32_t* rows, int64_t count, cudaStream_t st) {
    if (count <= 0) return;
    if (A.nf > 64 && A.ill_ratio == 0.f) {  // every system straight to the float64 elimination (comparison)
        ProfScope ps("solve_kernel", st);
        defer_all_kernel<<<(int)std::min<int64_t>((count + 255) / 256, (int64_t)dev().sms * 8), 256, 0, st>>>(
            A, rows, count);
    } else if (A.nf > 64) {  // fp32 register LU + float64 iterative refinement (sweep_solve_ir.cu)
        ProfScope ps("solve_kernel", st);
        allow_smem(solve_ir_kernel<128>);
        solve_ir_kernel<128><<<(int)std::min<int64_t>(count, (int64_t)dev().sms * 3), 128, solve_ir_smem(128), st>>>(
            A, rows, count);
    } else {
        launch_solve_fp32<NFP>(A, rows, count, st);
        if (A.ir_list != nullptr) {  // 32 < n_f <= 64: its ill-conditioned systems, mixed precision
            ProfScope ps("solve_ir_kernel", st);
            allow_smem(solve_ir_kernel<64>);
            solve_ir_kernel<64><<<(int)std::min<int64_t>(count, (int64_t)dev().sms * 8), 64, solve_ir_smem(64), st>>>(
                A, nullptr, 0);
            cudaMemsetAsync(A.ir_cnt, 0, sizeof(int), st);
        }
    }
    launch_refine(A, st, false);  // systems that need this batch's stored equations
}

template <int NFP>
void launch_solve_fp32(const SweepArgs& A, const int32_t* rows, int64_t count, cudaStream_t st) {
    ProfScope ps("solve_kernel", st);
    if constexpr (NFP > 0) {
        const int64_t warps = (count + (32 / NFP) - 1) / (32 / NFP);
        const int64_t blocks = std::min<int64_t>((warps + 7) / 8, kMaxSolveWarps / 8);
        solve_warp_kernel<NFP><<<(int)blocks, 256, 0, st>>>(A, rows, count);
    } else if (A.nf <= 64) {
        const int64_t blocks = std::min<int64_t>((count + 3) / 4, (int64_t)dev().sms * 3 * 4);
        if (A.nf <= 48) {
            const size_t smem = (size_t)4 * 48 * 49 * 4;
            allow_smem(solve_wide_kernel<48>);
            solve_wide_kernel<48><<<(int)blocks, 128, smem, st>>>(A, rows, count);
        } else {
            const size_t smem = (size_t)4 * 64 * 65 * 4;
            allow_smem(solve_wide_kernel<64>);
            solve_wide_kernel<64><<<(int)blocks, 128, smem, st>>>(A, rows, count);
        }
    }
    // n_f > 64: no fp32 LU, every system goes to the float64 pass (launch_solve)
}

template <int CPL>
void launch_gram(const SweepArgs& A, int grid, int threads, size_t smem, cudaStream_t st, const int32_t* rows,
                 int64_t cnt, int N, int S) {
    allow_smem(small_gram_kernel<CPL>);
    small_gram_kernel<CPL><<<grid, threads, smem, st>>>(A, rows, cnt, N, S);
}

template <int CPL>
int gram_grid(size_t smem, int64_t cnt, int threads) {
    allow_smem(small_gram_kernel<CPL>);
    return grid_for(small_gram_kernel<CPL>, smem, cnt, 16, threads);
}

template <int CPL>
int gram_occ(int threads, size_t smem) {
    allow_smem(small_gram_kernel<CPL>);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, small_gram_kernel<CPL>, threads, smem);
    return occ;
}

template <int CPL>
void launch_tiny(const SweepArgs& A, const int32_t* rows, int64_t cnt, cudaStream_t st) {
    const size_t smem = tiny_warp_bytes(A.nf) * kTinyWarps;
    allow_smem(tiny_gram_kernel<CPL>);
    const int64_t blocks = (cnt + kTinyWarps - 1) / kTinyWarps;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tiny_gram_kernel<CPL>, kTinyWarps * 32, smem);
    const int64_t cap = (int64_t)std::min(dev().sms, 160) * std::max(occ, 1);
    tiny_gram_kernel<CPL><<<(int)std::max<int64_t>(1, std::min(blocks, cap)), kTinyWarps * 32, smem, st>>>(A, rows, cnt);
}

template <int NFP>
int launch_small(SweepArgs A, const cals_plan* P, const Work& w, cudaStream_t st) {
    const int nq = xs_chunks(A.nf);
    const int CPL = nq <= 4 ? 1 : (nq <= 8 ? 2 : (nq <= 16 ? 4 : 8));
    for (int g = 0; g < 3; ++g) {
        const int64_t b = P->small_seg[g], e = P->small_seg[g + 1];
        if (e <= b) continue;
        const int N = P->small_seg_maxn[g];
        const int S = P->small_seg_maxs[g];
        if (N <= kTinyN) {  // warp-per-row kernel
            for (int64_t b0 = b; b0 < e; b0 += w.gbuf_rows) {
                const int64_t cnt = std::min<int64_t>(w.gbuf_rows, e - b0);
                {
                    ProfScope ps("tiny_gram_kernel", st);
                    const int32_t* rr = P->small_rows + b0;
                    if (CPL == 1) launch_tiny<1>(A, rr, cnt, st);
                    else if (CPL == 2) launch_tiny<2>(A, rr, cnt, st);
                    else if (CPL == 4) launch_tiny<4>(A, rr, cnt, st);
                    else launch_tiny<8>(A, rr, cnt, st);
                }
                launch_solve<NFP>(A, P->small_rows + b0, cnt, st);
            }
            continue;
        }
        // one big CTA per SM when two would not fit in shared memory
        int threads = N <= 256 ? 128 : 256;
        if (threads == 256 && T1Layout(N, S, A.nf, 256).total > 112 * 1024) threads = 512;
        {
            // wide ranks: more threads per CTA when that raises the resident warps
            auto warps_for = [&](int t) {
                const size_t sm = T1Layout(N, S, A.nf, t).total;
                if (sm > dev().smem_optin) return 0;
                if (CPL == 1) return gram_occ<1>(t, sm) * t / 32;
                if (CPL == 2) return gram_occ<2>(t, sm) * t / 32;
                if (CPL == 4) return gram_occ<4>(t, sm) * t / 32;
                return gram_occ<8>(t, sm) * t / 32;
            };
            const int base = warps_for(threads);
            int best = base, pick = threads;
            for (int t : {256, 512}) {
                const int wv = t > threads ? warps_for(t) : 0;
                if (wv > best) { best = wv; pick = t; }
            }
            if (best >= 2 * base) threads = pick;  // only when occupancy was the limiter
        }
        const size_t smem = T1Layout(N, S, A.nf, threads).total;
        for (int64_t b0 = b; b0 < e; b0 += w.gbuf_rows) {
            const int64_t cnt = std::min<int64_t>(w.gbuf_rows, e - b0);
            {
                ProfScope ps("small_gram_kernel", st);
                const int32_t* rr = P->small_rows + b0;
                if (CPL == 1) launch_gram<1>(A, gram_grid<1>(smem, cnt, threads), threads, smem, st, rr, cnt, N, S);
                else if (CPL == 2) launch_gram<2>(A, gram_grid<2>(smem, cnt, threads), threads, smem, st, rr, cnt, N, S);
                else if (CPL == 4) launch_gram<4>(A, gram_grid<4>(smem, cnt, threads), threads, smem, st, rr, cnt, N, S);
                else launch_gram<8>(A, gram_grid<8>(smem, cnt, threads), threads, smem, st, rr, cnt, N, S);
            }
            launch_solve<NFP>(A, P->small_rows + b0, cnt, st);
        }
    }
    return cuda_status("small tier");
}

template <int CPL, bool FAST = false>
void launch_big_gram(const SweepArgs& A, const BigArgs& B, size_t smem, cudaStream_t st) {
    constexpr int threads = big_gram_threads(CPL);
    if constexpr (CPL >= 4 && !FAST) {
        // float64 accumulation of the SIMT tiled Gram (n_f > 32): long rows of later iterations reach
        // cond ~1e6, where fp32 partial sums miss the 1e-4 contract (at 32 < n_f <= 64 the tensor-core
        // Gram is the default; above 64 this is the tiled Gram)
        {
            allow_smem(big_gram_kernel<CPL, false, true>);
            big_gram_kernel<CPL, false, true>
                <<<grid_for(big_gram_kernel<CPL, false, true>, smem, B.n_tiles, 8, threads), threads, smem, st>>>(A, B);
            return;
        }
    }
    allow_smem(big_gram_kernel<CPL, FAST>);
    big_gram_kernel<CPL, FAST>
        <<<grid_for(big_gram_kernel<CPL, FAST>, smem, B.n_tiles, 8, threads), threads, smem, st>>>(A, B);
}

// method 'fast_core': every row is a tiled row whose kept bits come from the
// whole-source mask; no calibration / scan / resolve.
template <int NFP>
int launch_fast(const SweepArgs& A, const cals_plan* P, const Work& w, const uint32_t* gmask, int gwords,
                cudaStream_t st) {
    const int nf = A.nf;
    const BigBatches bb = big_batches(P);
    const int64_t* tp = P->big_tile_ptr_host;
    for (size_t bi = 0; bi + 1 < bb.r.size(); ++bi) {
        const int64_t r0 = bb.r[bi], r1 = bb.r[bi + 1];
        BigArgs B{};
        B.calib_samples = g_tuning.calib_samples;
        B.calib_z = g_tuning.calib_z;
        B.fold_chunks = g_tuning.fold_chunks;
        B.rows = P->big_rows + r0;
        B.tile_ptr = P->big_tile_ptr + r0;
        B.cand_ptr = P->big_cand_ptr + r0;
        B.n_big = r1 - r0;
        B.tile_base = tp ? tp[r0] : 0;
        B.n_tiles = tp ? tp[r1] - tp[r0] : P->n_big_tiles;
        B.item_rows = P->item_rows;
        B.chunk = big_chunk(nf);
        B.part = w.part;
        B.rss_part = w.rss_part;
        B.tile_row = P->big_tile_row;
        B.row_base = r0;
        B.gmask = gmask;
        B.gwords = gwords;
        B.fcnt = w.fcnt;
        B.famax = w.famax;
        int64_t n_multi = 0;
        if (tp)
            while (n_multi < B.n_big && tp[r0 + n_multi + 1] - tp[r0 + n_multi] >= 2) ++n_multi;
        B.n_multi = tp ? n_multi : B.n_big;
        if (B.n_multi > 0) {
            cudaMemsetAsync(w.fcnt, 0, sizeof(int) * (size_t)B.n_multi * nf, st);
            cudaMemsetAsync(w.famax, 0, sizeof(unsigned long long) * (size_t)B.n_multi * nf, st);
        }
        const size_t gram_smem = big_gram_smem(nf, B.chunk, gwords);
        {
            ProfScope ps("fast_gram_kernel", st);
            const int nq = xs_chunks(nf);
            if (nq <= 4) launch_big_gram<1, true>(A, B, gram_smem, st);
            else if (nq <= 8) launch_big_gram<2, true>(A, B, gram_smem, st);
            else if (nq <= 16) launch_big_gram<4, true>(A, B, gram_smem, st);
            else launch_big_gram<8, true>(A, B, gram_smem, st);
        }
        if (B.n_big > w.gbuf_rows) return CALS_ERR_WORKSPACE;
        if (B.n_multi > 0) {
            {
                ProfScope ps("big_reduce_kernel", st);
                big_reduce_kernel<<<(int)std::min<int64_t>(B.n_multi, (int64_t)dev().sms * 8), kThreads, 0, st>>>(
                    A, B, 0, B.n_multi);
            }
            const int64_t warps = B.n_multi * nf;
            ProfScope ps("fast_fix_kernel", st);
            fast_fix_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)dev().sms * 8)),
                              kThreads, 0, st>>>(A, B);
        }
        launch_solve<NFP>(A, B.rows, B.n_big, st);
        const int rc = cuda_status("fast_core kernels");
        if (rc) return rc;
    }
    return CALS_OK;
}

template <int NFP>
int launch_big(const SweepArgs& A, const cals_plan* P, const Work& w, cudaStream_t st) {
    const int nf = A.nf;
    const BigBatches bb = big_batches(P);
    const int64_t* tp = P->big_tile_ptr_host;
    const int64_t* cp = P->big_cand_ptr_host;
    // row-local bracket levels of every multi-item row, in one launch (the long rows
    // are few per batch, so per-batch launches would leave most SMs idle)
    cudaMemsetAsync(w.brk, 0xFF, sizeof(uint32_t) * (size_t)P->n_big * nf, st);
    {
        int64_t n_calib = 0;
        if (tp)
            while (n_calib < P->n_big && tp[n_calib + 1] - tp[n_calib] >= 2) ++n_calib;
        if (n_calib > 0) {
            BigArgs C{};
            C.calib_samples = g_tuning.calib_samples;
            C.calib_z = g_tuning.calib_z;
            C.rows = P->big_rows;
            C.n_big = n_calib;
            C.brk = w.brk;
            const size_t smem = (size_t)2 * kCalibCols * (kQ + 1) * sizeof(uint32_t);
            allow_smem(big_calib_kernel);
            ProfScope ps("big_calib_kernel", st);
            big_calib_kernel<<<(int)std::min<int64_t>(n_calib, (int64_t)dev().sms * 16), kThreads, smem, st>>>(A, C,
                                                                                                       n_calib);
        }
    }
    // tensor-core Gram (sweep_tc.cu) at 32 < n_f <= 64: digit scales from the quantile table
    const bool tc_gram = nf > 32 && nf <= 64 && g_tuning.gram_path == 0 && A.qtab != nullptr &&
                         P->item_rows <= kTcMaxChunks * kTcKC;
    if (tc_gram && P->n_big > 0) {
        ProfScope ps("tc_scales_kernel", st);
        tc_scales_kernel<<<1, 256, 0, st>>>(A.qtab, nf, A.val, A.nnz, w.tc_scale, w.tc_alpha);
    }
    for (size_t bi = 0; bi + 1 < bb.r.size(); ++bi) {
        const int64_t r0 = bb.r[bi], r1 = bb.r[bi + 1];
        BigArgs B{};
        B.calib_samples = g_tuning.calib_samples;
        B.calib_z = g_tuning.calib_z;
        B.fold_chunks = g_tuning.fold_chunks;
        B.rows = P->big_rows + r0;
        B.tile_ptr = P->big_tile_ptr + r0;
        B.cand_ptr = P->big_cand_ptr + r0;
        B.n_big = r1 - r0;
        B.tile_base = tp ? tp[r0] : 0;
        B.cand_base = cp ? cp[r0] : 0;
        B.n_tiles = tp ? tp[r1] - tp[r0] : P->n_big_tiles;
        B.item_rows = P->item_rows;
        B.chunk = big_chunk(nf);
        B.cnt = w.cnt;
        B.cand = w.cand;
        B.thr = w.thr;
        B.part = w.part;
        B.rss_part = w.rss_part;
        B.hist = w.hist;
        B.icnt = w.icnt;
        B.brk = w.brk + (size_t)r0 * nf;
        B.tile_row = P->big_tile_row;
        B.row_base = r0;
        cudaMemsetAsync(w.cnt, 0, sizeof(int) * (size_t)B.n_big * nf * 2, st);
        // rows spanning >= 2 work items (a prefix: rows are sorted by length) had their
        // bracket levels calibrated above, and their partial normal equations are reduced
        // by big_reduce; single-item rows write theirs straight into gbuf
        int64_t n_calib = 0;
        if (tp)
            while (n_calib < B.n_big && tp[r0 + n_calib + 1] - tp[r0 + n_calib] >= 2) ++n_calib;
        B.n_multi = tp ? n_calib : B.n_big;  // without host offsets every row takes the partial path
        cudaMemsetAsync(w.hist, 0, sizeof(int) * (size_t)B.n_big * nf * kHB, st);
        {
            // pipelined scan: two staging buffers of scan_chunk rows, items claimed from a counter
            BigArgs S = B;
            S.chunk = scan_chunk(nf);
            S.item_ctr = w.item_ctr;
            S.icnt = w.icnt;
            cudaMemsetAsync(w.item_ctr, 0, sizeof(int), st);
            const size_t scan_smem = 2 * align16((size_t)S.chunk * xs_stride(nf) * 4) + align16((size_t)nf * kHB * 4);
            ProfScope ps("big_scan2_kernel", st);
            if (nf == 64 && S.chunk == 64 && xs_stride(nf) == 68) {
                allow_smem(big_scan2_kernel<4, 68, 64>);
                big_scan2_kernel<4, 68, 64><<<grid_for(big_scan2_kernel<4, 68, 64>, scan_smem, B.n_tiles), kThreads,
                                               scan_smem, st>>>(A, S);
            } else {
                allow_smem(big_scan2_kernel<0, 0, 0>);
                big_scan2_kernel<0, 0, 0><<<grid_for(big_scan2_kernel<0, 0, 0>, scan_smem, B.n_tiles), kThreads,
                                             scan_smem, st>>>(A, S);
            }
        }
        {
            const int64_t warps = B.n_big * nf;
            const int64_t blocks = std::min<int64_t>((warps + 7) / 8, (int64_t)dev().sms * 8);
            ProfScope ps("big_resolve_kernel", st);
            big_resolve_kernel<<<(int)std::max<int64_t>(1, blocks), kThreads, 0, st>>>(A, B);
        }
        const size_t gram_smem = big_gram_smem(nf, B.chunk);
        if (tc_gram) {
            ProfScope ps("big_gram_tc_kernel", st);
            allow_smem(big_gram_tc_kernel);
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(B.n_tiles, dev().sms));
            B.item_ctr = w.item_ctr;
            cudaMemsetAsync(w.item_ctr, 0, sizeof(int), st);
            big_gram_tc_kernel<<<grid, kTcThreads, TcSmem::total, st>>>(A, B, w.tc_scale, w.tc_alpha,
                                                                            g_tuning.tc_debug);
        } else {
            ProfScope ps("big_gram_kernel", st);
            const int nq = xs_chunks(nf);
            if (nq <= 4) launch_big_gram<1>(A, B, gram_smem, st);
            else if (nq <= 8) launch_big_gram<2>(A, B, gram_smem, st);
            else if (nq <= 16) launch_big_gram<4>(A, B, gram_smem, st);
            else launch_big_gram<8>(A, B, gram_smem, st);
        }
        if (B.n_big > w.gbuf_rows) return CALS_ERR_WORKSPACE;  // big_batches bounds rows per batch
        if (B.n_multi > 0) {
            ProfScope ps("big_reduce_kernel", st);
            big_reduce_kernel<<<(int)std::min<int64_t>(B.n_multi, (int64_t)dev().sms * 8), kThreads, 0, st>>>(
                A, B, 0, B.n_multi);
        }
        launch_solve<NFP>(A, B.rows, B.n_big, st);
        const int rc = cuda_status("big-row kernels");
        if (rc) return rc;
    }
    return CALS_OK;
}

}  // namespace

extern "C" {

int cals_budget_host(const int64_t* counts, int64_t n_rows, double rate, int32_t* out) {
    if (!counts || !out || n_rows < 0 || !(rate > 0.0) || rate > 1.0) return CALS_ERR_ARG;
    for (int64_t i = 0; i < n_rows; ++i) {
        const int64_t n = counts[i];
        volatile double prod = (double)n * rate;  // multiply, then add (core.py:54): no contraction
        const double f = std::floor(prod + 1e-9);
        int64_t s = (int64_t)f;
        if (s < 1) s = 1;
        if (s > n) s = n;
        out[i] = (int32_t)s;
    }
    return CALS_OK;
}

int cals_plan_build(const int64_t* counts, int64_t n_rows, int n_f, double rate, int32_t* budget,
                    int32_t* small_rows, int32_t* big_rows, int64_t* big_tile_ptr, int64_t* big_cand_ptr,
                    cals_plan* meta) {
    if (!counts || !budget || !small_rows || !big_rows || !big_tile_ptr || !big_cand_ptr || !meta) return CALS_ERR_ARG;
    if (n_f < 1 || n_f > CALS_MAX_NF || n_rows < 0 || n_rows > 0x7fffffff) return CALS_ERR_ARG;
    int rc = cals_budget_host(counts, n_rows, rate, budget);
    if (rc) return rc;
    std::memset(meta, 0, sizeof(*meta));
    meta->n_f = n_f;
    meta->n_rows = n_rows;
    int nmax = small_nmax(n_f, rate);
    if (g_tuning.staged_max_rows > 0) nmax = std::min(nmax, g_tuning.staged_max_rows);
    // above n_f = 64 the solve forms a staged row's residual from its slice (sweep_solve_ir.cu)
    if (n_f > 64) nmax = std::min(nmax, kIrSliceN);
    std::vector<int32_t> small, big;
    for (int64_t i = 0; i < n_rows; ++i) {
        if (counts[i] <= 0) continue;
        if (counts[i] > 0x7fffffffLL) return CALS_ERR_UNSUPPORTED;
        (counts[i] <= nmax ? small : big).push_back((int32_t)i);
    }
    auto by_len = [counts](int32_t a, int32_t b) { return counts[a] != counts[b] ? counts[a] > counts[b] : a < b; };
    std::stable_sort(small.begin(), small.end(), by_len);
    std::stable_sort(big.begin(), big.end(), by_len);
    std::copy(small.begin(), small.end(), small_rows);
    std::copy(big.begin(), big.end(), big_rows);
    meta->n_small = (int64_t)small.size();
    meta->n_big = (int64_t)big.size();
    // segments over the descending list: (256, nmax], (64, 256], [1, 64]
    const int64_t thresholds[3] = {nmax, 256, 64};
    int64_t pos = 0;
    for (int g = 0; g < 3; ++g) {
        const int64_t lo_bound = (g < 2) ? thresholds[g + 1] : 0;
        meta->small_seg[g] = pos;
        meta->small_seg_maxn[g] = pos < (int64_t)small.size() ? (int32_t)counts[small[pos]] : 1;
        meta->small_seg_maxs[g] = 1;
        while (pos < (int64_t)small.size() && counts[small[pos]] > lo_bound) {
            const int32_t sr = budget[small[pos]];
            if (sr < counts[small[pos]]) meta->small_seg_maxs[g] = std::max(meta->small_seg_maxs[g], sr);
            ++pos;
        }
    }
    meta->small_seg[3] = pos;
    // big rows: work items and candidate buffers
    const int chunk = big_chunk(n_f);
    meta->item_rows = std::max(g_tuning.item_rows > 0 ? g_tuning.item_rows : kItemRowsMin, chunk);
    const float dtab = delta_tab_for(kQSbig);
    big_tile_ptr[0] = 0;
    big_cand_ptr[0] = 0;
    for (size_t r = 0; r < big.size(); ++r) {
        const int64_t n = counts[big[r]];
        big_tile_ptr[r + 1] = big_tile_ptr[r] + (n + meta->item_rows - 1) / meta->item_rows;
        big_cand_ptr[r + 1] = big_cand_ptr[r] + (int64_t)n_f * cand_cap(n, dtab);
    }
    meta->n_big_tiles = big_tile_ptr[big.size()];
    meta->big_cand_total = big_cand_ptr[big.size()];
    return CALS_OK;
}

size_t cals_workspace_bytes(const cals_plan* plan) {
    if (!plan) return 0;
    size_t total = 0;
    carve(plan, nullptr, &total);
    return total;
}

int cals_core_half_sweep(const cals_side* side, const cals_plan* P, const float* source, int64_t n_src, int ld_src,
                         int n_f, double lam, float* target, int ld_tgt, const float* target_old, int ld_old,
                         double* rss_rows, double* pen_rows, uint64_t* thr_keys, int32_t* row_status,
                         uint64_t* status_summary, void* ws, size_t ws_bytes, void* stream) {
    if (!side || !P || !source || !target || !row_status) return CALS_ERR_ARG;
    if (rss_rows && (!target_old || ld_old < n_f)) return CALS_ERR_ARG;
    if (n_f < 1 || n_f > CALS_MAX_NF || n_f != P->n_f || ld_src < 4 * xs_chunks(n_f) || (ld_src & 3) || ld_tgt < n_f ||
        lam < 0 || ((uintptr_t)source & 15))
        return CALS_ERR_ARG;
    if ((P->n_small && !P->small_rows) || (P->n_big && (!P->big_rows || !P->big_tile_ptr || !P->big_cand_ptr)) ||
        !P->budget)
        return CALS_ERR_ARG;
    size_t need = 0;
    Work w = carve(P, ws, &need);
    if (ws_bytes < need || (!ws && need > 256)) return CALS_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    (void)dev();
    if (status_summary) cudaMemsetAsync(status_summary, 0, sizeof(uint64_t), st);

    SweepArgs A{};
    A.ptr = side->ptr;
    A.idx = side->idx;
    A.val = side->val;
    A.nnz = side->nnz;
    A.budget = P->budget;
    A.src = source;
    A.n_src = n_src;
    A.ld_src = ld_src;
    A.nf = n_f;
    A.tgt = target;
    A.ld_tgt = ld_tgt;
    A.lam = lam;
    A.tgt_old = target_old;
    A.ld_old = ld_old;
    A.rss_rows = rss_rows;
    A.pen_rows = pen_rows;
    A.thr_keys = thr_keys != nullptr ? thr_keys : w.thr_all;  // the float64 refinement reads them
    A.ill_ratio = g_tuning.ill_ratio >= 0.f ? g_tuning.ill_ratio : ill_ratio_for(n_f);
    A.rf_cnt = w.rf_cnt;
    A.rf_list = w.rf_list;
    A.rs_cnt = w.rf_cnt + 2;
    A.rs_list = w.rs_list;
    A.ir_cnt = w.rf_cnt + 4;
    A.ir_list = (n_f > 32 && n_f <= 64 && A.ill_ratio != 0.f) ? w.ir_list : nullptr;
    A.rf_slice_max = g_tuning.rf_slice_max >= 0 ? g_tuning.rf_slice_max : kRfSliceMax;
    cudaMemsetAsync(w.rf_cnt, 0, 8 * sizeof(int), st);
    A.gbuf = w.gbuf;
    A.stats = g_stats;
    A.status = row_status;
    A.summary = reinterpret_cast<unsigned long long*>(status_summary);
    A.qtab = nullptr;

    // the quantile table (one CTA per column sorting QS samples, ~30 us) pays off only on
    // sides with many ratings; below 2^20 the staged tier's exact column search is cheaper
    // (small config: 160k ratings)
    const int64_t qtab_min = g_tuning.qtab_min_nnz > 0 ? g_tuning.qtab_min_nnz : ((int64_t)1 << 20);
    const bool long_small = P->n_small > 0 && P->small_seg_maxn[0] > 16 && side->nnz >= qtab_min;
    if ((long_small || P->n_big > 0) && side->nnz > 0) {
        const int QS = P->n_big > 0 ? kQSbig : kQSsmall;
        allow_smem(quantile_table_kernel);
        {
            ProfScope ps("quantile_table_kernel", st);
            quantile_table_kernel<<<n_f, 1024, (size_t)QS * 4, st>>>(side->idx, side->nnz, source, ld_src, QS, w.qtab);
        }
        A.qtab = w.qtab;
        A.delta_tab = delta_tab_for(QS);
        int rc = cuda_status("quantile_table_kernel");
        if (rc) return rc;
    }
    int rc = CALS_OK;
    // the staged and tiled tiers touch disjoint rows: with both present the staged
    // tier runs on a second stream (own normal-equation buffer and float64 refinement lists)
    // beside the tiled tier, filling the SMs its low occupancy leaves idle
    const bool both = P->n_small > 0 && P->n_big > 0 && g_tuning.serial_tiers == 0;
    SweepArgs As = A;
    cudaStream_t ss = st;
    if (both) {
        As.gbuf = w.gbuf2;
        As.rf_cnt = w.rf_cnt + 1;
        As.rf_list = w.rf_list + w.gbuf_rows;
        As.rs_cnt = w.rf_cnt + 3;
        As.rs_list = w.rs_list + std::max<int64_t>(P->n_rows, 1);
        As.ir_cnt = w.rf_cnt + 5;
        if (As.ir_list != nullptr) As.ir_list = w.ir_list + w.gbuf_rows;
        ss = dev().side;
        cudaEventRecord(dev().fork, st);
        cudaStreamWaitEvent(ss, dev().fork, 0);
    }
    if (P->n_small > 0) {
        if (n_f <= 8) rc = launch_small<8>(As, P, w, ss);
        else if (n_f <= 16) rc = launch_small<16>(As, P, w, ss);
        else if (n_f <= 32) rc = launch_small<32>(As, P, w, ss);
        else rc = launch_small<0>(As, P, w, ss);
        launch_refine(As, ss, true);  // the tier's deferred short rows, from their slices
        if (both) {
            cudaEventRecord(dev().join, ss);
        }
        if (rc) {
            if (both) cudaStreamWaitEvent(st, dev().join, 0);
            return rc;
        }
    }
    if (P->n_big > 0) {
        if (n_f <= 8) rc = launch_big<8>(A, P, w, st);
        else if (n_f <= 16) rc = launch_big<16>(A, P, w, st);
        else if (n_f <= 32) rc = launch_big<32>(A, P, w, st);
        else rc = launch_big<0>(A, P, w, st);
        launch_refine(A, st, true);
    }
    if (both) cudaStreamWaitEvent(st, dev().join, 0);
    return rc;
}

int cals_plan_build_fast(const int64_t* counts, int64_t n_rows, int n_f, int complete, int32_t* budget,
                         int32_t* rows, int64_t* tile_ptr, int64_t* cand_ptr, cals_plan* meta) {
    if (!counts || !budget || !rows || !tile_ptr || !cand_ptr || !meta) return CALS_ERR_ARG;
    if (n_f < 1 || n_f > CALS_MAX_NF || n_rows < 0 || n_rows > 0x7fffffff) return CALS_ERR_ARG;
    std::memset(meta, 0, sizeof(*meta));
    meta->n_f = n_f;
    meta->n_rows = n_rows;
    std::vector<int32_t> act;
    for (int64_t i = 0; i < n_rows; ++i) {
        if (counts[i] > 0x7fffffffLL) return CALS_ERR_UNSUPPORTED;
        // the solve takes the exact SPD row only for a complete whole-source sketch
        budget[i] = complete ? (int32_t)counts[i] : 0;
        if (counts[i] > 0) act.push_back((int32_t)i);
    }
    std::stable_sort(act.begin(), act.end(),
                     [counts](int32_t a, int32_t b) { return counts[a] != counts[b] ? counts[a] > counts[b] : a < b; });
    std::copy(act.begin(), act.end(), rows);
    meta->n_big = (int64_t)act.size();
    meta->item_rows = std::max(g_tuning.item_rows > 0 ? g_tuning.item_rows : kItemRowsMin, big_chunk(n_f));
    tile_ptr[0] = 0;
    cand_ptr[0] = 0;
    for (size_t r = 0; r < act.size(); ++r) {
        tile_ptr[r + 1] = tile_ptr[r] + (counts[act[r]] + meta->item_rows - 1) / meta->item_rows;
        cand_ptr[r + 1] = 0;
    }
    meta->n_big_tiles = tile_ptr[act.size()];
    return CALS_OK;
}

size_t cals_fast_sketch_workspace_bytes(int n_f) {
    return (size_t)n_f * (2 * sizeof(unsigned long long) + 256 * sizeof(unsigned int)) + 256;
}

int cals_fast_sketch(const float* source, int64_t n_src, int ld_src, int n_f, int64_t s, uint64_t* thr,
                     uint32_t* gmask, void* ws, size_t ws_bytes, void* stream) {
    if (!source || !thr || !gmask || n_f < 1 || n_f > CALS_MAX_NF || ld_src < n_f || n_src < 1 || s < 1 ||
        s > n_src || n_src > 0xFFFFFFFFLL)
        return CALS_ERR_ARG;
    if (!ws || ws_bytes < cals_fast_sketch_workspace_bytes(n_f)) return CALS_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* prefix = reinterpret_cast<unsigned long long*>(thr);
    unsigned long long* above = reinterpret_cast<unsigned long long*>(ws);
    unsigned int* hist = reinterpret_cast<unsigned int*>(above + n_f);
    cudaMemsetAsync(prefix, 0, sizeof(unsigned long long) * n_f, st);
    cudaMemsetAsync(above, 0, sizeof(unsigned long long) * n_f, st);
    cudaMemsetAsync(hist, 0, sizeof(unsigned int) * 256 * n_f, st);
    const int gwords = (n_f + 31) / 32;
    const dim3 hgrid((unsigned)std::min<int64_t>((n_src + 7) / 8, (int64_t)dev().sms * 4), (unsigned)gwords);
    ProfScope ps("fast_sketch_kernels", st);
    for (int pass = 0; pass < 8; ++pass) {
        fast_hist_kernel<<<hgrid, 256, 0, st>>>(source, n_src, ld_src, n_f, pass, prefix, hist);
        fast_pick_kernel<<<(n_f + 7) / 8, 256, 0, st>>>(n_f, s, pass, prefix, above, hist);
    }
    fast_mask_kernel<<<(int)std::min<int64_t>((n_src * gwords + 255) / 256, (int64_t)dev().sms * 16), 256, 0, st>>>(
        source, n_src, ld_src, n_f, prefix, gwords, gmask);
    return cuda_status("cals_fast_sketch");
}

int cals_fast_half_sweep(const cals_side* side, const cals_plan* P, const float* source, int64_t n_src, int ld_src,
                         int n_f, double lam, const uint32_t* gmask, float* target, int ld_tgt,
                         const float* target_old, int ld_old, double* rss_rows, double* pen_rows,
                         int32_t* row_status, uint64_t* status_summary, void* ws, size_t ws_bytes, void* stream) {
    if (!side || !P || !source || !target || !row_status || !gmask) return CALS_ERR_ARG;
    if (rss_rows && (!target_old || ld_old < n_f)) return CALS_ERR_ARG;
    if (n_f < 1 || n_f > CALS_MAX_NF || n_f != P->n_f || ld_src < 4 * xs_chunks(n_f) || (ld_src & 3) || ld_tgt < n_f ||
        lam < 0 || ((uintptr_t)source & 15) || P->n_small != 0)
        return CALS_ERR_ARG;
    if (P->n_big && (!P->big_rows || !P->big_tile_ptr || !P->big_cand_ptr || !P->budget)) return CALS_ERR_ARG;
    size_t need = 0;
    Work w = carve(P, ws, &need);
    if (ws_bytes < need || (!ws && need > 256)) return CALS_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    (void)dev();
    if (status_summary) cudaMemsetAsync(status_summary, 0, sizeof(uint64_t), st);
    SweepArgs A{};
    A.ptr = side->ptr;
    A.idx = side->idx;
    A.val = side->val;
    A.nnz = side->nnz;
    A.budget = P->budget;
    A.src = source;
    A.n_src = n_src;
    A.ld_src = ld_src;
    A.nf = n_f;
    A.tgt = target;
    A.ld_tgt = ld_tgt;
    A.lam = lam;
    A.tgt_old = target_old;
    A.ld_old = ld_old;
    A.rss_rows = rss_rows;
    A.pen_rows = pen_rows;
    A.thr_keys = w.thr_all;
    A.ill_ratio = g_tuning.ill_ratio >= 0.f ? g_tuning.ill_ratio : ill_ratio_for(n_f);
    A.rf_cnt = w.rf_cnt;
    A.rf_list = w.rf_list;
    A.rs_cnt = w.rf_cnt + 2;
    A.rs_list = w.rs_list;
    A.ir_cnt = w.rf_cnt + 4;
    A.ir_list = (n_f > 32 && n_f <= 64 && A.ill_ratio != 0.f) ? w.ir_list : nullptr;
    A.rf_slice_max = 0;  // fast_core rows keep their stored equations (whole-source sketch)
    cudaMemsetAsync(w.rf_cnt, 0, 8 * sizeof(int), st);
    A.gbuf = w.gbuf;
    A.stats = g_stats;
    A.status = row_status;
    A.summary = reinterpret_cast<unsigned long long*>(status_summary);
    if (P->n_big == 0) return CALS_OK;
    const int gwords = (n_f + 31) / 32;
    if (n_f <= 8) return launch_fast<8>(A, P, w, gmask, gwords, st);
    if (n_f <= 16) return launch_fast<16>(A, P, w, gmask, gwords, st);
    if (n_f <= 32) return launch_fast<32>(A, P, w, gmask, gwords, st);
    return launch_fast<0>(A, P, w, gmask, gwords, st);
}

int cals_residual(const cals_side* side, const float* source, int ld_src, int n_f, const float* rows_w, int ld_w,
                  double* rss_rows, void* stream) {
    if (!side || !source || !rows_w || !rss_rows || n_f < 1 || n_f > CALS_MAX_NF || ld_src < 4 * xs_chunks(n_f) ||
        (ld_src & 3) || ((uintptr_t)source & 15) || ld_w < n_f)
        return CALS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((side->n_rows + 7) / 8, (int64_t)dev().sms * 16));
    ProfScope ps("residual_kernel", st);
    residual_kernel<<<(int)blocks, 256, 0, st>>>(side->ptr, side->idx, side->val, side->n_rows, source, ld_src, n_f,
                                                rows_w, ld_w, rss_rows);
    return cuda_status("cals_residual");
}

int cals_sum_f64(const double* x, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream) {
    if (!out || (n > 0 && !x) || !ws || ws_bytes < kRedBlocks * sizeof(double)) return CALS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    double* partials = (double*)ws;
    ProfScope ps("sum_f64", st);
    sum_partial_kernel<<<kRedBlocks, 256, 0, st>>>(x, n, partials);
    finish_sum_kernel<<<1, 256, 0, st>>>(partials, kRedBlocks, out);
    return cuda_status("cals_sum_f64");
}

int cals_weighted_sqnorm(const float* F, int64_t n_rows, int n_f, int ld, const int64_t* ptr, double* out, void* ws,
                         size_t ws_bytes, void* stream) {
    if (!F || !ptr || !out || !ws || ws_bytes < kRedBlocks * sizeof(double) || ld < n_f) return CALS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    double* partials = (double*)ws;
    ProfScope ps("weighted_sqnorm", st);
    sqnorm_partial_kernel<<<kRedBlocks, 256, 0, st>>>(F, n_rows, n_f, ld, ptr, partials);
    finish_sum_kernel<<<1, 256, 0, st>>>(partials, kRedBlocks, out);
    return cuda_status("cals_weighted_sqnorm");
}

size_t cals_ces_sketch_workspace_bytes(int64_t n, int p) {
    return (size_t)p * (size_t)std::max<int64_t>(n, 32) * sizeof(uint64_t) + 256;
}

int cals_ces_sketch(const float* X, int64_t n, int p, int32_t s, int32_t* rows_out, float* vals_out, void* ws,
                    size_t ws_bytes, void* stream) {
    if (!X || !rows_out || !vals_out || n < 1 || p < 1 || s < 1 || s > n || n > 0x7fffffff) return CALS_ERR_ARG;
    if (!ws || ws_bytes < cals_ces_sketch_workspace_bytes(n, p)) return CALS_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = (p * 32 + 255) / 256;
    ces_sketch_kernel<<<blocks, 256, 0, st>>>(X, (int)n, p, s, rows_out, vals_out, (uint64_t*)ws);
    return cuda_status("cals_ces_sketch");
}

int cals_ces_sketch_f64(const double* X, int64_t n, int p, int32_t s, int32_t* rows_out, void* ws, size_t ws_bytes,
                        void* stream) {
    if (!X || !rows_out || n < 1 || p < 1 || s < 1 || s > n || n > 0x7fffffff) return CALS_ERR_ARG;
    if (!ws || ws_bytes < (size_t)n * p) return CALS_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)p);
    ces_rank_f64_kernel<<<grid, 256, 0, st>>>(X, (int)n, p, s, (uint8_t*)ws);
    ces_emit_f64_kernel<<<(p * 32 + 255) / 256, 256, 0, st>>>(X, (int)n, p, s, (const uint8_t*)ws, rows_out);
    return cuda_status("cals_ces_sketch_f64");
}

int cals_update_core(const double* X, int64_t n, int p, const int64_t* col_ptr, const int32_t* rows, const double* y,
                     double lam_n, int complete, double* w_out, int32_t* status_out, void* stream) {
    if (!X || !y || !w_out || !status_out || n < 1 || p < 1 || p > CALS_MAX_NF) return CALS_ERR_ARG;
    if (!complete && (!col_ptr || !rows)) return CALS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t smem = (size_t)(2 * p * (p + 1) + p) * sizeof(double);
    allow_smem(update_core_kernel);
    update_core_kernel<<<1, 256, smem, st>>>(X, (int)n, p, col_ptr, rows, y, lam_n, complete, w_out, status_out);
    return cuda_status("cals_update_core");
}

int cals_predict_entries(const float* U, const float* M, int n_f, int ld_u, int ld_m, const int64_t* users,
                         const int64_t* items, int64_t n, double* out, void* stream) {
    if (!U || !M || !users || !items || !out || n_f < 1 || ld_u < n_f || ld_m < n_f) return CALS_ERR_ARG;
    if (n == 0) return CALS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)dev().sms * 16);
    predict_entries_kernel<<<(int)blocks, 256, 0, st>>>(U, M, n_f, ld_u, ld_m, users, items, n, out);
    return cuda_status("cals_predict_entries");
}

int cals_predict_entries_f64(const double* U, const double* M, int n_f, int ld_u, int ld_m, const int64_t* users,
                             const int64_t* items, int64_t n, double* out, void* stream) {
    if (!U || !M || !users || !items || !out || n_f < 1 || ld_u < n_f || ld_m < n_f) return CALS_ERR_ARG;
    if (n == 0) return CALS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)dev().sms * 16);
    predict_entries_f64_kernel<<<(int)blocks, 256, 0, st>>>(U, M, n_f, ld_u, ld_m, users, items, n, out);
    return cuda_status("cals_predict_entries_f64");
}

int cals_predict_full_f64(const double* U, const double* M, int64_t n_users, int64_t n_items, int n_f, int ld_u,
                          int ld_m, double* out, int64_t ld_out, void* stream) {
    if (!U || !M || !out || n_f < 1 || ld_u < n_f || ld_m < n_f || n_users < 0 || n_items < 0 || ld_out < n_items)
        return CALS_ERR_ARG;
    if (n_users == 0 || n_items == 0) return CALS_OK;
    const int64_t gx = (n_items + 63) / 64, gy = (n_users + 63) / 64;
    if (gy > 65535) return CALS_ERR_UNSUPPORTED;  // > 4M users: call it per block of rows
    predict_full_f64_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, (cudaStream_t)stream>>>(
        U, M, n_users, n_items, n_f, ld_u, ld_m, out, ld_out);
    return cuda_status("cals_predict_full_f64");
}

int cals_rank_metrics(const int64_t* seg_ptr, int64_t n_seg, const int32_t* perm, const double* truths,
                      const double* scores, int k_hit, double threshold, int k_ndcg, double* qual, double* hit,
                      double* ratio, double* used, void* stream) {
    if (!seg_ptr || !perm || !truths || !scores || !qual || !hit || !ratio || !used || n_seg < 0) return CALS_ERR_ARG;
    if (n_seg == 0) return CALS_OK;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n_seg + 7) / 8, (int64_t)dev().sms * 8));
    rank_metrics_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(seg_ptr, n_seg, perm, truths, scores, k_hit,
                                                                      threshold, k_ndcg, qual, hit, ratio, used);
    return cuda_status("cals_rank_metrics");
}

void cals_debug_stats(void* device_counters) { g_stats = (unsigned long long*)device_counters; }
void cals_debug_big_batch(int64_t cand_keys, int64_t tiles) {
    g_big_cand_budget = cand_keys;
    g_big_tile_budget = tiles;
}
void cals_set_tuning(const cals_tuning* t) {
    static const cals_tuning defaults = {0, -1.0f, -1, 0, 0, 0.0f, 0, 0, 0, 0, 0};
    g_tuning = t != nullptr ? *t : defaults;
}
void cals_get_tuning(cals_tuning* t) {
    if (t != nullptr) *t = g_tuning;
}

void cals_profile_enable(int on) {
    Prof& P = prof();
    std::lock_guard<std::mutex> lk(P.mu);
    P.on = on != 0;
}
int cals_profile_enabled(void) {
    Prof& P = prof();
    std::lock_guard<std::mutex> lk(P.mu);
    return P.on ? 1 : 0;
}

int cals_profile_collect(char* buf, size_t len) {
    Prof& P = prof();
    std::lock_guard<std::mutex> lk(P.mu);
    struct Agg {
        const char* name;
        int count;
        double ms;
    };
    std::vector<Agg> agg;
    for (auto& r : P.live) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto it = std::find_if(agg.begin(), agg.end(), [&](const Agg& g) { return std::strcmp(g.name, r.name) == 0; });
        if (it == agg.end()) agg.push_back({r.name, 1, (double)ms});
        else { it->count += 1; it->ms += ms; }
        P.pool.push_back(r.a);
        P.pool.push_back(r.b);
    }
    P.live.clear();
    size_t off = 0;
    if (buf && len) buf[0] = 0;
    for (auto& g : agg) {
        if (!buf || off >= len) break;
        off += (size_t)std::snprintf(buf + off, len - off, "%s %d %.6f\n", g.name, g.count, g.ms);
    }
    return (int)agg.size();
}

const char* cals_strerror(int status) {
    switch (status) {
        case CALS_OK: return "ok";
        case CALS_ERR_ARG: return "invalid argument";
        case CALS_ERR_CUDA: return g_err[0] ? g_err : "CUDA error";
        case CALS_ERR_WORKSPACE: return "workspace too small";
        case CALS_ERR_UNSUPPORTED: return "unsupported shape";
        default: return "unknown status";
    }
}

const char* cals_build_info(void) {
    return "coreals_b200: sm_100a, nvcc " CALS_NVCC_VERSION ", warp sample-select + masked-dense SIMT Gram v1";
}

}  // extern "C"
