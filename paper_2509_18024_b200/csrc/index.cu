// index.cu -- the rating matrix's dual index built on the device.
//
// The reference builds CSR over users and CSC over items on the host with
// two lexsorts (ratings.py:74-92: order by (user, item), reject the first
// duplicate pair, then order by (item, user)).  Here both orders come from
// one device primitive, "group by key, order by secondary":
//
//   count    per (key, secondary block) segment: hist[key * nb + (sec >> kSecShift)]
//   scan     exclusive prefix of the segment counts (key-major): segment offsets,
//            and ptr[key] = offset of the key's first segment
//   scatter  each entry to its segment (atomic slot; order inside the segment
//            is arbitrary) as one 64-bit word (sec << 32 | value bits)
//   sort     every segment by its secondaries (at most 2^kSecShift distinct
//            values per segment: a warp sort up to 32 words, a presence
//            bitmap + popcount ranks above), split into idx / val
//
// Segments cover disjoint ascending secondary ranges, so each key's run is
// sorted once its segments are.  COO -> CSR uses key = user, sec = item;
// CSR -> CSC uses key = item, sec = user (the row of the CSR entry).  The
// first duplicate pair in (key, sec) order -- the one the reference names --
// is the minimum over duplicated pairs of (key << 32 | sec), found with
// adjacent-word compares after a warp sort, or as an already-set bit of a
// longer segment's presence bitmap.
// Everything is integer work: results are exact and run-to-run identical.

namespace cals {

constexpr int kSecShift = 14;                 // secondary ids per segment: 16384
constexpr int kSegMax = 1 << kSecShift;       // largest duplicate-free segment
constexpr int kIxScanTile = 4096;             // scan: elements per CTA (1024 threads x 4)

__device__ __forceinline__ uint64_t ix_word(uint32_t sec, float v) {
    return ((uint64_t)sec << 32) | (uint64_t)__float_as_uint(v);
}

// ---- count ------------------------------------------------------------------
__global__ void __launch_bounds__(256) ix_count_coo_kernel(const int32_t* __restrict__ keys,
                                                           const int32_t* __restrict__ secs, int64_t nnz, int64_t nb,
                                                           uint32_t* __restrict__ hist) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(hist + (int64_t)__ldg(keys + e) * nb + (__ldg(secs + e) >> kSecShift), 1u);
}

// CSR input: warp per row; the row's entries all share secondary block row >> kSecShift.
__global__ void __launch_bounds__(256) ix_count_csr_kernel(const int64_t* __restrict__ ptr,
                                                           const int32_t* __restrict__ idx, int64_t n_rows, int64_t nb,
                                                           uint32_t* __restrict__ hist) {
    const int lane = threadIdx.x & 31;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += wstride) {
        const int64_t lo = __ldg(ptr + r), hi = __ldg(ptr + r + 1);
        const int64_t sb = r >> kSecShift;
        for (int64_t e = lo + lane; e < hi; e += 32) atomicAdd(hist + (int64_t)__ldg(idx + e) * nb + sb, 1u);
    }
}

// ---- scan (exclusive, u32 counts -> int64 offsets, three phases) -------------
__device__ __forceinline__ int64_t block_scan_excl_i64(int64_t v, int64_t* s_warp, int64_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(CALS_FULL_MASK, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < nw ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(CALS_FULL_MASK, w, o);
            if (lane >= o) w += t;
        }
        if (lane < nw) s_warp[lane] = w;  // inclusive warp prefixes
    }
    __syncthreads();
    total = s_warp[nw - 1];
    return incl - v + (warp ? s_warp[warp - 1] : 0);
}

__global__ void __launch_bounds__(1024) ix_tile_sum_kernel(const uint32_t* __restrict__ hist, int64_t n,
                                                           int64_t* __restrict__ tile_sums) {
    __shared__ int64_t s_warp[32];
    const int64_t base = (int64_t)blockIdx.x * kIxScanTile;
    int64_t v = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t e = base + (int64_t)threadIdx.x * 4 + j;
        v += e < n ? hist[e] : 0u;
    }
    int64_t total;
    block_scan_excl_i64(v, s_warp, total);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// one CTA: exclusive scan of the tile sums in place (n_tiles is at most a few hundred thousand)
__global__ void __launch_bounds__(1024) ix_scan_tiles_kernel(int64_t* __restrict__ tile_sums, int64_t n_tiles) {
    __shared__ int64_t s_warp[32];
    int64_t carry = 0;
    for (int64_t b = 0; b < n_tiles; b += blockDim.x) {
        const int64_t e = b + threadIdx.x;
        const int64_t v = e < n_tiles ? tile_sums[e] : 0;
        int64_t total;
        const int64_t ex = block_scan_excl_i64(v, s_warp, total);
        if (e < n_tiles) tile_sums[e] = carry + ex;
        carry += total;
    }
}

__global__ void __launch_bounds__(1024) ix_scan_apply_kernel(const uint32_t* __restrict__ hist, int64_t n,
                                                             const int64_t* __restrict__ tile_off,
                                                             int64_t* __restrict__ off) {
    __shared__ int64_t s_warp[32];
    const int64_t base = (int64_t)blockIdx.x * kIxScanTile;
    uint32_t c[4];
    int64_t v = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t e = base + (int64_t)threadIdx.x * 4 + j;
        c[j] = e < n ? hist[e] : 0u;
        v += c[j];
    }
    int64_t total;
    int64_t run = tile_off[blockIdx.x] + block_scan_excl_i64(v, s_warp, total);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t e = base + (int64_t)threadIdx.x * 4 + j;
        if (e <= n) off[e] = run;  // off[n] = total count
        run += c[j];
    }
}

// ptr[k] = off[k * nb]  (k = 0 .. n_keys)
__global__ void __launch_bounds__(256) ix_ptr_kernel(const int64_t* __restrict__ off, int64_t n_keys, int64_t nb,
                                                     int64_t* __restrict__ ptr) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= n_keys; k += (int64_t)gridDim.x * blockDim.x)
        ptr[k] = off[k * nb];
}

// ---- scatter ----------------------------------------------------------------
__global__ void __launch_bounds__(256) ix_scatter_coo_kernel(const int32_t* __restrict__ keys,
                                                             const int32_t* __restrict__ secs,
                                                             const float* __restrict__ vals, int64_t nnz, int64_t nb,
                                                             const int64_t* __restrict__ off,
                                                             uint32_t* __restrict__ fill, uint64_t* __restrict__ words) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t sec = (uint32_t)__ldg(secs + e);
        const int64_t seg = (int64_t)__ldg(keys + e) * nb + (sec >> kSecShift);
        const int64_t pos = __ldg(off + seg) + atomicAdd(fill + seg, 1u);
        words[pos] = ix_word(sec, __ldg(vals + e));
    }
}

__global__ void __launch_bounds__(256) ix_scatter_csr_kernel(const int64_t* __restrict__ ptr,
                                                             const int32_t* __restrict__ idx,
                                                             const float* __restrict__ val, int64_t n_rows, int64_t nb,
                                                             const int64_t* __restrict__ off,
                                                             uint32_t* __restrict__ fill, uint64_t* __restrict__ words) {
    const int lane = threadIdx.x & 31;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += wstride) {
        const int64_t lo = __ldg(ptr + r), hi = __ldg(ptr + r + 1);
        const int64_t sb = r >> kSecShift;
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const int64_t seg = (int64_t)__ldg(idx + e) * nb + sb;
            const int64_t pos = __ldg(off + seg) + atomicAdd(fill + seg, 1u);
            words[pos] = ix_word((uint32_t)r, __ldg(val + e));
        }
    }
}

// ---- sort -------------------------------------------------------------------
__device__ __forceinline__ void ix_emit(uint64_t w, int64_t pos, int32_t* __restrict__ out_idx,
                                        float* __restrict__ out_val) {
    out_idx[pos] = (int32_t)(w >> 32);
    out_val[pos] = __uint_as_float((uint32_t)w);
}

__device__ __forceinline__ uint64_t warp_sort_asc(uint64_t v, int lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const uint64_t o = __shfl_xor_sync(CALS_FULL_MASK, v, stride);
            const bool lower = (lane & stride) == 0;
            const bool asc_block = (lane & size) == 0 || size == 32;
            const bool keep_min = (lower == asc_block);
            v = keep_min ? (v < o ? v : o) : (v > o ? v : o);
        }
    }
    return v;
}

// Segments of <= 32 words (thread per segment classifies; the warp sorts the
// small ones together); longer segments are queued for ix_sort_big_kernel.
// dup: min over duplicated pairs of (key << 32 | sec), or ~0.
__global__ void __launch_bounds__(256) ix_sort_small_kernel(const int64_t* __restrict__ off, int64_t n_seg, int64_t nb,
                                                            const uint64_t* __restrict__ words,
                                                            int32_t* __restrict__ out_idx, float* __restrict__ out_val,
                                                            int64_t* __restrict__ big_list,
                                                            unsigned long long* __restrict__ big_count,
                                                            unsigned long long* __restrict__ dup) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x; s0 < n_seg; s0 += stride) {
        const int64_t seg = s0 + threadIdx.x;
        int64_t lo = 0, len = 0;
        if (seg < n_seg) {
            lo = off[seg];
            len = off[seg + 1] - lo;
        }
        if (len == 1) ix_emit(words[lo], lo, out_idx, out_val);
        if (len > 32) big_list[atomicAdd(big_count, 1ull)] = seg;
        uint32_t todo = __ballot_sync(CALS_FULL_MASK, len >= 2 && len <= 32);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t slo = __shfl_sync(CALS_FULL_MASK, lo, src);
            const int slen = (int)__shfl_sync(CALS_FULL_MASK, len, src);
            const int64_t sseg = __shfl_sync(CALS_FULL_MASK, seg, src);
            uint64_t v = lane < slen ? words[slo + lane] : ~0ull;
            v = warp_sort_asc(v, lane);
            const uint64_t prev = __shfl_up_sync(CALS_FULL_MASK, v, 1);
            if (lane < slen) {
                ix_emit(v, slo + lane, out_idx, out_val);
                if (lane > 0 && (prev >> 32) == (v >> 32))
                    atomicMin(dup, ((unsigned long long)(sseg / nb) << 32) | (v >> 32));
            }
        }
    }
}

// One CTA per queued segment (> 32 words).  A segment's secondaries are
// distinct values inside one kSegMax-wide block, so the segment is sorted by
// presence: a kSegMax-bit bitmap of its secondaries (shared memory), an
// exclusive prefix of the word popcounts, and every word goes straight to the
// rank of its secondary -- O(len + kSegMax / 32), two passes over the words.
// A bit found already set is a duplicate pair: the smallest one is reported
// (the outputs of such a segment do not matter, the build fails).
__global__ void __launch_bounds__(1024) ix_sort_big_kernel(const int64_t* __restrict__ off, int64_t nb,
                                                           const int64_t* __restrict__ big_list,
                                                           const unsigned long long* __restrict__ big_count,
                                                           const uint64_t* __restrict__ words,
                                                           int32_t* __restrict__ out_idx, float* __restrict__ out_val,
                                                           unsigned long long* __restrict__ dup) {
    constexpr int NW = kSegMax / 32;  // bitmap words
    __shared__ uint32_t s_bits[NW];
    __shared__ int s_pre[NW];
    __shared__ int s_wsum[32];
    __shared__ int s_dup;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n_big = (int64_t)*big_count;
    for (int64_t b = blockIdx.x; b < n_big; b += gridDim.x) {
        const int64_t seg = big_list[b];
        const int64_t lo = off[seg];
        const int64_t len = off[seg + 1] - lo;
        const uint64_t key_hi = (unsigned long long)(seg / nb) << 32;
        __syncthreads();
        for (int i = tid; i < NW; i += nt) s_bits[i] = 0u;
        if (tid == 0) s_dup = 0;
        __syncthreads();
        for (int64_t i = tid; i < len; i += nt) {
            const uint32_t sec = (uint32_t)(words[lo + i] >> 32);
            const uint32_t rel = sec & (kSegMax - 1);
            const uint32_t m = 1u << (rel & 31);
            if (atomicOr(&s_bits[rel >> 5], m) & m) {
                atomicMin(dup, key_hi | sec);
                s_dup = 1;
            }
        }
        __syncthreads();
        if (s_dup) continue;  // uniform
        // exclusive prefix of the popcounts (NW = 512 words, 1024 threads: one word per thread)
        int v = tid < NW ? __popc(s_bits[tid]) : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(CALS_FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int w = lane < (nt >> 5) ? s_wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(CALS_FULL_MASK, w, o);
                if (lane >= o) w += t;
            }
            s_wsum[lane] = w;  // inclusive prefix over warps
        }
        __syncthreads();
        if (tid < NW) s_pre[tid] = incl - v + (warp ? s_wsum[warp - 1] : 0);
        __syncthreads();
        for (int64_t i = tid; i < len; i += nt) {
            const uint64_t w = words[lo + i];
            const uint32_t rel = (uint32_t)(w >> 32) & (kSegMax - 1);
            const int rank = s_pre[rel >> 5] + __popc(s_bits[rel >> 5] & ((1u << (rel & 31)) - 1u));
            ix_emit(w, lo + rank, out_idx, out_val);
        }
    }
}

}  // namespace cals

namespace {

struct IxWs {
    uint32_t* hist;
    int64_t* off;
    int64_t* tiles;
    int64_t* big_list;
    unsigned long long* counters;  // [0] big_count, [1] dup
    uint64_t* words;
    size_t total;
};

IxWs ix_layout(void* base, int64_t n_keys, int64_t n_sec, int64_t nnz) {
    const int64_t nb = std::max<int64_t>(1, (n_sec + kSegMax - 1) / kSegMax);
    const int64_t n_seg = std::max<int64_t>(1, n_keys * nb);
    const int64_t n_tiles = (n_seg + 1 + kIxScanTile - 1) / kIxScanTile;
    IxWs w{};
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o += (bytes + 255) & ~(size_t)255;
        return static_cast<char*>(base) + at;
    };
    w.hist = reinterpret_cast<uint32_t*>(take((size_t)n_seg * 4));
    w.off = reinterpret_cast<int64_t*>(take((size_t)(n_seg + 1) * 8));
    w.tiles = reinterpret_cast<int64_t*>(take((size_t)n_tiles * 8));
    w.big_list = reinterpret_cast<int64_t*>(take((size_t)n_seg * 8));
    w.counters = reinterpret_cast<unsigned long long*>(take(16));
    w.words = reinterpret_cast<uint64_t*>(take((size_t)std::max<int64_t>(nnz, 1) * 8));
    w.total = o;
    return w;
}

// count -> scan -> scatter -> sort, shared by both entry points
template <typename Count, typename Scatter>
int ix_group(Count count, Scatter scatter, int64_t n_keys, int64_t n_sec, int64_t nnz, int64_t* ptr, int32_t* out_idx,
             float* out_val, void* ws, size_t ws_bytes, cudaStream_t st) {
    const int64_t nb = std::max<int64_t>(1, (n_sec + kSegMax - 1) / kSegMax);
    const int64_t n_seg = std::max<int64_t>(1, n_keys * nb);
    IxWs w = ix_layout(ws, n_keys, n_sec, nnz);
    if (ws_bytes < w.total) return CALS_ERR_WORKSPACE;
    const int sms = dev().sms;
    const int grid = sms * 8;
    cudaMemsetAsync(w.hist, 0, (size_t)n_seg * 4, st);
    cudaMemsetAsync(w.counters, 0, 8, st);
    cudaMemsetAsync(w.counters + 1, 0xFF, 8, st);
    {
        ProfScope ps("ix_count", st);
        count(w.hist, nb, grid, st);
    }
    const int64_t n_tiles = (n_seg + 1 + kIxScanTile - 1) / kIxScanTile;
    {
        ProfScope ps("ix_scan", st);
        ix_tile_sum_kernel<<<(unsigned)n_tiles, 1024, 0, st>>>(w.hist, n_seg, w.tiles);
        ix_scan_tiles_kernel<<<1, 1024, 0, st>>>(w.tiles, n_tiles);
        ix_scan_apply_kernel<<<(unsigned)n_tiles, 1024, 0, st>>>(w.hist, n_seg, w.tiles, w.off);
        ix_ptr_kernel<<<(unsigned)std::min<int64_t>((n_keys + 256) / 256, grid), 256, 0, st>>>(w.off, n_keys, nb, ptr);
    }
    cudaMemsetAsync(w.hist, 0, (size_t)n_seg * 4, st);  // fill cursors
    {
        ProfScope ps("ix_scatter", st);
        scatter(w.off, w.hist, w.words, nb, grid, st);
    }
    {
        ProfScope ps("ix_sort", st);
        ix_sort_small_kernel<<<(unsigned)std::min<int64_t>((n_seg + 255) / 256, grid), 256, 0, st>>>(
            w.off, n_seg, nb, w.words, out_idx, out_val, w.big_list, w.counters, w.counters + 1);
        ix_sort_big_kernel<<<sms * 2, 1024, 0, st>>>(w.off, nb, w.big_list, w.counters, w.words, out_idx, out_val,
                                                  w.counters + 1);
    }
    return cuda_status("dual-index build");
}

}  // namespace

extern "C" {

size_t cals_index_workspace_bytes(int64_t n_keys, int64_t n_sec, int64_t nnz) {
    if (n_keys < 0 || n_sec < 0 || nnz < 0) return 0;
    return ix_layout(nullptr, n_keys, n_sec, nnz).total;
}

int cals_coo_to_csr(const int32_t* keys, const int32_t* secs, const float* vals, int64_t nnz, int64_t n_keys,
                    int64_t n_sec, int64_t* ptr, int32_t* out_idx, float* out_val, uint64_t* dup_out, void* ws,
                    size_t ws_bytes, void* stream) {
    if (nnz < 0 || n_keys < 0 || n_sec < 0 || n_keys > INT32_MAX || n_sec > INT32_MAX || !ptr || !dup_out || !ws)
        return CALS_ERR_ARG;
    if (nnz > 0 && (!keys || !secs || !vals || !out_idx || !out_val)) return CALS_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto count = [&](uint32_t* hist, int64_t nb, int grid, cudaStream_t s) {
        if (nnz) ix_count_coo_kernel<<<grid, 256, 0, s>>>(keys, secs, nnz, nb, hist);
    };
    auto scatter = [&](const int64_t* off, uint32_t* fill, uint64_t* words, int64_t nb, int grid, cudaStream_t s) {
        if (nnz) ix_scatter_coo_kernel<<<grid, 256, 0, s>>>(keys, secs, vals, nnz, nb, off, fill, words);
    };
    const int rc = ix_group(count, scatter, n_keys, n_sec, nnz, ptr, out_idx, out_val, ws, ws_bytes, st);
    if (rc) return rc;
    IxWs w = ix_layout(ws, n_keys, n_sec, nnz);
    cudaMemcpyAsync(dup_out, w.counters + 1, 8, cudaMemcpyDeviceToDevice, st);
    return cuda_status("cals_coo_to_csr");
}

int cals_csr_to_csc(const int64_t* ptr, const int32_t* idx, const float* val, int64_t n_rows, int64_t n_cols,
                    int64_t nnz, int64_t* col_ptr, int32_t* col_idx, float* col_val, void* ws, size_t ws_bytes,
                    void* stream) {
    if (nnz < 0 || n_rows < 0 || n_cols < 0 || n_rows > INT32_MAX || n_cols > INT32_MAX || !ptr || !col_ptr || !ws)
        return CALS_ERR_ARG;
    if (nnz > 0 && (!idx || !val || !col_idx || !col_val)) return CALS_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto count = [&](uint32_t* hist, int64_t nb, int grid, cudaStream_t s) {
        if (nnz) ix_count_csr_kernel<<<grid, 256, 0, s>>>(ptr, idx, n_rows, nb, hist);
    };
    auto scatter = [&](const int64_t* off, uint32_t* fill, uint64_t* words, int64_t nb, int grid, cudaStream_t s) {
        if (nnz) ix_scatter_csr_kernel<<<grid, 256, 0, s>>>(ptr, idx, val, n_rows, nb, off, fill, words);
    };
    return ix_group(count, scatter, n_cols, n_rows, nnz, col_ptr, col_idx, col_val, ws, ws_bytes, st);
}

}  // extern "C"
