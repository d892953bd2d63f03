// select.cuh -- exact top-s selection (per slice column) on sm_100a.
//
// Restates the reference's per-column selection (_kernels.py:26-96:
// quickselect threshold + strict-then-tied emission, ties to the smallest
// row) as a search for the s-th largest UNIQUE key (common.cuh).  The kept
// set is then exactly {k : key(k) >= T}.
//
// Algorithm: warp-level sample-select.  A candidate set is held as a list
// (slice-row indices whose keys are recomputed from the staged slice, or the
// keys themselves).  Each round sorts a 32-key positional sample with a
// warp bitonic network, brackets the target rank with a binomial margin,
// counts, and compacts the bracket in place.  Every round strictly shrinks
// the candidate range (the bracket ends are candidates), so the loop always
// terminates; the final <= 32 candidates are sorted and indexed directly.
#pragma once
#include "sweep_common.cuh"

namespace cals {


// Candidate list of explicit keys (big rows; may live in global memory).
struct KeyList {
    uint64_t* buf;
    __device__ __forceinline__ uint64_t key(int i) const { return buf[i]; }
};

// Binomial bracket around the estimated sample position of the target.
__device__ __forceinline__ void choose_bracket(int m, int need, int& a, int& b) {
    float p = ((float)need - 0.5f) / (float)m;
    int e = (int)(p * 32.0f);
    e = e < 0 ? 0 : (e > 31 ? 31 : e);
    float sig = sqrtf(32.0f * p * (1.0f - p));
    int D = (int)(2.5f * sig) + 1;
    a = e - D;
    b = e + D;
}

// Warp-level select on a key list (in place).
__device__ uint64_t warp_select_keys(KeyList L, int m, int need, uint64_t lo, uint64_t hi, int lane) {
    while (true) {
        if (m <= 32) return warp_kth_desc(lane < m ? L.key(lane) : 0ull, m, need, lane);
        int pos = (int)(((2ll * lane + 1) * (long long)m) >> 6);
        uint64_t smp = warp_sort_desc(L.key(pos), lane);
        int a, b;
        choose_bracket(m, need, a, b);
        uint64_t nhi = a >= 0 ? __shfl_sync(CALS_FULL_MASK, smp, a) : hi;
        uint64_t nlo = b <= 31 ? __shfl_sync(CALS_FULL_MASK, smp, b) : lo;
        int c_hi = 0, c_in = 0;
        for (int i0 = 0; i0 < m; i0 += 32) {
            int i = i0 + lane;
            bool v = i < m;
            uint64_t kk = v ? L.key(i) : 0ull;
            c_hi += __popc(__ballot_sync(CALS_FULL_MASK, v && kk >= nhi));
            c_in += __popc(__ballot_sync(CALS_FULL_MASK, v && kk >= nlo && kk < nhi));
        }
        uint64_t rlo, rhi;
        int nneed;
        if (c_hi < need && need <= c_hi + c_in) { rlo = nlo; rhi = nhi; nneed = need - c_hi; }
        else if (c_hi >= need) { rlo = nhi; rhi = hi; nneed = need; }
        else { rlo = lo; rhi = nlo; nneed = need - c_hi - c_in; }
        int w = 0;
        for (int i0 = 0; i0 < m; i0 += 32) {
            int i = i0 + lane;
            bool v = i < m;
            uint64_t kk = v ? L.key(i) : 0ull;
            bool in = v && kk >= rlo && kk < rhi;
            uint32_t bal = __ballot_sync(CALS_FULL_MASK, in);
            __syncwarp();
            if (in) L.buf[w + __popc(bal & lanemask_lt())] = kk;
            w += __popc(bal);
        }
        __syncwarp();
        m = w;
        need = nneed;
        lo = rlo;
        hi = rhi;
    }
}

// Column-mode select over a full column of n keys given by a functor
// (key_at(k) for k in [0, n)), restricted to [lo, hi) holding m candidates.
// Used as the fallback when the table bracket of the fast path fails.
// Candidates are compacted into `out` (key list, capacity cap >= 32) once
// the range holds <= cap of them; ordinal sampling keeps the rounds
// balanced even for adversarial (sorted / tied) columns.
template <class KeyAt>
__device__ uint64_t warp_select_column(const KeyAt& key_at, int n, int m, int need, uint64_t lo,
                                       uint64_t hi, uint64_t* out, int cap, int lane) {
    while (true) {
        if (m <= cap) {
            int w = 0;
            for (int k0 = 0; k0 < n; k0 += 32) {
                int k = k0 + lane;
                uint64_t kk = k < n ? key_at(k) : 0ull;
                bool in = k < n && kk >= lo && kk < hi;
                uint32_t bal = __ballot_sync(CALS_FULL_MASK, in);
                if (in) out[w + __popc(bal & lanemask_lt())] = kk;
                w += __popc(bal);
            }
            __syncwarp();
            KeyList L{out};
            return warp_select_keys(L, w, need, lo, hi, lane);
        }
        // ordinal sample: the in-range element with ordinal floor((2j+1)m/64) -> slot j
        int base = 0;
        for (int k0 = 0; k0 < n; k0 += 32) {
            int k = k0 + lane;
            uint64_t kk = k < n ? key_at(k) : 0ull;
            bool in = k < n && kk >= lo && kk < hi;
            uint32_t bal = __ballot_sync(CALS_FULL_MASK, in);
            if (in) {
                long long q = base + __popc(bal & lanemask_lt());
                long long je = (64ll * q) / (2ll * m);
                for (long long j = je - 1; j <= je + 1; ++j) {
                    if (j >= 0 && j < 32 && ((2 * j + 1) * (long long)m) / 64 == q) out[j] = kk;
                }
            }
            base += __popc(bal);
        }
        __syncwarp();
        uint64_t smp = warp_sort_desc(out[lane], lane);
        __syncwarp();
        int a, b;
        choose_bracket(m, need, a, b);
        uint64_t nhi = a >= 0 ? __shfl_sync(CALS_FULL_MASK, smp, a) : hi;
        uint64_t nlo = b <= 31 ? __shfl_sync(CALS_FULL_MASK, smp, b) : lo;
        int c_hi = 0, c_in = 0;
        for (int k0 = 0; k0 < n; k0 += 32) {
            int k = k0 + lane;
            bool v = k < n;
            uint64_t kk = v ? key_at(k) : 0ull;
            v = v && kk >= lo && kk < hi;
            c_hi += __popc(__ballot_sync(CALS_FULL_MASK, v && kk >= nhi));
            c_in += __popc(__ballot_sync(CALS_FULL_MASK, v && kk >= nlo && kk < nhi));
        }
        if (c_hi < need && need <= c_hi + c_in) { lo = nlo; hi = nhi; need -= c_hi; m = c_in; }
        else if (c_hi >= need) { lo = nhi; m = c_hi; }
        else { hi = nlo; need -= c_hi + c_in; m = m - c_hi - c_in; }
    }
}

}  // namespace cals
