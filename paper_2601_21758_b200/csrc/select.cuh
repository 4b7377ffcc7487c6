// select.cuh — warp-level K-th key selection shared by the streaming tick
// (stream.cu) and the Θ sweep (sweep.cu).  Keys are unique nonzero u64
// (score or FIFO high word, ~id low word; common.cuh).
#pragma once
#include "common.cuh"

namespace ewsjf {

// K-th largest of the nonzero keys held in registers (R per lane, 0 = empty;
// requires #nonzero >= K >= 1).  MSB-first search for the largest t with
// #(>= t) >= K, one warp reduction per bit, starting below the keys' common
// prefix.  It stops early, returning t itself, once bits below `stop_bit`
// are reached with #(>= t) <= limit: a valid bound (K real keys >= t) within
// 2^(stop_bit-32) relative of the K-th key's high word, not necessarily a key.
// When #(>= t) hits K exactly the exact K-th key min{key >= t} is returned.
// stop_bit = 0 (or limit = K) gives the exact K-th key.
constexpr int kRegSel = 8;
constexpr int kApproxBit = 40;   // keep 24 bits of the key's high word (s' / ord(arrival))
template <int R>
__device__ __forceinline__ u64 warp_kth_regs(const u64 (&v)[R], int K, int stop_bit = 0, int limit = 0) {
    u64 mx = 0ull, mn = ~0ull;
    int n = 0;
#pragma unroll
    for (int r = 0; r < R; r++)
        if (v[r]) { mx = v[r] > mx ? v[r] : mx; mn = v[r] < mn ? v[r] : mn; n++; }
    mx = warp_max_u64(mx);
    mn = warp_min_u64(mn);
    n = __reduce_add_sync(0xffffffffu, n);
    const u64 diff = mx ^ mn;
    if (!diff) return mx;
    int bit = 63 - __clzll((long long)diff);
    u64 t = mn & ~((bit == 63) ? ~0ull : ((2ull << bit) - 1ull));   // common prefix, low bits clear
    if (t == 0ull) t = 1ull;                                        // keys are nonzero
    int ct = n;                                                     // #(>= t)
    bool exact = false;
    for (; bit >= 0; bit--) {
        if (bit < stop_bit && ct <= limit) break;
        const u64 tt = t | (1ull << bit);
        int c = 0;
#pragma unroll
        for (int r = 0; r < R; r++) c += v[r] >= tt;
        c = __reduce_add_sync(0xffffffffu, c);
        if (c >= K) {
            t = tt;
            ct = c;
            if (c == K) { exact = true; break; }
        }
    }
    if (!exact && bit >= 0) return t;   // early stop: valid bound, ct in [K, limit]
    u64 m = ~0ull;
#pragma unroll
    for (int r = 0; r < R; r++)
        if (v[r] && v[r] >= t) m = v[r] < m ? v[r] : m;
    return warp_min_u64(m);
}
// K-th largest of a[0..n), n <= 32*kRegSel (a shared-memory array); see warp_kth_regs.
__device__ __forceinline__ u64 warp_kth_arr(const u64* a, int n, int K, int stop_bit = 0, int limit = 0) {
    const int lane = threadIdx.x & 31;
    u64 v[kRegSel];
#pragma unroll
    for (int r = 0; r < kRegSel; r++) {
        const int j = lane + 32 * r;
        v[r] = j < n ? a[j] : 0ull;
    }
    return warp_kth_regs<kRegSel>(v, K, stop_bit, limit);
}

// Keep the keys >= t of a[0..n) in place (stable: writes never pass reads); returns the count.
__device__ __forceinline__ int warp_keep_ge(u64* a, int n, u64 t) {
    const int lane = threadIdx.x & 31;
    int outc = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        const u64 v = j < n ? a[j] : 0ull;
        const bool keep = j < n && v >= t;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) a[outc + __popc(m & ((1u << lane) - 1u))] = v;
        outc += __popc(m);
        __syncwarp();
    }
    return outc;
}

}  // namespace ewsjf
