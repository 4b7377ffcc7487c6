// partition.cu — Refine-and-Prune (§4.2) on sm_100a: the strategic
// loop's offline optimizer.  Bit-exact with the oracle: integer
// histogram / RLE / prefix sums, and every fp64 decision evaluated with the
// canonical expression and explicit _rn intrinsics (no FMA contraction).
//
//  A1 hist_kernel      counting sort of the history into hist[len] (smem-
//                      privatised sub-histograms, 128-bit loads)
//  A2 rle_* kernels    run-length encode the non-zero bins -> (v, c)[M] and
//                      exclusive int64 prefixes N, S1, S2
//  A3 kmeans kernels   exact 1-D k-means, k <= 3: argmax of the canonical
//                      F(i,j) over all distinct-index cut pairs, ties -> the
//                      lexicographically smallest (i, j) (reading R9)
//  A4 refine_kernel    Eq. 2, level-synchronous: every live segment splits at
//                      every gap with g*(n-1) > alpha*span (R10-R14)
//  A5+A6 prune_kernel  midpoint finalisation (R15) then Eq. 3 greedy merges with
//                      a 32-ary tournament tree over adjacent pairs (R16-R18)
#include <climits>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <vector>
#include "ctx.h"

namespace ewsjf {

constexpr int kHistMax = 1 << 20;       // lengths >= 2^20 take the overflow list (A1 long tail)
constexpr int kOvfCap = 32768;          // over-long history lengths per call (sorted in one CTA's shared memory)
constexpr int kHistSmem = 49152;        // bins privatised in shared memory (192 KB)
constexpr int kHT = 1024;               // threads of the histogram / RLE / refine / prune CTAs
constexpr int kRleChunk = 16384;        // bins per RLE block

struct RpScratch {
    unsigned int* hist;                 // [kHistMax]
    unsigned long long* stat;           // [0] invalid, [1] over, [2] max len, [3..] scratch
    int32_t* ovf;                       // [kOvfCap] history lengths >= kHistMax (unsorted)
    int32_t* v;                         // [kHistMax]
    int64_t* c;                         // [kHistMax]
    int64_t *N, *S1, *S2;               // [kHistMax + 1]
    int64_t* blk;                       // [rle blocks][4]: nonzero, sumc, sumcv, sumcv2 (and prefixes)
    double *t1, *t3;                    // [kHistMax + 1]
    double* kbF;                        // [kmeans blocks] best F
    int64_t* kbI;                       // [kmeans blocks] packed (i << 32 | j)
    int32_t* seg;                       // [kHistMax + 1] segment starts (output of refine)
    int32_t* segend;                    // [kHistMax + 1]
    uint8_t* flag;                      // [kHistMax]
    int32_t* out_i;                     // refine: [0] m, [1] depth; kmeans: [2] t1, [3] t2
    int32_t* q_lo;                      // prune outputs [256]
    int32_t* q_hi;
    int64_t *q_n, *q_s1, *q_s2;
    int64_t* merges;
    // prune working set
    int32_t *plo, *phi_, *pnext, *pprev;
    int64_t *pn, *ps1, *ps2;
    double* tree;                       // 32-ary tournament tree: (U, index) pairs
    int32_t* treei;
    int kblocks;
    int64_t tree_n;
    int32_t* kdp_a;                     // k-means DP argmax table [k][M + 1] (grown on demand)
    int64_t kdp_cap;
    int32_t* kcuts;                     // [256] k-means-only cuts
    int prune_cap;                      // largest m the shared-memory prune holds
    int prune_cap_lg;                   // ... with its leaves in global scratch
    cudaEvent_t ev[6];
};

// ------------------------------------------------------------------ A1 ---
__global__ void __launch_bounds__(kHT, 1)
    hist_kernel(const int32_t* __restrict__ len, int64_t n, unsigned int* hist, unsigned long long* stat,
                int32_t* ovf) {
    extern __shared__ unsigned int sh[];
    for (int i = threadIdx.x; i < kHistSmem; i += kHT) sh[i] = 0u;
    __syncthreads();
    unsigned int bad = 0;
    int mx = 0;
    auto one = [&](int b) {
        if (b < 1) { bad++; return; }
        if (b >= kHistMax) {            // rare (prompts of >= 2^20 tokens): the overflow list
            const unsigned long long i = atomicAdd(&stat[1], 1ull);
            if (ovf && i < (unsigned long long)kOvfCap) ovf[i] = b;
            return;
        }
        mx = b > mx ? b : mx;
        if (b < kHistSmem) atomicAdd(&sh[b], 1u);
        else atomicAdd(&hist[b], 1u);
    };
    const bool al = ((uintptr_t)len & 15) == 0;
    const int64_t stride = (int64_t)gridDim.x * kHT;
    if (al) {
        const int64_t n4 = n / 4;
        const int4* l4 = (const int4*)len;
        for (int64_t i = (int64_t)blockIdx.x * kHT + threadIdx.x; i < n4; i += stride) {
            const int4 q = __ldcs(l4 + i);
            one(q.x); one(q.y); one(q.z); one(q.w);
        }
        for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * kHT + threadIdx.x; i < n; i += stride) one(__ldcs(len + i));
    } else {
        for (int64_t i = (int64_t)blockIdx.x * kHT + threadIdx.x; i < n; i += stride) one(__ldcs(len + i));
    }
    bad = __reduce_add_sync(0xffffffffu, bad);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicAdd(&stat[0], (unsigned long long)bad);
        if (mx) atomicMax(&stat[2], (unsigned long long)mx);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistSmem; i += kHT)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// ------------------------------------------------------------------ A2 ---
// Block b covers bins [1 + b*kRleChunk, ...) up to lmax.  Each thread owns 16
// consecutive bins.  Pass 1: per-block totals; pass 2: scan of the totals
// (one block); pass 3: write v, c and the inclusive prefixes.
__device__ __forceinline__ void block_scan_excl4(int64_t (&x)[4], int64_t (&tot)[4], int64_t* sm) {
    // exclusive scan of 4 int64 fields across the 1024 threads; sm: [32][4]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t inc[4] = {x[0], x[1], x[2], x[3]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int f = 0; f < 4; f++) {
            const int64_t u = __shfl_up_sync(0xffffffffu, inc[f], o);
            if (lane >= o) inc[f] += u;
        }
    }
    if (lane == 31)
#pragma unroll
        for (int f = 0; f < 4; f++) sm[w * 4 + f] = inc[f];
    __syncthreads();
    if (w == 0) {
        int64_t s[4];
#pragma unroll
        for (int f = 0; f < 4; f++) s[f] = sm[lane * 4 + f];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int f = 0; f < 4; f++) {
                const int64_t u = __shfl_up_sync(0xffffffffu, s[f], o);
                if (lane >= o) s[f] += u;
            }
        }
#pragma unroll
        for (int f = 0; f < 4; f++) sm[128 + lane * 4 + f] = s[f];   // inclusive per-warp prefix
    }
    __syncthreads();
#pragma unroll
    for (int f = 0; f < 4; f++) {
        const int64_t warp_excl = w ? sm[128 + (w - 1) * 4 + f] : 0;
        x[f] = warp_excl + inc[f] - x[f];
        tot[f] = sm[128 + 31 * 4 + f];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kHT) rle_count_kernel(const unsigned int* hist, int lmax, int64_t* blk) {
    __shared__ int64_t sm[256];
    const int64_t base = 1 + (int64_t)blockIdx.x * kRleChunk + (int64_t)threadIdx.x * 16;
    int64_t x[4] = {0, 0, 0, 0}, tot[4];
    for (int k = 0; k < 16; k++) {
        const int64_t b = base + k;
        if (b > lmax) break;
        const int64_t c = hist[b];
        if (c) { x[0] += 1; x[1] += c; x[2] += c * b; x[3] += c * b * b; }
    }
    block_scan_excl4(x, tot, sm);
    if (threadIdx.x == 0)
        for (int f = 0; f < 4; f++) blk[(int64_t)blockIdx.x * 4 + f] = tot[f];
}

__global__ void __launch_bounds__(kHT) rle_scan_kernel(int64_t* blk, int nb, int64_t* out_tot) {
    __shared__ int64_t sm[256];
    int64_t carry[4] = {0, 0, 0, 0};
    for (int b0 = 0; b0 < nb; b0 += kHT) {
        const int b = b0 + threadIdx.x;
        int64_t x[4] = {0, 0, 0, 0}, tot[4];
        if (b < nb)
            for (int f = 0; f < 4; f++) x[f] = blk[(int64_t)b * 4 + f];
        block_scan_excl4(x, tot, sm);
        if (b < nb)
            for (int f = 0; f < 4; f++) blk[(int64_t)b * 4 + f] = x[f] + carry[f];
        for (int f = 0; f < 4; f++) carry[f] += tot[f];
    }
    if (threadIdx.x == 0)
        for (int f = 0; f < 4; f++) out_tot[f] = carry[f];
}

__global__ void __launch_bounds__(kHT) rle_write_kernel(const unsigned int* hist, int lmax, const int64_t* blk,
                                                       int32_t* v, int64_t* cc, int64_t* N, int64_t* S1,
                                                       int64_t* S2) {
    __shared__ int64_t sm[256];
    const int64_t base = 1 + (int64_t)blockIdx.x * kRleChunk + (int64_t)threadIdx.x * 16;
    int64_t x[4] = {0, 0, 0, 0}, tot[4];
    for (int k = 0; k < 16; k++) {
        const int64_t b = base + k;
        if (b > lmax) break;
        const int64_t c = hist[b];
        if (c) { x[0] += 1; x[1] += c; x[2] += c * b; x[3] += c * b * b; }
    }
    block_scan_excl4(x, tot, sm);
    int64_t run[4];
    for (int f = 0; f < 4; f++) run[f] = x[f] + blk[(int64_t)blockIdx.x * 4 + f];
    if (blockIdx.x == 0 && threadIdx.x == 0) { N[0] = 0; S1[0] = 0; S2[0] = 0; }
    for (int k = 0; k < 16; k++) {
        const int64_t b = base + k;
        if (b > lmax) break;
        const int64_t c = hist[b];
        if (c) {
            const int64_t j = run[0];
            v[j] = (int32_t)b;
            cc[j] = c;
            run[0] += 1; run[1] += c; run[2] += c * b; run[3] += c * b * b;
            N[j + 1] = run[1]; S1[j + 1] = run[2]; S2[j + 1] = run[3];
        }
    }
}

// A1/A2 long tail: the over-long lengths (>= kHistMax, unsorted in ovf[0..n)) are
// sorted in shared memory (bitonic, one CTA) and run-length encoded; every one of
// them exceeds every histogram length, so their runs are appended after the
// histogram's M0 runs and the prefixes continue from its totals tot[0..3] = (M0,
// N, S1, S2), which are updated in place.  runpos: scratch [kOvfCap + 1].
__global__ void __launch_bounds__(kHT) ovf_rle_kernel(const int32_t* __restrict__ ovf, int n, int64_t* tot,
                                                      int32_t* v, int64_t* cc, int64_t* N, int64_t* S1, int64_t* S2,
                                                      int32_t* runpos) {
    extern __shared__ int32_t so[];                 // [P]
    __shared__ int64_t sm[256];
    __shared__ int s_runs;
    const int tid = threadIdx.x;
    int P = 1;
    while (P < n) P <<= 1;
    for (int i = tid; i < P; i += kHT) so[i] = i < n ? ovf[i] : INT_MAX;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < P; i += kHT) {
                const int l = i ^ j;
                if (l > i) {
                    const int a = so[i], b = so[l];
                    if (((i & k) == 0) == (a > b)) { so[i] = b; so[l] = a; }
                }
            }
            __syncthreads();
        }
    // run starts: thread t owns positions [t*E, (t+1)*E); an exclusive scan of the
    // per-thread start counts numbers the runs
    const int E = (n + kHT - 1) / kHT;
    const int i0 = min(n, tid * E), i1 = min(n, i0 + E);
    int64_t x[4] = {0, 0, 0, 0}, t4[4];
    for (int i = i0; i < i1; i++) x[0] += (i == 0 || so[i] != so[i - 1]);
    block_scan_excl4(x, t4, sm);
    {
        int r = (int)x[0];
        for (int i = i0; i < i1; i++)
            if (i == 0 || so[i] != so[i - 1]) runpos[r++] = i;
        if (tid == 0) { s_runs = (int)t4[0]; runpos[t4[0]] = n; }
    }
    __syncthreads();
    const int runs = s_runs;
    const int64_t M0 = tot[0], N0 = tot[1], A0 = tot[2], B0 = tot[3];
    // runs [r0, r1) of this thread: counts, values, and the S1 / S2 prefixes (block scan)
    const int RE = (runs + kHT - 1) / kHT;
    const int r0 = min(runs, tid * RE), r1 = min(runs, r0 + RE);
    int64_t y[4] = {0, 0, 0, 0}, u4[4];
    for (int r = r0; r < r1; r++) {
        const int64_t c = runpos[r + 1] - runpos[r], b = so[runpos[r]];
        y[0] += c * b;
        y[1] = (int64_t)((unsigned long long)y[1] + (unsigned long long)c * b * b);   // sumsq wraps mod 2^64 past 2^63 (no decision reads S2)
    }
    block_scan_excl4(y, u4, sm);
    int64_t s1 = A0 + y[0], s2 = B0 + y[1];
    if (M0 == 0 && tid == 0) { N[0] = 0; S1[0] = 0; S2[0] = 0; }
    for (int r = r0; r < r1; r++) {
        const int64_t c = runpos[r + 1] - runpos[r], b = so[runpos[r]];
        const int64_t j = M0 + r;
        v[j] = (int32_t)b;
        cc[j] = c;
        s1 += c * b;
        s2 = (int64_t)((unsigned long long)s2 + (unsigned long long)c * b * b);
        N[j + 1] = N0 + runpos[r + 1];
        S1[j + 1] = s1;
        S2[j + 1] = s2;
    }
    __syncthreads();
    if (tid == 0) {
        tot[0] = M0 + runs;
        tot[1] = N0 + n;
        tot[2] = A0 + u4[0];
        tot[3] = (int64_t)((unsigned long long)B0 + (unsigned long long)u4[1]);
    }
}

// ------------------------------------------------------------------ A3 ---
// Canonical pieces: sq(s)/n with s exact in int64, each op rounded once.
__device__ __forceinline__ double sq_over(int64_t s, int64_t n) {
    const double d = (double)s;
    return __ddiv_rn(__dmul_rn(d, d), (double)n);
}

__global__ void kmeans_terms_kernel(const int64_t* N, const int64_t* S1, int64_t M, double* t1, double* t3) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= M; i += (int64_t)gridDim.x * blockDim.x) {
        t1[i] = (i >= 1) ? sq_over(S1[i], N[i]) : 0.0;
        t3[i] = (i <= M - 1) ? sq_over(S1[M] - S1[i], N[M] - N[i]) : 0.0;
    }
}

// Argmax of F over (i, j): lexicographic tie-break = smallest i, then smallest j.
__device__ __forceinline__ bool better(double F, int64_t ij, double bF, int64_t bij) {
    return F > bF || (F == bF && ij < bij);
}

// k = 3: block b handles tiles of kKmTile consecutive i (tile b, b + grid, ...), its
// threads sweep j; each (S1[j], N[j], t3[j]) load serves the tile's kKmTile pairs
// (one load triple per pair made the pair loop load-bound).  One result per block.
constexpr int kKmTile = 8;
__global__ void __launch_bounds__(256) kmeans3_kernel(const int64_t* __restrict__ N, const int64_t* __restrict__ S1,
                                                     const double* __restrict__ t1, const double* __restrict__ t3,
                                                     int64_t M, double* outF, int64_t* outIJ) {
    double bF = -1.0;
    int64_t bij = INT64_MAX;
    for (int64_t i0 = 1 + (int64_t)blockIdx.x * kKmTile; i0 <= M - 2; i0 += (int64_t)gridDim.x * kKmTile) {
        int64_t Ni[kKmTile], Si[kKmTile];
        double ti[kKmTile];
#pragma unroll
        for (int u = 0; u < kKmTile; u++) {
            const int64_t i = min(i0 + u, M - 2);
            Ni[u] = N[i]; Si[u] = S1[i]; ti[u] = t1[i];
        }
        for (int64_t j = i0 + 1 + threadIdx.x; j <= M - 1; j += blockDim.x) {
            const int64_t Sj = S1[j], Nj = N[j];
            const double tj = t3[j];
#pragma unroll
            for (int u = 0; u < kKmTile; u++) {
                const int64_t i = i0 + u;
                if (i > M - 2 || j <= i) continue;
                const double F = __dadd_rn(__dadd_rn(ti[u], sq_over(Sj - Si[u], Nj - Ni[u])), tj);
                const int64_t ij = (i << 32) | j;
                if (better(F, ij, bF, bij)) { bF = F; bij = ij; }
            }
        }
    }
    // block reduce
    __shared__ double sF[256];
    __shared__ int64_t sI[256];
    sF[threadIdx.x] = bF;
    sI[threadIdx.x] = bij;
    __syncthreads();
    for (int s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s && better(sF[threadIdx.x + s], sI[threadIdx.x + s], sF[threadIdx.x], sI[threadIdx.x])) {
            sF[threadIdx.x] = sF[threadIdx.x + s];
            sI[threadIdx.x] = sI[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { outF[blockIdx.x] = sF[0]; outIJ[blockIdx.x] = sI[0]; }
}

// k = 2 (or the final reduction of the per-block results when k = 3).
__global__ void __launch_bounds__(1024) kmeans_final_kernel(const int64_t* N, const int64_t* S1, int64_t M, int k,
                                                           const double* inF, const int64_t* inIJ, int nin,
                                                           int32_t* out) {
    double bF = -1.0;
    int64_t bij = INT64_MAX;
    if (k == 2) {
        for (int64_t i = 1 + threadIdx.x; i <= M - 1; i += blockDim.x) {
            const double F = __dadd_rn(sq_over(S1[i], N[i]), sq_over(S1[M] - S1[i], N[M] - N[i]));
            if (better(F, i, bF, bij)) { bF = F; bij = i; }
        }
    } else {
        for (int b = threadIdx.x; b < nin; b += blockDim.x)
            if (inIJ[b] != INT64_MAX && better(inF[b], inIJ[b], bF, bij)) { bF = inF[b]; bij = inIJ[b]; }
    }
    __shared__ double sF[1024];
    __shared__ int64_t sI[1024];
    sF[threadIdx.x] = bF;
    sI[threadIdx.x] = bij;
    __syncthreads();
    for (int s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s && better(sF[threadIdx.x + s], sI[threadIdx.x + s], sF[threadIdx.x], sI[threadIdx.x])) {
            sF[threadIdx.x] = sF[threadIdx.x + s];
            sI[threadIdx.x] = sI[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (k == 2) { out[2] = (int32_t)sI[0]; out[3] = 0; }
        else { out[2] = (int32_t)(sI[0] >> 32); out[3] = (int32_t)(sI[0] & 0xffffffff); }
    }
}

// ------------------------------------------------------------------ A4 ---
// Level-synchronous Eq. 2 over distinct-index segments.  flag[j] = 1 if a
// segment starts at j.  One CTA; per level: (1) segment starts compacted by a
// block scan of the flags, every index j keeping its segment's ordinal in
// sidx[j]; (2) one thread per segment: n, span and the Eq. 2 threshold
// alpha * span (segments too small or too narrow get -1: final); (3) one thread
// per index j tests the gap (v[j], v[j+1]) of its segment: g * (n - 1) > alpha * span.
// (One warp per segment in (2)-(3) left the few wide coarse clusters of the first
// levels to a handful of warps: 0.74 ms at 1M.)
__global__ void __launch_bounds__(kHT, 1)
    refine_kernel(const int32_t* __restrict__ v, const int64_t* __restrict__ N, int64_t M, double alpha,
                  int min_width, uint8_t* flag, int32_t* seg, int32_t* out, int* segend, int32_t* sidx,
                  double* srhs, double* sscale) {
    __shared__ int s_changed, s_m, s_level;
    __shared__ int wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) { s_level = 1; }
    __syncthreads();
    for (;;) {
        // 1) compact segment starts: seg[0..m) (ascending) ; sidx[j] = segment of j
        __syncthreads();
        if (tid == 0) s_m = 0;
        __syncthreads();
        for (int64_t c0 = 0; c0 < M; c0 += kHT) {
            const int64_t j = c0 + tid;
            const int f = (j < M) ? flag[j] : 0;
            const unsigned b = __ballot_sync(0xffffffffu, f);
            if (lane == 0) wsum[w] = __popc(b);
            __syncthreads();
            if (w == 0) {
                int x = wsum[lane];
                for (int o = 1; o < 32; o <<= 1) { const int u = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += u; }
                wsum[lane] = x;   // inclusive
            }
            __syncthreads();
            const int base = s_m + (w ? wsum[w - 1] : 0);
            const int rank = base + __popc(b & ((1u << lane) - 1u));     // starts before j in the level
            if (f) seg[rank] = (int32_t)j;
            if (j < M) sidx[j] = rank + f - 1;                              // the last start <= j
            __syncthreads();
            if (tid == 0) s_m += wsum[31];
            __syncthreads();
        }
        const int m = s_m;
        // 2) per segment: its end, and the Eq. 2 threshold (or -1: the segment is final)
        for (int k = tid; k < m; k += kHT) {
            const int64_t x = seg[k], y = (k + 1 < m) ? seg[k + 1] : M;
            segend[k] = (int)y;
            const int64_t n = N[y] - N[x];
            const int64_t span = (int64_t)v[y - 1] - (int64_t)v[x];
            const bool fin = n < 2 || span == 0 || span < (int64_t)min_width;
            srhs[k] = fin ? -1.0 : __dmul_rn(alpha, (double)span);
            sscale[k] = (double)(n - 1);
        }
        if (tid == 0) s_changed = 0;
        __syncthreads();
        // 3) per index: new starts after qualifying gaps (marked 2 this level)
        int changed = 0;
        for (int64_t j = tid; j + 1 < M; j += kHT) {
            const int k = sidx[j];
            if (j + 1 >= segend[k]) continue;             // the gap after j leaves the segment
            const double rhs = srhs[k];
            if (rhs < 0.0) continue;
            const int64_t g = (int64_t)v[j + 1] - (int64_t)v[j];
            if (__dmul_rn((double)g, sscale[k]) > rhs) { flag[j + 1] = 2; changed = 1; }
        }
        if (__any_sync(0xffffffffu, changed) && lane == 0) s_changed = 1;
        __syncthreads();
        if (!s_changed) break;
        for (int64_t j = tid; j < M; j += kHT)
            if (flag[j] == 2) flag[j] = 1;
        if (tid == 0) s_level++;
        __syncthreads();
    }
    if (tid == 0) { out[0] = s_m; out[1] = s_level; }
}

// ------------------------------------------------------------- A5 + A6 ---
// One CTA.  Finalisation: B_0 = lo_1, B_i = floor((hi_i + lo_{i+1})/2) + 1,
// B_m = hi_m + 1 (R15).  Pruning: while m > max_queues merge the adjacent pair
// with the smallest (MIN_U) / largest (MAX_U) U, ties -> lowest pair.
// The pair minima live in a 32-ary tournament tree updated by warp 0.
__device__ __forceinline__ double rho_of(int64_t n, int32_t lo, int32_t hi) {
    return __ddiv_rn((double)n, (double)((int64_t)hi - (int64_t)lo));
}
__device__ __forceinline__ double mean_of(int64_t s1, int64_t n) {
    return n > 0 ? __ddiv_rn((double)s1, (double)n) : 0.0;
}
__device__ __forceinline__ double util_of(int64_t nl, int64_t sl, int32_t lol, int32_t hil, int64_t nr, int64_t sr,
                                          int32_t lor, int32_t hir, double eps) {
    const double rl = rho_of(nl, lol, hil), rr = rho_of(nr, lor, hir);
    const double ml = mean_of(sl, nl), mr = mean_of(sr, nr);
    return __ddiv_rn(__dadd_rn(rl, rr), __dadd_rn(fabs(__dsub_rn(mr, ml)), eps));
}

__global__ void __launch_bounds__(kHT, 1)
    prune_kernel(const int32_t* __restrict__ v, const int64_t* __restrict__ N, const int64_t* __restrict__ S1,
                 const int64_t* __restrict__ S2, int64_t M, const int32_t* seg, const int32_t* rout, int max_queues, double eps, int rule, int32_t* plo, int32_t* phi,
                 int32_t* pnext, int32_t* pprev, int64_t* pn, int64_t* ps1, int64_t* ps2, double* tree,
                 int32_t* treei, int32_t* q_lo, int32_t* q_hi, int64_t* q_n, int64_t* q_s1, int64_t* q_s2,
                 int64_t* merges_out, const int32_t* done) {
    if (*done) return;                  // prune_smem_kernel handled this partition
    const int m0 = rout[0];
    const int tid = threadIdx.x, lane = tid & 31;
    // finalisation
    for (int i = tid; i < m0; i += kHT) {
        const int64_t x = seg[i], y = (i + 1 < m0) ? seg[i + 1] : M;
        const int64_t seg_hi = v[y - 1];
        int32_t lo;
        if (i == 0) lo = v[x];
        else {
            const int64_t px = seg[i - 1];
            (void)px;
            const int64_t prev_hi = v[x - 1];
            lo = (int32_t)((prev_hi + (int64_t)v[x]) / 2 + 1);
        }
        const int32_t hi = (i + 1 < m0) ? (int32_t)((seg_hi + (int64_t)v[y]) / 2 + 1) : (int32_t)(seg_hi + 1);
        plo[i] = lo; phi[i] = hi;
        pn[i] = N[y] - N[x]; ps1[i] = S1[y] - S1[x]; ps2[i] = S2[y] - S2[x];
        pnext[i] = i + 1 < m0 ? i + 1 : -1;
        pprev[i] = i - 1;
    }
    __syncthreads();
    // tree: leaves = pairs p (left segment p, right pnext[p]); level sizes by 32
    const bool maxu = rule == 1;
    const double INF = maxu ? -1.0 / 0.0 : 1.0 / 0.0;
    const int npair = m0 - 1;
    int lv_off[6], lv_n[6], nl = 0;
    {
        int off = 0, cnt = npair > 0 ? npair : 1;
        for (;;) {
            lv_off[nl] = off; lv_n[nl] = cnt; nl++;
            off += cnt;
            if (cnt == 1) break;
            cnt = (cnt + 31) / 32;
        }
    }
    auto cmp = [&](double a, int ia, double b, int ib) -> bool {   // a strictly better than b
        if (ia < 0) return false;
        if (ib < 0) return true;
        if (maxu) return a > b || (a == b && ia < ib);
        return a < b || (a == b && ia < ib);
    };
    for (int p = tid; p < npair; p += kHT) {
        tree[p] = util_of(pn[p], ps1[p], plo[p], phi[p], pn[p + 1], ps1[p + 1], plo[p + 1], phi[p + 1], eps);
        treei[p] = p;
    }
    __syncthreads();
    for (int l = 1; l < nl; l++) {   // build
        for (int q = tid; q < lv_n[l]; q += kHT) {
            double bu = INF; int bi = -1;
            for (int c = q * 32; c < min(lv_n[l - 1], q * 32 + 32); c++) {
                const double u = tree[lv_off[l - 1] + c]; const int i = treei[lv_off[l - 1] + c];
                if (cmp(u, i, bu, bi)) { bu = u; bi = i; }
            }
            tree[lv_off[l] + q] = bu; treei[lv_off[l] + q] = bi;
        }
        __syncthreads();
    }
    if (tid >= 32) return;
    // warp 0: sequential merges
    auto update_leaf = [&](int p, double u, int id) {   // set leaf p, then recompute its ancestors
        if (lane == 0) { tree[p] = u; treei[p] = id; }
        __syncwarp();
        int c = p;
        for (int l = 1; l < nl; l++) {
            const int q = c / 32;
            const int cc = q * 32 + lane;
            double bu = INF; int bi = -1;
            if (cc < lv_n[l - 1]) { bu = tree[lv_off[l - 1] + cc]; bi = treei[lv_off[l - 1] + cc]; }
            for (int o = 16; o; o >>= 1) {
                const double ou = __shfl_xor_sync(0xffffffffu, bu, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (cmp(ou, oi, bu, bi)) { bu = ou; bi = oi; }
            }
            if (lane == 0) { tree[lv_off[l] + q] = bu; treei[lv_off[l] + q] = bi; }
            __syncwarp();
            c = q;
        }
    };
    int m = m0;
    int64_t merges = 0;
    while (m > max_queues && m > 1) {
        const int p = treei[lv_off[nl - 1]];         // best pair: left segment p
        const int r = pnext[p];
        // merge r into p
        const int32_t nhi = phi[r];
        const int64_t nn = pn[p] + pn[r], ns1 = ps1[p] + ps1[r], ns2 = ps2[p] + ps2[r];
        const int rn = pnext[r];
        __syncwarp();
        if (lane == 0) {
            phi[p] = nhi; pn[p] = nn; ps1[p] = ns1; ps2[p] = ns2;
            pnext[p] = rn;
            if (rn >= 0) pprev[rn] = p;
        }
        __syncwarp();
        if (r < npair) update_leaf(r, INF, -1);   // the pair keyed by r disappears
        if (rn >= 0)
            update_leaf(p, util_of(nn, ns1, plo[p], nhi, pn[rn], ps1[rn], plo[rn], phi[rn], eps), p);
        else
            update_leaf(p, INF, -1);
        const int q = pprev[p];
        if (q >= 0) update_leaf(q, util_of(pn[q], ps1[q], plo[q], phi[q], nn, ns1, plo[p], nhi, eps), q);
        m--;
        merges++;
    }
    __syncwarp();
    if (lane == 0) {
        int k = 0;
        for (int i = 0; i >= 0 && k < 256; i = pnext[i]) {
            q_lo[k] = plo[i]; q_hi[k] = phi[i]; q_n[k] = pn[i]; q_s1[k] = ps1[i]; q_s2[k] = ps2[i];
            k++;
            if (pnext[i] < 0) break;
        }
        merges_out[0] = merges;
        merges_out[1] = k;
    }
}


// ---- A5 + A6 in shared memory (m <= cap).  Same decisions as prune_kernel:
// U per adjacent pair from the canonical util_of, argmin (MIN_U) / argmax (MAX_U)
// with ties to the lowest pair.  A merged segment is always a run of original
// segments [p, next[p]), so its statistics come from constant per-segment
// prefixes (lo, N, S1 at each original start; prune_prep_kernel) and the only
// mutable state is the linked list (u16 next/prev) and the tournament tree of
// 64-bit order keys (leaves: key only; inner nodes: key + pair index), all in
// shared memory.  One warp merges; a tree node is a 32-way redux.min over keys.
constexpr uint64_t kDead = ~0ull;
constexpr uint16_t kNone = 0xffffu;
constexpr int kPL = 5;
constexpr int kSpec = 7;          // speculative chain-run depth (2*kSpec+1 queues x 2 profiles <= 32 lanes)
// tree fan-out: 128 (4 children per lane) when the leaves are in shared memory,
// 32 when they are read from global scratch (fewer bytes per node on the L2 path)
__host__ __device__ constexpr int prune_fan(bool leaf_global) { return leaf_global ? 32 : 128; }

__global__ void prune_prep_kernel(const int32_t* __restrict__ v, const int64_t* __restrict__ N,
                                  const int64_t* __restrict__ S1, const int32_t* __restrict__ seg, int64_t M,
                                  const int32_t* rout, int32_t* lo, int64_t* nx, int64_t* s1x) {
    const int m0 = rout[0];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= m0; i += gridDim.x * blockDim.x) {
        const int64_t x = i < m0 ? seg[i] : M;
        int32_t l;
        if (i == 0) l = v[x];
        else if (i < m0) l = (int32_t)(((int64_t)v[x - 1] + (int64_t)v[x]) / 2 + 1);
        else l = v[M - 1] + 1;
        lo[i] = l; nx[i] = N[x]; s1x[i] = S1[x];
    }
}

__device__ __forceinline__ uint64_t ukey(double u, bool maxu) {
    const uint64_t b = (uint64_t)__double_as_longlong(u);
    const uint64_t o = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    return maxu ? ~o : o;
}

// smem bytes for m segments (npair = m - 1 leaves)
__host__ __device__ inline size_t prune_smem_bytes(int m, int* nl_out, int* lv_off, int* lv_n, bool leaf_global) {
    const int npair = m > 1 ? m - 1 : 1;
    int nl = 0, off = 0, cnt = npair;
    for (;;) {
        if (lv_off) { lv_off[nl] = off; lv_n[nl] = cnt; }
        if (nl > 0) off += cnt;
        nl++;
        if (cnt == 1) break;
        cnt = (cnt + prune_fan(leaf_global) - 1) / prune_fan(leaf_global);
    }
    if (nl_out) *nl_out = nl;
    // leaves u64[npair] | inner keys u64[off] | inner idx i32[off] | next, prev u16[m + 1]
    size_t b = (leaf_global ? 0 : (size_t)npair * 8) + (size_t)off * 12;
    b = (b + 15) & ~(size_t)15;
    return b + (size_t)(m + 1) * 4 + 16;
}

// LG: leaves in global scratch (read past L1), inner nodes and links in shared
// memory — partitions up to ~50k segments; otherwise everything in shared memory.
template <bool LG>
__global__ void __launch_bounds__(kHT, 1)
    prune_smem_kernel(uint64_t* gleaf, const int32_t* __restrict__ lo, const int64_t* __restrict__ nx, const int64_t* __restrict__ s1x,
                      const int64_t* __restrict__ S2, const int32_t* __restrict__ seg, int64_t M, const int32_t* rout,
                      int cap_m, int max_queues, double eps, int rule, int32_t* q_lo, int32_t* q_hi, int64_t* q_n,
                      int64_t* q_s1, int64_t* q_s2, int64_t* merges_out, int32_t* done) {
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr int kFan = prune_fan(LG), kFanSh = LG ? 5 : 7;
    const int m0 = rout[0];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (LG) {
        if (*done || m0 > cap_m) return;
    } else if (m0 > cap_m) {
        if (tid == 0) *done = 0;
        return;
    }
    // tree levels (static indices after unrolling: kPL levels cover 32^4 > kHistMax leaves)
    int lv_off[kPL], lv_n[kPL], nl = kPL;
    {
        int off = 0, cnt = m0 > 1 ? m0 - 1 : 1;
#pragma unroll
        for (int l = 0; l < kPL; l++) {
            lv_off[l] = off; lv_n[l] = cnt;
            if (l > 0) off += cnt;
            if (cnt == 1 && nl == kPL) nl = l + 1;
            cnt = (cnt + kFan - 1) / kFan;   // kFan = prune_fan(LG)
        }
    }
    const int npair = m0 - 1;
    uint64_t* leaf = LG ? gleaf : (uint64_t*)sm;
    int n_inner = 0;
#pragma unroll
    for (int l = 1; l < kPL; l++)
        if (l < nl) n_inner += lv_n[l];
    uint64_t* ikey = LG ? (uint64_t*)sm : leaf + lv_n[0];  // inner node (l, j) at ikey[lv_off[l] + j]
    int32_t* iidx = (int32_t*)(ikey + n_inner);
    size_t b = (LG ? 0 : (size_t)lv_n[0] * 8) + (size_t)n_inner * 12;
    b = (b + 15) & ~(size_t)15;
    uint16_t* nxt = (uint16_t*)(sm + b);
    uint16_t* prv = nxt + (m0 + 1);
    const bool maxu = rule == 1;
    // segment [a, e) of original segments: n, S1, lo, hi
    auto U = [&](int a, int e, int f) -> uint64_t {    // pair ([a,e), [e,f))
        const int64_t nl_ = __ldg(nx + e) - __ldg(nx + a), sl = __ldg(s1x + e) - __ldg(s1x + a);
        const int64_t nr = __ldg(nx + f) - __ldg(nx + e), sr = __ldg(s1x + f) - __ldg(s1x + e);
        return ukey(util_of(nl_, sl, __ldg(lo + a), __ldg(lo + e), nr, sr, __ldg(lo + e), __ldg(lo + f), eps), maxu);
    };
    for (int i = tid; i <= m0; i += kHT) {
        nxt[i] = (uint16_t)(i < m0 ? i + 1 : kNone);
        prv[i] = (uint16_t)(i > 0 ? i - 1 : kNone);
    }
    for (int p = tid; p < npair; p += kHT) leaf[p] = U(p, p + 1, p + 2);
    if (npair < 1 && tid == 0) leaf[0] = kDead;
    __syncthreads();
    // node (l, j) <- best of its <= 32 children at level l-1 (one warp)
    auto node = [&](int l, int j) {
        if (j >= lv_n[l]) return;                           // warp-uniform
        // kFan children: lane holds kFan/32 consecutive ones (lowest index wins ties locally,
        // then the lowest lane across the warp)
        uint64_t k = kDead;
        int id = -1;
#pragma unroll
        for (int u = 0; u < kFan / 32; u++) {
            const int c = j * kFan + lane * (kFan / 32) + u;
            uint64_t kc = kDead;
            int ic = -1;
            if (c < lv_n[l - 1]) {
                if (l == 1) { kc = LG ? __ldcg(leaf + c) : leaf[c]; ic = kc == kDead ? -1 : c; }
                else { kc = ikey[lv_off[l - 1] + c]; ic = iidx[lv_off[l - 1] + c]; }
            }
            if (kc < k) { k = kc; id = ic; }
        }
        const unsigned hi = (unsigned)(k >> 32), lw = (unsigned)k;
        const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lw : 0xffffffffu);
        const int win = __ffs(__ballot_sync(0xffffffffu, hi == mh && lw == ml)) - 1;
        const int wid = __shfl_sync(0xffffffffu, id, win);
        if (lane == 0) { ikey[lv_off[l] + j] = ((uint64_t)mh << 32) | ml; iidx[lv_off[l] + j] = wid; }
    };
#pragma unroll
    for (int l = 1; l < kPL; l++) {
        if (l < nl)
            for (int j = warp; j < lv_n[l]; j += kHT / 32) node(l, j);
        __syncthreads();
    }
    if (warp != 0) return;
    int off_top = 0;
#pragma unroll
    for (int l = 1; l < kPL; l++)
        if (l == nl - 1) off_top = lv_off[l];
    // Merge chains (exact).  Under Eq. 3 the queue a merge produces nearly always
    // takes part in the next merge (measured: 99.8 % of merges on the 1M heavy
    // history, 100 % on bimodal), so after each tree argmin the merged queue Q is
    // followed: its two pairs (L, Q) and (Q, R) are "dynamic" (kept out of the
    // tree, evaluated directly from the per-segment prefixes), every other pair
    // is static.  Leaves the chain touches are only marked dead (no node
    // updates), so the root is a LOWER bound of the static minimum; a chain step
    // whose best dynamic pair beats the root is exactly Eq. 3's argmin.  Otherwise
    // the nodes over the touched leaf range are recomputed (exact static min S)
    // and the step is decided against S with the lowest-pair tie rule; losing it
    // ends the chain (dynamic pairs back into the tree).  Same merge sequence as
    // one argmin per merge, ~50 tree refreshes per 15k merges.
    auto refresh_range = [&](int x0, int x1) {     // recompute the nodes over leaves [x0, x1]
#pragma unroll
        for (int l = 1; l < kPL; l++) {
            if (l >= nl) break;
            const int j0 = x0 >> (kFanSh * l), j1 = x1 >> (kFanSh * l);
            for (int j = j0; j <= j1; j++) node(l, j);
            __syncwarp();
        }
    };
    auto root_key = [&]() -> uint64_t { return nl > 1 ? ikey[off_top] : (LG ? __ldcg(leaf) : leaf[0]); };
    auto root_idx = [&]() -> int { return nl > 1 ? iidx[off_top] : 0; };
    int m = m0;
    int64_t merges = 0;
    while (m > max_queues && m > 1) {
        int p = root_idx();
        {
            const int r = nxt[p];
            const int rn = nxt[r];                  // m0 = end sentinel
            const int q = prv[p];
            __syncwarp();                           // every lane has read the links before lane 0 writes
            if (lane == 0) {
                nxt[p] = (uint16_t)rn;
                if (rn < m0) prv[rn] = (uint16_t)p;
                if (r < npair) leaf[r] = kDead;
                leaf[p] = kDead;                    // Q's right pair: dynamic
                if (q != kNone) leaf[q] = kDead;    // Q's left pair: dynamic
            }
            __syncwarp();
            m--;
            merges++;
            int d0 = q != kNone ? q : p, d1 = r < npair ? r : p;
            uint64_t lb = root_key();               // stale-low bound of the static minimum
            bool exact = false;
            int dir = -1;                           // direction of the last chain merge: 0 left, 1 right
            while (m > max_queues && m > 1) {
                if (dir >= 0) {
                    // ---- speculative direction run: assume the next kSpec merges all absorb
                    // the neighbour on side `dir` (chains run one way for hundreds of merges:
                    // 600 on average on the 1M heavy history).  Step k's two pairs are
                    // evaluated for all k at once (30 lanes: rho/mean of the 2*kSpec+1 queues
                    // involved, then 14 lanes: the pair utilities); the run is confirmed up to
                    // the first step where the predicted pair is not Eq. 3's strict winner
                    // (beaten by the other dynamic pair, not below the static lower bound lb,
                    // a missing neighbour, or the budget reached) and the rest is left to the
                    // general step below, so the merge sequence is unchanged.
                    const int a0 = p;
                    const int lim = min(kSpec, m - max_queues);
                    // walk: x_t = t-th queue start on side dir (x_0 = the side's first neighbour)
                    const int fixed_nb = dir == 0 ? nxt[a0] : prv[a0];          // bq (left run) / L (right run)
                    const int fixed_end = dir == 0 ? (fixed_nb < m0 ? nxt[fixed_nb] : m0) : a0;
                    // per lane: queue j = lane >> 1 (0..kSpec-1: Q_j, kSpec..2kSpec-1: N_{j-kSpec}, 2kSpec: F)
                    const int j = lane >> 1;
                    int xs = -1, xe = -1;                   // [xs, xe) of this lane's queue
                    {
                        // x[t] for t = 0..kSpec: left run x_0 = a0, x_{t+1} = prv[x_t];
                        //                        right run x_0 = nxt[a0], x_{t+1} = nxt[x_t]
                        int x = dir == 0 ? a0 : nxt[a0];
                        int xq_s = -1, xn_s = -1, xn_e = -1;
#pragma unroll
                        for (int t = 0; t <= kSpec; t++) {
                            const int xt = x;
                            if (dir == 0) {
                                if (j < kSpec && t == j) xq_s = xt;                      // Q_j = [x_j, bq)
                                if (j >= kSpec && j < 2 * kSpec) {
                                    if (t == j - kSpec + 1) xn_s = xt;                   // N_k = [x_{k+1}, x_k)
                                    if (t == j - kSpec) xn_e = xt;
                                }
                                x = (xt != kNone && xt < m0) ? (int)prv[xt] : (int)kNone;
                            } else {
                                if (j < kSpec && t == j) xq_s = xt;                      // Q_j = [a0, x_j)
                                if (j >= kSpec && j < 2 * kSpec) {
                                    if (t == j - kSpec) xn_s = xt;                       // N_k = [x_k, x_{k+1})
                                    if (t == j - kSpec + 1) xn_e = xt;
                                }
                                x = (xt != kNone && xt < m0) ? (int)nxt[xt] : (int)kNone;
                            }
                        }
                        if (j < kSpec) {
                            if (dir == 0) { xs = xq_s; xe = fixed_nb; } else { xs = a0; xe = xq_s; }
                        } else if (j < 2 * kSpec) {
                            xs = xn_s; xe = xn_e;
                        } else if (j == 2 * kSpec) {
                            if (dir == 0) { xs = fixed_nb; xe = fixed_end; } else { xs = fixed_nb; xe = a0; }
                        }
                    }
                    const bool live = xs >= 0 && xs != kNone && xs < m0 && xe >= 0 && xe != kNone && xe <= m0 && xs < xe;
                    double pv = 0.0;
                    if (lane < 2 * (2 * kSpec + 1) && live) {
                        const int64_t nn = __ldg(nx + xe) - __ldg(nx + xs);
                        if (lane & 1) {
                            const int64_t ss = __ldg(s1x + xe) - __ldg(s1x + xs);
                            pv = nn > 0 ? __ddiv_rn((double)ss, (double)nn) : 0.0;
                        } else {
                            pv = __ddiv_rn((double)nn, (double)((int64_t)__ldg(lo + xe) - (int64_t)__ldg(lo + xs)));
                        }
                    }
                    const unsigned livem = __ballot_sync(0xffffffffu, live && (lane & 1) == 0);
                    // pair lanes u = 0..2kSpec-1: step k = u >> 1; side 0 = the run's pair (N_k with Q_k),
                    // side 1 = the other dynamic pair (Q_k with F).  In the pair's left-right order.
                    const int k = lane >> 1, side = lane & 1;
                    const int qa = 2 * k, na = 2 * (kSpec + k), fa = 2 * (2 * kSpec);
                    int s1l, s2l;                            // profile lanes of the pair's left / right queue
                    if (dir == 0) { s1l = side == 0 ? na : qa; s2l = side == 0 ? qa : fa; }
                    else          { s1l = side == 0 ? qa : fa; s2l = side == 0 ? na : qa; }
                    const double r1 = __shfl_sync(0xffffffffu, pv, s1l & 31), m1 = __shfl_sync(0xffffffffu, pv, (s1l + 1) & 31);
                    const double r2 = __shfl_sync(0xffffffffu, pv, s2l & 31), m2 = __shfl_sync(0xffffffffu, pv, (s2l + 1) & 31);
                    uint64_t ku = kDead;
                    const bool has = lane < 2 * kSpec && ((livem >> s1l) & 1u) && ((livem >> s2l) & 1u);
                    if (lane < 2 * kSpec) {
                        const double u = __ddiv_rn(__dadd_rn(r1, r2), __dadd_rn(fabs(__dsub_rn(m2, m1)), eps));
                        if (has) ku = ukey(u, maxu);
                    }
                    // lane k (< kSpec): does step k go the predicted way?
                    const uint64_t krun = __shfl_sync(0xffffffffu, ku, (2 * lane) & 31);
                    const uint64_t koth = __shfl_sync(0xffffffffu, ku, (2 * lane + 1) & 31);
                    // left run: the run pair is the LEFT pair, wins ties; right run: must beat the left pair strictly
                    const bool wins = dir == 0 ? krun <= koth : krun < koth;
                    const bool okk = lane < lim && krun != kDead && wins && krun < lb;
                    const unsigned okm = __ballot_sync(0xffffffffu, okk);
                    const int kst = __ffs(~okm) - 1;        // confirmed merges (leading ones)
                    if (kst > 0) {
                        __syncwarp();                       // the walk's reads before the commit's writes
                        // commit: the new Q and its links; leaves of every pair touched -> dead
                        if (dir == 0) {
                            // Q = [x_kst, bq): x_kst = start of N_{kst-1} = [x_kst, x_{kst-1})
                            const int newa = __shfl_sync(0xffffffffu, xs, (2 * (kSpec + kst - 1)) & 31);
                            const int nL = prv[newa];                 // the new left neighbour (links of newa intact)
                            // x_0..x_{kst-1} (Q_t's starts, lanes 2t) stop being queue starts
                            if ((lane & 1) == 0 && (lane >> 1) < kst && xs >= 0 && xs < npair) leaf[xs] = kDead;
                            if (lane == 0) {
                                nxt[newa] = (uint16_t)fixed_nb;
                                if (fixed_nb < m0) prv[fixed_nb] = (uint16_t)newa;
                                if (newa < npair) leaf[newa] = kDead;          // (Q, F): dynamic
                                if (nL != kNone && nL < npair) leaf[nL] = kDead;  // (N, Q): dynamic
                            }
                            d0 = min(d0, nL != kNone ? nL : newa);
                            p = newa;
                        } else {
                            // Q = [a0, x_kst): x_kst = end of N_{kst-1} = [x_{kst-1}, x_kst)
                            const int newe = __shfl_sync(0xffffffffu, xe, (2 * (kSpec + kst - 1)) & 31);
                            const int lastabs = __shfl_sync(0xffffffffu, xe, (2 * (kst - 1)) & 31);   // x_{kst-1}
                            // absorbed starts x_0..x_{kst-1} (Q_t's ends, lanes 2t)
                            if ((lane & 1) == 0 && (lane >> 1) < kst && xe >= 0 && xe < npair) leaf[xe] = kDead;
                            if (lane == 0) {
                                nxt[a0] = (uint16_t)newe;
                                if (newe < m0) prv[newe] = (uint16_t)a0;
                                if (a0 < npair) leaf[a0] = kDead;              // (Q, N): dynamic
                            }
                            d1 = max(d1, lastabs < npair ? lastabs : a0);
                        }
                        __syncwarp();
                        m -= kst;
                        merges += kst;
                        exact = false;
                        if (kst == lim && lim == kSpec) continue;   // the whole run held: speculate again
                        if (!(m > max_queues && m > 1)) break;
                    }
                }
                const int a = p, bq = nxt[a], L = prv[a];
                const int c = bq < m0 ? nxt[bq] : m0;
                // lanes 0..5: rho / mean of L = [L, a), Q = [a, bq), R = [bq, c) in parallel (one
                // converged __ddiv_rn each: the canonical rho_of / mean_of); lanes 0 / 1 then form
                // U(L, Q) / U(Q, R) from them (util_of's order).  Lanes 8..13 prefetch the
                // per-segment prefixes ~24 segments beyond both ends into L1.
                double pv = 0.0;
                if (lane < 6) {
                    const int qx = lane >> 1;                   // 0 = L, 1 = Q, 2 = R
                    const int sx = qx == 0 ? L : (qx == 1 ? a : bq);
                    const int ex = qx == 0 ? a : (qx == 1 ? bq : c);
                    const bool live = qx == 0 ? L != kNone : (qx == 1 ? true : bq < m0);
                    if (live) {
                        const int64_t nn = __ldg(nx + ex) - __ldg(nx + sx);
                        if (lane & 1) {                         // mean = S1 / n
                            const int64_t ss = __ldg(s1x + ex) - __ldg(s1x + sx);
                            pv = nn > 0 ? __ddiv_rn((double)ss, (double)nn) : 0.0;
                        } else {                                // rho = n / width
                            pv = __ddiv_rn((double)nn, (double)((int64_t)__ldg(lo + ex) - (int64_t)__ldg(lo + sx)));
                        }
                    }
                } else if (lane >= 8 && lane < 14) {
                    const int side = lane & 1, arr = (lane - 8) >> 1;
                    const int ix = side ? min(c + 24, m0) : max(L == kNone ? 0 : L - 24, 0);
                    const void* ad = arr == 0 ? (const void*)(nx + ix) : arr == 1 ? (const void*)(s1x + ix)
                                                                                  : (const void*)(lo + ix);
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(ad));
                }
                const double rL = __shfl_sync(0xffffffffu, pv, 0), mL = __shfl_sync(0xffffffffu, pv, 1);
                const double rQ = __shfl_sync(0xffffffffu, pv, 2), mQ = __shfl_sync(0xffffffffu, pv, 3);
                const double rR = __shfl_sync(0xffffffffu, pv, 4), mR = __shfl_sync(0xffffffffu, pv, 5);
                const bool has = lane == 0 ? L != kNone : (lane == 1 && bq < m0);
                uint64_t ku = kDead;
                if (lane < 2) {                                 // converged: same expression, lane-selected operands
                    const double r1 = lane == 0 ? rL : rQ, r2 = lane == 0 ? rQ : rR;
                    const double m1 = lane == 0 ? mL : mQ, m2 = lane == 0 ? mQ : mR;
                    const double u = __ddiv_rn(__dadd_rn(r1, r2), __dadd_rn(fabs(__dsub_rn(m2, m1)), eps));
                    if (has) ku = ukey(u, maxu);
                }
                const uint64_t kl = __shfl_sync(0xffffffffu, ku, 0), kr = __shfl_sync(0xffffffffu, ku, 1);
                const bool left = kl <= kr;         // equal keys: the left pair has the lower position
                const uint64_t cand = left ? kl : kr;
                const int pos = left ? L : a;
                bool ok = cand < lb;
                if (!ok) {
                    if (!exact) { refresh_range(d0, d1); exact = true; }
                    const uint64_t S = root_key();
                    const int si = root_idx();
                    lb = S;
                    ok = cand < S || (cand == S && cand != kDead && pos < si);
                }
                if (!ok) {                          // chain ends: the dynamic pairs go back into the tree
                    __syncwarp();
                    if (lane == 0) {
                        if (L != kNone) leaf[L] = kl;
                        if (bq < m0) leaf[a] = kr;
                    }
                    __syncwarp();
                    refresh_range(L != kNone ? L : a, a);
                    break;
                }
                if (left) {                         // Q absorbs L: Q = [L, bq)
                    const int LL = prv[L];
                    __syncwarp();
                    if (lane == 0) {
                        nxt[L] = (uint16_t)bq;
                        if (bq < m0) prv[bq] = (uint16_t)L;
                        leaf[L] = kDead;
                        if (a < npair) leaf[a] = kDead;
                        if (LL != kNone) leaf[LL] = kDead;
                    }
                    d0 = min(d0, LL != kNone ? LL : L);
                    p = L;
                    dir = 0;
                } else {                            // Q absorbs R: Q = [a, c)
                    __syncwarp();
                    if (lane == 0) {
                        nxt[a] = (uint16_t)c;
                        if (c < m0) prv[c] = (uint16_t)a;
                        if (bq < npair) leaf[bq] = kDead;
                        leaf[a] = kDead;
                    }
                    d1 = max(d1, bq < npair ? bq : a);
                    dir = 1;
                }
                __syncwarp();
                exact = false;
                m--;
                merges++;
            }
            if (!(m > max_queues && m > 1)) break;
        }
    }
    if (lane == 0) {
        int k = 0;
        for (int i = 0; i < m0 && k < 256; i = nxt[i]) {
            const int e = nxt[i];
            const int64_t xi = seg[i], xe = e < m0 ? seg[e] : M;
            q_lo[k] = lo[i]; q_hi[k] = lo[e]; q_n[k] = nx[e] - nx[i]; q_s1[k] = s1x[e] - s1x[i];
            q_s2[k] = S2[xe] - S2[xi];
            k++;
        }
        merges_out[0] = merges;
        merges_out[1] = k;
        *done = 1;
    }
}

// ---- Table 3 "EWSJF (K-Means)": exact 1-D k-means for any
// k by dynamic programming over the distinct-value prefixes (oracle O14, R32):
//   D_1[j] = S1[j]^2/N[j],  D_l[j] = max_{l-1 <= i < j} D_{l-1}[i] + (S1[j]-S1[i])^2/(N[j]-N[i])
// in the oracle's left-to-right rounding order (__dmul_rn/__ddiv_rn/__dadd_rn, no
// contraction), smallest i on ties; backtracking from j = M.  One warp per j,
// lanes stride over i (ascending, strict > keeps each lane's smallest i), then a
// (value, smallest i) warp reduction.  fp64-ALU bound: ~M^2/2 divisions per layer.
__device__ __forceinline__ double kdp_term(int64_t s, int64_t n) {
    const double d = (double)s;
    return __ddiv_rn(__dmul_rn(d, d), (double)n);
}
__global__ void kdp_first_kernel(const int64_t* __restrict__ N, const int64_t* __restrict__ S1, int64_t M, double* D) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= M; j += (int64_t)gridDim.x * blockDim.x)
        D[j] = j >= 1 ? kdp_term(S1[j], N[j]) : 0.0;
}
__global__ void __launch_bounds__(256)
    kdp_layer_kernel(const int64_t* __restrict__ N, const int64_t* __restrict__ S1, int64_t M, int l,
                     const double* __restrict__ Dp, double* __restrict__ Dc, int32_t* __restrict__ Al) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // largest j first: the longest rows start early (balance)
    for (int64_t t = w0; t <= M - l; t += nw) {
        const int64_t j = M - t;
        const int64_t nj = N[j], sj = S1[j];
        double best = 0.0;
        int64_t bi = -1;
        for (int64_t i = l - 1 + lane; i < j; i += 32) {
            const double F = __dadd_rn(Dp[i], kdp_term(sj - S1[i], nj - N[i]));
            if (bi < 0 || F > best) { best = F; bi = i; }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; }
        }
        if (lane == 0) { Dc[j] = best; Al[j] = (int32_t)bi; }
    }
}
// backtracking (one thread) + the clusters' queue bounds / statistics (R15 midpoints)
__global__ void kdp_finish_kernel(const int32_t* __restrict__ v, const int64_t* __restrict__ N,
                                  const int64_t* __restrict__ S1, const int64_t* __restrict__ S2, int64_t M, int k,
                                  const int32_t* __restrict__ A, int32_t* cuts, int32_t* q_lo, int32_t* q_hi,
                                  int64_t* q_n, int64_t* q_s1, int64_t* q_s2, int64_t* merges) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t j = M;
    cuts[0] = 0;
    for (int l = k; l >= 2; l--) {
        j = A[(size_t)(l - 1) * (M + 1) + j];
        cuts[l - 1] = (int32_t)j;
    }
    for (int i = 0; i < k; i++) {
        const int64_t x = cuts[i], y = i + 1 < k ? cuts[i + 1] : M;
        q_lo[i] = i == 0 ? v[x] : (int32_t)(((int64_t)v[x - 1] + (int64_t)v[x]) / 2 + 1);
        q_hi[i] = i + 1 < k ? (int32_t)(((int64_t)v[y - 1] + (int64_t)v[y]) / 2 + 1) : v[M - 1] + 1;
        q_n[i] = N[y] - N[x];
        q_s1[i] = S1[y] - S1[x];
        q_s2[i] = S2[y] - S2[x];
    }
    merges[0] = 0;
    merges[1] = k;
}

__global__ void iota_kernel(int64_t* a, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

__global__ void set_flags_kernel(uint8_t* flag, const int32_t* out, int k) {
    flag[0] = 1;
    if (k >= 2) flag[out[2]] = 1;
    if (k >= 3) flag[out[3]] = 1;
}

// ------------------------------------------------------------------ host ---
void rp_free(ewsjf_ctx* ctx) {
    RpScratch* R = ctx->rp;
    if (!R) return;
    void* p[] = {R->ovf, R->hist, R->stat, R->v, R->c, R->N, R->S1, R->S2, R->blk, R->t1, R->t3, R->kbF, R->kbI,
                 R->seg, R->segend, R->flag, R->out_i, R->q_lo, R->q_hi, R->q_n, R->q_s1, R->q_s2, R->merges,
                 R->plo, R->phi_, R->pnext, R->pprev, R->pn, R->ps1, R->ps2, R->tree, R->treei, R->kdp_a, R->kcuts};
    for (void* x : p)
        if (x) cudaFree(x);
    for (auto e : R->ev)
        if (e) cudaEventDestroy(e);
    delete R;
    ctx->rp = nullptr;
}

ewsjf_status rp_alloc(ewsjf_ctx* ctx) {
    RpScratch* R = new RpScratch();
    memset(R, 0, sizeof *R);
    ctx->rp = R;
    const size_t H = kHistMax + kOvfCap + 1;      // distinct lengths: histogram runs + long-tail runs
    R->kblocks = 2048;
    int64_t tn = 0, cnt = kHistMax + kOvfCap;
    for (;;) { tn += cnt; if (cnt == 1) break; cnt = (cnt + 31) / 32; }
    R->tree_n = tn;
    bool ok = cudaMalloc(&R->hist, H * 4) == cudaSuccess && cudaMalloc(&R->stat, 16 * 8) == cudaSuccess &&
              cudaMalloc(&R->ovf, (size_t)kOvfCap * 4) == cudaSuccess &&
              cudaMalloc(&R->v, H * 4) == cudaSuccess && cudaMalloc(&R->c, H * 8) == cudaSuccess &&
              cudaMalloc(&R->N, H * 8) == cudaSuccess && cudaMalloc(&R->S1, H * 8) == cudaSuccess &&
              cudaMalloc(&R->S2, H * 8) == cudaSuccess &&
              cudaMalloc(&R->blk, (kHistMax / kRleChunk + 2) * 4 * 8) == cudaSuccess &&
              cudaMalloc(&R->t1, H * 8) == cudaSuccess && cudaMalloc(&R->t3, H * 8) == cudaSuccess &&
              cudaMalloc(&R->kbF, R->kblocks * 8) == cudaSuccess && cudaMalloc(&R->kbI, R->kblocks * 8) == cudaSuccess &&
              cudaMalloc(&R->seg, H * 4) == cudaSuccess && cudaMalloc(&R->segend, H * 4) == cudaSuccess &&
              cudaMalloc(&R->flag, H) == cudaSuccess && cudaMalloc(&R->out_i, 16 * 4) == cudaSuccess &&
              cudaMalloc(&R->q_lo, 256 * 4) == cudaSuccess && cudaMalloc(&R->q_hi, 256 * 4) == cudaSuccess &&
              cudaMalloc(&R->q_n, 256 * 8) == cudaSuccess && cudaMalloc(&R->q_s1, 256 * 8) == cudaSuccess &&
              cudaMalloc(&R->q_s2, 256 * 8) == cudaSuccess && cudaMalloc(&R->merges, 4 * 8) == cudaSuccess &&
              cudaMalloc(&R->plo, H * 4) == cudaSuccess && cudaMalloc(&R->phi_, H * 4) == cudaSuccess &&
              cudaMalloc(&R->pnext, H * 4) == cudaSuccess && cudaMalloc(&R->pprev, H * 4) == cudaSuccess &&
              cudaMalloc(&R->pn, H * 8) == cudaSuccess && cudaMalloc(&R->ps1, H * 8) == cudaSuccess &&
              cudaMalloc(&R->ps2, H * 8) == cudaSuccess && cudaMalloc(&R->tree, tn * 8) == cudaSuccess &&
              cudaMalloc(&R->treei, tn * 4) == cudaSuccess && cudaMalloc(&R->kcuts, 256 * 4) == cudaSuccess;
    for (auto& e : R->ev) ok = ok && cudaEventCreate(&e) == cudaSuccess;
    if (!ok) { rp_free(ctx); return EWSJF_ERR_CUDA; }
    return EWSJF_OK;
}

}  // namespace ewsjf

namespace ewsjf {
// A2..A6 from a finished histogram (bins 1..lmax); S carries the A1 statistics.
// Table 3's k-means-only partition from the RLE prefixes (N, S1, S2 of M distinct values).
static ewsjf_status rp_kmeans_only(ewsjf_ctx* ctx, int64_t M, const ewsjf_partition_params* p,
                                   ewsjf_partition_t* out, ewsjf_partition_stats* stats, ewsjf_partition_stats& S) {
    RpScratch* R = ctx->rp;
    cudaStream_t st = ctx->stream;
    const int k = (int)std::min<int64_t>(p->kmeans_k, M);
    S.k_used = k;
    const int64_t need = (int64_t)k * (M + 1);
    if (need > R->kdp_cap) {                 // strategic call: grow the DP table once, keep it
        CU(cudaStreamSynchronize(st));
        if (R->kdp_a) cudaFree(R->kdp_a);
        R->kdp_a = nullptr;
        R->kdp_cap = 0;
        CU(cudaMalloc(&R->kdp_a, (size_t)need * 4));
        R->kdp_cap = need;
    }
    double* D[2] = {R->t1, R->t3};
    {
        LaunchScope ls(ctx, KIND_PARTITION);
        kdp_first_kernel<<<(int)std::min<int64_t>(1024, (M + 256) / 256), 256, 0, st>>>(R->N, R->S1, M, D[0]);
    }
    const int grid = ctx->num_sms * 8;
    for (int l = 2; l <= k; l++) {
        LaunchScope ls(ctx, KIND_PARTITION);
        kdp_layer_kernel<<<grid, 256, 0, st>>>(R->N, R->S1, M, l, D[l & 1], D[(l & 1) ^ 1],
                                               R->kdp_a + (size_t)(l - 1) * (M + 1));
    }
    {
        LaunchScope ls(ctx, KIND_PARTITION);
        kdp_finish_kernel<<<1, 32, 0, st>>>(R->v, R->N, R->S1, R->S2, M, k, R->kdp_a, R->kcuts, R->q_lo, R->q_hi,
                                            R->q_n, R->q_s1, R->q_s2, R->merges);
    }
    CU(cudaGetLastError());
    CU(cudaEventRecord(R->ev[4], st));
    int32_t cuts[256], qlo[256], qhi[256];
    int64_t qn[256], qs1[256], qs2[256];
    CU(cudaMemcpyAsync(cuts, R->kcuts, 4 * k, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qlo, R->q_lo, 4 * k, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qhi, R->q_hi, 4 * k, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qn, R->q_n, 8 * k, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qs1, R->q_s1, 8 * k, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qs2, R->q_s2, 8 * k, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    S.segments = k;
    S.t1 = k >= 2 ? cuts[1] : 0;
    S.t2 = k >= 3 ? cuts[2] : 0;
    S.merges = 0;
    const uint64_t ver = out->version;
    memset(out, 0, sizeof *out);
    out->n = k;
    out->next_id = k;
    out->version = ver + 1;
    for (int i = 0; i < k; i++) {
        ewsjf_queue& q = out->q[i];
        q.id = i;
        q.index = i + 1;
        q.min_len = qlo[i];
        q.max_len = qhi[i];
        q.count = qn[i];
        q.sum = qs1[i];
        q.sumsq = qs2[i];
        volatile double m = qn[i] > 0 ? (double)qs1[i] / (double)qn[i] : 0.0;
        q.mean = m;
        q.density = (double)qn[i] / (double)((int64_t)qhi[i] - (int64_t)qlo[i]);
        volatile double sq = (double)qs1[i] * (double)qs1[i];
        q.sse = (double)qs2[i] - sq / (double)qn[i];
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, R->ev[0], R->ev[1]); S.ms_hist = ms;
    cudaEventElapsedTime(&ms, R->ev[1], R->ev[4]); S.ms_kmeans = ms;
    cudaEventElapsedTime(&ms, R->ev[0], R->ev[4]); S.ms_total = ms;
    if (stats) *stats = S;
    return S.n_invalid ? EWSJF_ERR_DOMAIN : EWSJF_OK;
}

static ewsjf_status rp_from_hist(ewsjf_ctx* ctx, const unsigned int* hist, int lmax, const ewsjf_partition_params* p,
                                 ewsjf_partition_t* out, ewsjf_partition_stats* stats, ewsjf_partition_stats& S,
                                 int n_ovf = 0) {
    RpScratch* R = ctx->rp;
    cudaStream_t st = ctx->stream;
    const int nb = (lmax + kRleChunk - 1) / kRleChunk;
    if (nb == 0) {        // every valid length is over-long
        CU(cudaMemsetAsync(R->stat + 4, 0, 4 * 8, st));
    } else {
    {
        LaunchScope ls(ctx, KIND_PARTITION);
        rle_count_kernel<<<nb, kHT, 0, st>>>(hist, lmax, R->blk);
    }
    {
        LaunchScope ls(ctx, KIND_PARTITION);
        rle_scan_kernel<<<1, kHT, 0, st>>>(R->blk, nb, (int64_t*)(R->stat + 4));
    }
    {
        LaunchScope ls(ctx, KIND_PARTITION);
        rle_write_kernel<<<nb, kHT, 0, st>>>(hist, lmax, R->blk, R->v, R->c, R->N, R->S1, R->S2);
    }
    }
    if (n_ovf > 0) {
        int P = 1;
        while (P < n_ovf) P <<= 1;
        CU(cudaFuncSetAttribute(ovf_rle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kOvfCap * 4));
        LaunchScope ls(ctx, KIND_PARTITION);
        ovf_rle_kernel<<<1, kHT, (size_t)P * 4, st>>>(R->ovf, n_ovf, (int64_t*)(R->stat + 4), R->v, R->c, R->N, R->S1,
                                                      R->S2, R->segend);
    }
    CU(cudaGetLastError());
    int64_t tot[4];
    CU(cudaMemcpyAsync(tot, R->stat + 4, 4 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const int64_t M = tot[0];
    S.distinct = M;
    S.n_valid = tot[1];
    if (M > kHistMax) {   // the Stage-3 tree's static depth covers 2^20 leaves
        if (stats) *stats = S;
        return fail(ctx, EWSJF_ERR_UNSUPPORTED, "%lld distinct history lengths (at most 2^20)", (long long)M);
    }
    if (M == 0) {
        if (stats) *stats = S;
        return fail(ctx, EWSJF_ERR_EMPTY, "no history length >= 1");
    }
    if (p->kmeans_k > 0) return rp_kmeans_only(ctx, M, p, out, stats, S);
    const int k = p->coarse_k < M ? p->coarse_k : (int)M;
    S.k_used = k;
    if (k == 3) {
        {
            LaunchScope ls(ctx, KIND_PARTITION);
            kmeans_terms_kernel<<<256, 256, 0, st>>>(R->N, R->S1, M, R->t1, R->t3);
        }
        const int kb = (int)std::min<int64_t>(R->kblocks, std::max<int64_t>(1, (M - 2 + kKmTile - 1) / kKmTile));
        {
            LaunchScope ls(ctx, KIND_PARTITION);
            kmeans3_kernel<<<kb, 256, 0, st>>>(R->N, R->S1, R->t1, R->t3, M, R->kbF, R->kbI);
        }
        {
            LaunchScope ls(ctx, KIND_PARTITION);
            kmeans_final_kernel<<<1, 1024, 0, st>>>(R->N, R->S1, M, 3, R->kbF, R->kbI, kb, R->out_i);
        }
    } else if (k == 2) {
        LaunchScope ls(ctx, KIND_PARTITION);
        kmeans_final_kernel<<<1, 1024, 0, st>>>(R->N, R->S1, M, 2, nullptr, nullptr, 0, R->out_i);
    }
    CU(cudaGetLastError());
    CU(cudaEventRecord(R->ev[2], st));
    CU(cudaMemsetAsync(R->flag, 0, (size_t)M, st));
    set_flags_kernel<<<1, 1, 0, st>>>(R->flag, R->out_i, k);
    {
        LaunchScope ls(ctx, KIND_PARTITION);
        // gap_rule 1 (set reading of G): Eq. 2 counts distinct lengths -> identity prefix
        if (p->gap_rule) iota_kernel<<<(int)((M + 1 + 255) / 256), 256, 0, st>>>(R->ps2, M + 1);
        refine_kernel<<<1, kHT, 0, st>>>(R->v, p->gap_rule ? R->ps2 : R->N, M, p->alpha, p->min_width, R->flag,
                                          R->seg, R->out_i, R->segend, R->plo, R->t1, R->t3);
    }
    CU(cudaGetLastError());
    CU(cudaEventRecord(R->ev[3], st));
    {
        // shared-memory prune for m <= cap (every partition up to ~18k segments), else the
        // global-memory tree (prune_kernel skips itself when the first one finished)
        const int budget = (ctx->smem_optin > 0 ? ctx->smem_optin : 232448) - 1024;
        if (R->prune_cap == 0) {
            for (int g = 0; g < 2; g++) {
                int lo_ = 2, hi_ = 65534;                   // u16 links
                while (lo_ < hi_) {
                    const int mid = (lo_ + hi_ + 1) / 2;
                    if (prune_smem_bytes(mid, nullptr, nullptr, nullptr, g == 1) <= (size_t)budget) lo_ = mid;
                    else hi_ = mid - 1;
                }
                (g ? R->prune_cap_lg : R->prune_cap) = lo_;
            }
            CU(cudaFuncSetAttribute(prune_smem_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
            CU(cudaFuncSetAttribute(prune_smem_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
        }
        LaunchScope ls(ctx, KIND_PARTITION);
        prune_prep_kernel<<<64, 256, 0, st>>>(R->v, R->N, R->S1, R->seg, M, R->out_i, R->plo, R->pn, R->ps1);
        prune_smem_kernel<false><<<1, kHT, budget, st>>>(nullptr, R->plo, R->pn, R->ps1, R->S2, R->seg, M, R->out_i,
                                                         R->prune_cap, p->max_queues, p->epsilon, p->merge_rule,
                                                         R->q_lo, R->q_hi, R->q_n, R->q_s1, R->q_s2, R->merges,
                                                         R->out_i + 8);
        prune_smem_kernel<true><<<1, kHT, budget, st>>>((uint64_t*)R->tree, R->plo, R->pn, R->ps1, R->S2, R->seg, M,
                                                        R->out_i, R->prune_cap_lg, p->max_queues, p->epsilon,
                                                        p->merge_rule, R->q_lo, R->q_hi, R->q_n, R->q_s1, R->q_s2,
                                                        R->merges, R->out_i + 8);
        prune_kernel<<<1, kHT, 0, st>>>(R->v, R->N, R->S1, R->S2, M, R->seg, R->out_i, p->max_queues, p->epsilon,
                                         p->merge_rule, R->plo, R->phi_, R->pnext, R->pprev, R->pn, R->ps1, R->ps2,
                                         R->tree, R->treei, R->q_lo, R->q_hi, R->q_n, R->q_s1, R->q_s2, R->merges,
                                         R->out_i + 8);
    }
    CU(cudaGetLastError());
    CU(cudaEventRecord(R->ev[4], st));
    int32_t oi[4];
    int32_t qlo[256], qhi[256];
    int64_t qn[256], qs1[256], qs2[256], mg[2];
    CU(cudaMemcpyAsync(oi, R->out_i, 16, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(mg, R->merges, 16, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qlo, R->q_lo, sizeof qlo, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qhi, R->q_hi, sizeof qhi, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qn, R->q_n, sizeof qn, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qs1, R->q_s1, sizeof qs1, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(qs2, R->q_s2, sizeof qs2, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    S.segments = oi[0];
    S.depth = oi[1];
    S.t1 = k >= 2 ? oi[2] : 0;
    S.t2 = k >= 3 ? oi[3] : 0;
    S.merges = mg[0];
    const int nq = (int)mg[1];
    const uint64_t ver = out->version;
    memset(out, 0, sizeof *out);
    out->n = nq;
    out->next_id = nq;
    out->version = ver + 1;
    for (int i = 0; i < nq; i++) {
        ewsjf_queue& q = out->q[i];
        q.id = i;
        q.index = i + 1;
        q.min_len = qlo[i];
        q.max_len = qhi[i];
        q.count = qn[i];
        q.sum = qs1[i];
        q.sumsq = qs2[i];
        // the oracle's canonical expressions (host code built with -ffp-contract=off)
        volatile double m = qn[i] > 0 ? (double)qs1[i] / (double)qn[i] : 0.0;
        q.mean = m;
        q.density = (double)qn[i] / (double)((int64_t)qhi[i] - (int64_t)qlo[i]);
        volatile double sq = (double)qs1[i] * (double)qs1[i];
        q.sse = (double)qs2[i] - sq / (double)qn[i];
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, R->ev[0], R->ev[1]); S.ms_hist = ms;
    cudaEventElapsedTime(&ms, R->ev[1], R->ev[2]); S.ms_kmeans = ms;
    cudaEventElapsedTime(&ms, R->ev[2], R->ev[3]); S.ms_refine = ms;
    cudaEventElapsedTime(&ms, R->ev[3], R->ev[4]); S.ms_prune = ms;
    cudaEventElapsedTime(&ms, R->ev[0], R->ev[4]); S.ms_total = ms;
    if (stats) *stats = S;
    return S.n_invalid ? EWSJF_ERR_DOMAIN : EWSJF_OK;
}
}  // namespace ewsjf

static ewsjf_status check_rp_params(ewsjf_ctx* ctx, const ewsjf_partition_params* p, ewsjf_partition_t* out) {
    if (!p || !out) return fail(ctx, EWSJF_ERR_INVALID_ARG, "null params/out");
    if (p->kmeans_k < 0 || p->kmeans_k > EWSJF_MAX_QUEUES)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "kmeans_k out of range");
    if (p->kmeans_k > 0) return EWSJF_OK;      // k-means-only: the R&P parameters are not used
    if (!(p->alpha > 1.0) || p->min_width < 1 || p->max_queues < 1 || p->max_queues > EWSJF_MAX_QUEUES ||
        !(p->epsilon > 0.0) || p->coarse_k < 1 || p->coarse_k > 3 || (p->merge_rule != 0 && p->merge_rule != 1) ||
        (p->gap_rule != 0 && p->gap_rule != 1))
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "partition params out of range (S:121)");
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_partition(ewsjf_ctx* ctx, const int32_t* d_len, int64_t n,
                                        const ewsjf_partition_params* p, ewsjf_partition_t* out,
                                        ewsjf_partition_stats* stats) {
    using namespace ewsjf;
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    {
        ewsjf_status c = check_rp_params(ctx, p, out);
        if (c != EWSJF_OK) return c;
    }
    if (n < 0 || n > ctx->max_history) return fail(ctx, EWSJF_ERR_INVALID_ARG, "n=%lld > max_history", (long long)n);
    if (n > 0 && !d_len) return fail(ctx, EWSJF_ERR_INVALID_ARG, "null history");
    RpScratch* R = ctx->rp;
    if (!R) return fail(ctx, EWSJF_ERR_INVALID_ARG, "ctx created with max_history = 0");
    CU(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    ewsjf_partition_stats S;
    memset(&S, 0, sizeof S);
    CU(cudaEventRecord(R->ev[0], st));
    CU(cudaMemsetAsync(R->hist, 0, (size_t)(kHistMax + 1) * 4, st));
    CU(cudaMemsetAsync(R->stat, 0, 16 * 8, st));
    if (n > 0) {
        LaunchScope ls(ctx, KIND_PARTITION);
        CU(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistSmem * 4));
        hist_kernel<<<ctx->num_sms, kHT, kHistSmem * 4, st>>>(d_len, n, R->hist, R->stat, R->ovf);
        CU(cudaGetLastError());
    }
    CU(cudaEventRecord(R->ev[1], st));
    unsigned long long hs[3];
    CU(cudaMemcpyAsync(hs, R->stat, 3 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    S.n_invalid = (int64_t)hs[0];
    S.n_valid = n - (int64_t)hs[0];
    if (hs[1] > (unsigned long long)kOvfCap) {
        if (stats) *stats = S;
        return fail(ctx, EWSJF_ERR_UNSUPPORTED, "%llu history lengths >= 2^20 (at most %d per call)", hs[1], kOvfCap);
    }
    if (S.n_valid == 0) {
        if (stats) *stats = S;
        return fail(ctx, EWSJF_ERR_EMPTY, "no history length >= 1");
    }
    return rp_from_hist(ctx, R->hist, (int)hs[2], p, out, stats, S, (int)hs[1]);
}

extern "C" ewsjf_status ewsjf_history_hist(ewsjf_ctx* ctx, const int32_t* d_len, int64_t n, uint32_t* d_hist,
                                           int64_t* h_info) {
    using namespace ewsjf;
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (!d_hist || !h_info || n < 0 || (n > 0 && !d_len)) return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad history_hist arguments");
    RpScratch* R = ctx->rp;
    if (!R) return fail(ctx, EWSJF_ERR_INVALID_ARG, "ctx created with max_history = 0");
    CU(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    CU(cudaMemsetAsync(d_hist, 0, (size_t)(kHistMax + 1) * 4, st));
    CU(cudaMemsetAsync(R->stat, 0, 16 * 8, st));
    if (n > 0) {
        LaunchScope ls(ctx, KIND_PARTITION);
        CU(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistSmem * 4));
        hist_kernel<<<ctx->num_sms, kHT, kHistSmem * 4, st>>>(d_len, n, (unsigned int*)d_hist, R->stat, nullptr);
        CU(cudaGetLastError());
    }
    unsigned long long hs[3];
    CU(cudaMemcpyAsync(hs, R->stat, 3 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    h_info[0] = (int64_t)hs[0];
    h_info[1] = (int64_t)hs[1];
    h_info[2] = (int64_t)hs[2];
    return hs[1] ? fail(ctx, EWSJF_ERR_UNSUPPORTED, "%llu history lengths >= 2^20", hs[1]) : EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_partition_from_hist(ewsjf_ctx* ctx, const uint32_t* d_hist, int32_t max_len,
                                                  int64_t n_invalid, const ewsjf_partition_params* p,
                                                  ewsjf_partition_t* out, ewsjf_partition_stats* stats) {
    using namespace ewsjf;
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    ewsjf_status c = check_rp_params(ctx, p, out);
    if (c != EWSJF_OK) return c;
    if (!d_hist || max_len < 0 || max_len >= kHistMax || n_invalid < 0)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad histogram arguments");
    RpScratch* R = ctx->rp;
    if (!R) return fail(ctx, EWSJF_ERR_INVALID_ARG, "ctx created with max_history = 0");
    CU(cudaSetDevice(ctx->device));
    ewsjf_partition_stats S;
    memset(&S, 0, sizeof S);
    S.n_invalid = n_invalid;
    CU(cudaEventRecord(R->ev[0], ctx->stream));
    CU(cudaEventRecord(R->ev[1], ctx->stream));
    if (max_len == 0) {
        if (stats) *stats = S;
        return fail(ctx, EWSJF_ERR_EMPTY, "no history length >= 1");
    }
    return rp_from_hist(ctx, (const unsigned int*)d_hist, max_len, p, out, stats, S);
}

// ------------------------------------------- online adjust (R31) ---
// One CTA per interior boundary B between queues [L, B) and [B, U): each thread
// sums one contiguous slab of the window's histogram over [L, U), one block scan
// gives every slab's starting count, and each thread walks its slab; the target T is
// the smallest x with (#window < x in [L, U)) * (c_a + c_b) >= m * c_a (m = the
// window's members in [L, U)), then the move is clamped to floor(max_shift *
// adjacent width) on each side — the same fp64 product as the oracle.
namespace ewsjf {
struct AdjustArgs {
    int32_t L[EWSJF_MAX_QUEUES], B[EWSJF_MAX_QUEUES], U[EWSJF_MAX_QUEUES];
    int64_t ca[EWSJF_MAX_QUEUES], cb[EWSJF_MAX_QUEUES];
    double max_shift;
};

__device__ __forceinline__ int64_t block_excl_scan(int64_t x, int64_t* sm, int64_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) sm[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < (int)(blockDim.x >> 5) ? sm[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sm[32 + lane] = w;                    // inclusive warp-sum prefix
    }
    __syncthreads();
    const int64_t before = warp ? sm[32 + warp - 1] : 0;
    *total = sm[32 + (blockDim.x >> 5) - 1];
    __syncthreads();
    return before + v - x;
}

__global__ void __launch_bounds__(kHT) adjust_kernel(const unsigned int* __restrict__ hist,
                                                     const __grid_constant__ AdjustArgs A, int32_t* newb) {
    __shared__ int64_t sm[64];
    __shared__ int s_hit;
    const int i = blockIdx.x + 1;                               // boundary index 1..nq-1
    const int32_t L = A.L[i], B = A.B[i], U = A.U[i];
    const int64_t ca = A.ca[i], cb = A.cb[i];
    if (L < 0 || ca + cb == 0) { if (threadIdx.x == 0) newb[i] = B; return; }   // L < 0: not shared
    // one contiguous slab of bins per thread: slab sums, one block scan (m = total)
    const int width = U - L;
    const int slab = (width + (int)blockDim.x - 1) / (int)blockDim.x;
    const int xs = L + (int)threadIdx.x * slab, xe = min(U, xs + slab);
    int64_t part = 0;
    for (int x = xs; x < xe; x++) part += hist[x];
    int64_t m;
    const int64_t before = block_excl_scan(part, sm, &m);       // window members in [L, xs)
    if (m == 0) { if (threadIdx.x == 0) newb[i] = B; return; }
    // smallest x in [L, U] with cum(< x) * (ca + cb) >= m * ca (x = U always qualifies);
    // cum is monotone in x, so each thread walks its slab until it qualifies
    const int64_t rhs = m * ca, den = ca + cb;
    if (threadIdx.x == 0) s_hit = U;
    __syncthreads();
    int64_t cum = before;
    for (int x = xs; x < xe; x++) {
        if (cum * den >= rhs) { atomicMin(&s_hit, x); break; }
        cum += hist[x];
    }
    __syncthreads();
    const int32_t T = s_hit;
    if (threadIdx.x == 0) {
        int64_t d = (int64_t)T - B;
        const int64_t left = (int64_t)floor(__dmul_rn(A.max_shift, (double)(B - L)));
        const int64_t right = (int64_t)floor(__dmul_rn(A.max_shift, (double)(U - B)));
        if (d < -left) d = -left;
        if (d > right) d = right;
        newb[i] = (int32_t)(B + d);
    }
}
}  // namespace ewsjf

extern "C" ewsjf_status ewsjf_online_adjust(ewsjf_ctx* ctx, const int32_t* d_window, int64_t n, double max_shift,
                                            ewsjf_partition_t* part, int32_t* moved) {
    using namespace ewsjf;
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (!part || n < 0 || (n > 0 && !d_window) || !(max_shift >= 0.0 && max_shift < 0.5) || part->n < 0 ||
        part->n > EWSJF_MAX_QUEUES)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad online_adjust arguments (max_shift in [0, 0.5))");
    if (moved) *moved = 0;
    const int nq = part->n;
    if (nq < 2 || n == 0) return EWSJF_OK;
    RpScratch* R = ctx->rp;
    if (!R) return fail(ctx, EWSJF_ERR_INVALID_ARG, "ctx created with max_history = 0");
    for (int i = 1; i < nq; i++)
        if (part->q[i].min_len < part->q[i - 1].max_len || part->q[i].max_len > kHistMax)
            return fail(ctx, EWSJF_ERR_INVALID_ARG, "partition not sorted / bounds above 2^20");
    CU(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    CU(cudaMemsetAsync(R->hist, 0, (size_t)(kHistMax + 1) * 4, st));
    CU(cudaMemsetAsync(R->stat, 0, 16 * 8, st));
    {
        LaunchScope ls(ctx, KIND_PARTITION);
        CU(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistSmem * 4));
        hist_kernel<<<ctx->num_sms, kHT, kHistSmem * 4, st>>>(d_window, n, R->hist, R->stat, nullptr);
    }
    static thread_local AdjustArgs A;
    A.max_shift = max_shift;
    for (int i = 1; i < nq; i++) {
        const ewsjf_queue& a = part->q[i - 1];
        const ewsjf_queue& b = part->q[i];
        A.L[i] = a.max_len == b.min_len ? a.min_len : -1;      // only shared boundaries move
        A.B[i] = b.min_len;
        A.U[i] = b.max_len;
        A.ca[i] = a.count;
        A.cb[i] = b.count;
    }
    {
        LaunchScope ls(ctx, KIND_PARTITION);
        adjust_kernel<<<nq - 1, kHT, 0, st>>>(R->hist, A, R->seg);
    }
    CU(cudaGetLastError());
    int32_t nb[EWSJF_MAX_QUEUES];
    unsigned long long hs[3];
    CU(cudaMemcpyAsync(nb, R->seg, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(hs, R->stat, 3 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (hs[1]) return fail(ctx, EWSJF_ERR_UNSUPPORTED, "%llu window lengths >= 2^20", hs[1]);
    int32_t mv = 0;
    for (int i = 1; i < nq; i++) {
        if (nb[i] == part->q[i].min_len) continue;
        part->q[i - 1].max_len = nb[i];
        part->q[i].min_len = nb[i];
        mv++;
    }
    if (mv) part->version++;
    if (moved) *moved = mv;
    return EWSJF_OK;
}
