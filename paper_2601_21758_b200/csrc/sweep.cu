// sweep.cu — Θ-batched score + select (A12, config C5; §4.4.2).
//
// The meta-optimizer evaluates candidate scoring parameters Θ over
// one snapshot of the pending pool: for each Θ, A7 (per-queue weights
// w_x = max(0, a_x b̄ + b_x)) then A10 (Eq. 4) and A11 (per-queue
// top-K, head, ArgMax).  Eq. 4 is linear in the weights:
//     s' = Φ / q_i = w_base·f0 + w_urg·f1 + w_fair·f2,
//     f0 = 1/(b+1),  f1 = W/(C (b+1)),  f2 = ln(b+1)/(b+1)
// so after one Θ-independent pass (K1-K3: validity, per-queue counts, FIFO
// head, features, and the snapshot regrouped by queue) every (request, Θ) pair
// costs three FMAs and a compare.
//
//   K1 sweep_count_kernel   per-queue member counts, FIFO heads, excluded/invalid
//   K2 sweep_plan_kernel    per-queue offsets and chunk prefix (one CTA)
//   K3 sweep_scatter_kernel float4 {f0, f1, f2, id} records grouped by queue
//   K4 sweep_select_kernel  persistent warps over tasks (Θ block of kSwT, queue,
//                           chunk): thresholded candidates in warp-private
//                           buffers, exact K-th cuts, thresholds shared per
//                           (Θ, queue) through global atomicMax
//   K5 sweep_merge_kernel   one warp per (Θ, queue): merge the task rows,
//                           exact top-K, head score, max score
//   K6 sweep_summary_kernel one warp per Θ: Alg. 1 ArgMax + summary
// No CTA-wide barrier inside K4/K5; nothing is shared between warps but the
// monotone (Θ, queue) thresholds.
#include <climits>
#include <cstring>
#include <algorithm>
#include "tick.cuh"
#include "select.cuh"
#include "ctx.h"

namespace ewsjf {

constexpr int kSwT = 16;            // Θ per task (weights and thresholds held in registers)
constexpr int kSwBatch = 128;       // Θ per kernel sequence (scratch is sized for one batch)
constexpr int kSwMaxK = 96;         // cap = 2K+32 <= 256 keys (register K-th selection)
constexpr int kSwPrepThreads = 512;
constexpr int kSwWarps = 8;         // warps per CTA in K4 / K5
// Θ-independent candidate prefilter (K3a-K3g): lengths 2 <= b < kSkyBins are
// grouped; blocks of kSkyBlk consecutive lengths; K <= 32 (one key per lane)
constexpr int kSkyBins = 1 << 16;
constexpr int kSkyBlk = 64;
constexpr int kSkyMaxBlocks = kSkyBins / kSkyBlk + kMaxSlots + 1;
constexpr int kSkyMaxK = 32;
constexpr int kSwDirectMax = 4096;  // K5d: one warp per (Θ, queue) scans its queue's survivors directly

struct SweepScratch {
    int64_t n_cap = 0;              // records capacity
    int64_t task_cap = 0;           // task rows capacity
    float4* rec = nullptr;          // [n] grouped by queue position
    int64_t* qcount = nullptr;      // [256] valid members per position
    int64_t* qoff = nullptr;        // [257] record offsets
    int32_t* cpre = nullptr;        // [257] chunk prefix
    int32_t* qfill = nullptr;       // [256] scatter cursors
    u64* head = nullptr;            // [256] FIFO key of the head (max), 0 = empty
    float4* headf = nullptr;        // [256] head features
    unsigned long long* bad = nullptr;   // [4] invalid, excluded, diagnostics: cuts, inserts
    unsigned int* task_ctr = nullptr;
    u64* gthr = nullptr;            // [kSwBatch][256] shared thresholds (exact keys)
    u64* rows = nullptr;            // [task][kSwT][K]
    int32_t* rowcnt = nullptr;      // [task][kSwT]
    float* w = nullptr;             // [kSwBatch][nq][3] weights by position (device, A7, uploaded per batch)
    float* h_w = nullptr;           // pinned staging [2][kSwBatch][256][3] (ring of two, w_ev)
    cudaEvent_t w_ev[2] = {};
    int w_next = 0;
    // prefilter scratch: bin counts -> starts, scatter cursors, per-length list bounds,
    // per-block top keys, prefix bounds, the compacted records + layout (rec2 holds the
    // records sorted by length until the compaction)
    int32_t* bcnt = nullptr;        // [kSkyBins + 1]
    int32_t* bfill = nullptr;       // [kSkyBins]
    u64* lenkth = nullptr;          // [kSkyBins][2] per length: K-th of its two lists (0: keep all)
    int32_t* biglist = nullptr;     // [kSkyBins] lengths with > kSkyBig records (K3d's CTA kernel)
    int32_t* nbig = nullptr;        // [1]
    u64* blktop = nullptr;          // [kSkyMaxBlocks][kSkyMaxK]
    u64* blkid = nullptr;           // [kSkyMaxBlocks][kSkyMaxK]
    u64* lentop = nullptr;          // [kSkyBins][kSkyMaxK] per length: its K best (f1, id) keys
    u64* lenid = nullptr;           // [kSkyBins][kSkyMaxK] per length: its K lowest id keys
    u64* qidk = nullptr;            // [256]
    uint32_t* pref = nullptr;       // [kSkyMaxBlocks]
    float4* rec2 = nullptr;         // [n]
    int64_t* qoff2 = nullptr;       // [257]
    int32_t* cpre2 = nullptr;       // [257]
    int32_t* qfill2 = nullptr;      // [256]
    int64_t* qcnt2 = nullptr;       // [256]
    int32_t* direct = nullptr;      // [1] 1: the prefilter left <= kSwDirectMax records per queue (K5d path)
    size_t attr_smem = 0;           // select kernel: dynamic smem attribute set for this ctx's device
    bool sky_attr = false;          // prefilter kernels' dynamic smem attributes set
    // kernel arguments live in device memory (SweepArgs is ~13 KB: as a kernel parameter
    // every launch paid for copying it): a ring of pinned staging slots, each uploaded
    // with one stream-ordered copy; a slot is rewritten once its previous copy has run
    static constexpr int kArgSlots = 8;
    unsigned char* h_args = nullptr;
    unsigned char* d_args = nullptr;
    size_t arg_slot = 0;
    cudaEvent_t arg_ev[kArgSlots] = {};
    int arg_next = 0;
    unsigned char* d_fix = nullptr;   // [3] fixed argument blocks the sweep's graphs read (prep A, batch A, batch O)
    cudaGraphExec_t g_prep = nullptr, g_batch = nullptr;
    int64_t g_prep_key = -1, g_batch_key = -1;
    int g_prep_kernels = 0, g_batch_kernels = 0;   // kernels per replay (launch accounting)
    cudaStream_t cap_st = nullptr;                  // private stream the graphs are captured on
    int occ = 1;
    int last_nq = 0;                // diagnostics: the last sweep's queue count and record offsets used
    bool last_sky = false;
};

struct SweepArgs {
    const int32_t* len;
    const float* arrival;
    const float* cost;
    const int32_t* qid;
    int64_t n;
    int32_t nq;
    int32_t K, cap, chunk, chunk0, rcap;
    int32_t n_theta;                // in this batch
    float now, c0, c1, c2;
    double theta[kSwBatch][6];      // this batch's Θ (a_b, b_b, a_u, b_u, a_f, b_f)
    double mean[kMaxSlots];         // b̄ by position
    int32_t nids;
    int32_t sorted_ids[kMaxSlots];
    int32_t sorted_pos[kMaxSlots];
    // prefilter: per position the grouped length range [qbin_lo, qbin_hi) and its first block
    int32_t qbin_lo[kMaxSlots], qbin_hi[kMaxSlots], qblk[kMaxSlots + 1];
    int32_t sky_nbins;              // bins in use: > every qbin_hi, multiple of 1024, <= kSkyBins
    SweepScratch s;
};

__device__ __forceinline__ int sw_pos(const SweepArgs& A, const int* ids, const int* pos, int q) {
    int lo = 0, hi = A.nids;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ids[mid] < q) lo = mid + 1; else hi = mid;
    }
    return (lo < A.nids && ids[lo] == q) ? pos[lo] : -1;
}

// Validity and features of request r (same preconditions as score_sp: b >= 1,
// W >= 0, C > 0; fp32 like the tick).  Returns the position or -1 / -2.
__device__ __forceinline__ int sw_request(const SweepArgs& A, const int* ids, const int* pos, int64_t r,
                                          float4* f, u64* fk) {
    const int b = __ldg(A.len + r);
    const int q = __ldg(A.qid + r);
    const int p = b >= 1 ? sw_pos(A, ids, pos, q) : -1;
    if (p < 0) return -1;                                   // invalid (len < 1 / unknown qid)
    const float a = __ldg(A.arrival + r);
    const float W = A.now - a;
    const float bf = (float)b;
    const float C = A.cost ? __ldg(A.cost + r) : fmaf(fmaf(A.c2, bf, A.c1), bf, A.c0);
    if (!(W >= 0.0f) || !(C > 0.0f)) return -2;             // excluded
    const float b1 = bf + 1.0f;
    const float f0 = 1.0f / b1;
    f->x = f0;
    f->y = W / (C * b1);
    f->z = logf(b1) * f0;
    f->w = __uint_as_float((uint32_t)r);
    *fk = fifo_key(a, (uint32_t)r);
    return p;
}

// K1: counts, FIFO heads, invalid / excluded totals.
__global__ void __launch_bounds__(kSwPrepThreads) sweep_count_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    __shared__ int s_ids[kMaxSlots], s_pos[kMaxSlots];
    __shared__ unsigned int s_cnt[kMaxSlots];
    __shared__ u64 s_head[kMaxSlots];
    __shared__ unsigned int s_bad[2];
    for (int i = threadIdx.x; i < kMaxSlots; i += blockDim.x) {
        s_ids[i] = A.sorted_ids[i]; s_pos[i] = A.sorted_pos[i]; s_cnt[i] = 0; s_head[i] = 0;
    }
    if (threadIdx.x < 2) s_bad[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < A.n; r += (int64_t)gridDim.x * blockDim.x) {
        float4 f;
        u64 fk;
        const int p = sw_request(A, s_ids, s_pos, r, &f, &fk);
        if (p >= 0) {
            atomicAdd(&s_cnt[p], 1u);
            if (fk > *(volatile u64*)&s_head[p]) atomicMax(&s_head[p], fk);
        } else {
            atomicAdd(&s_bad[p == -1 ? 0 : 1], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < A.nq; i += blockDim.x) {
        if (s_cnt[i]) atomicAdd((unsigned long long*)&A.s.qcount[i], (unsigned long long)s_cnt[i]);
        if (s_head[i]) atomicMax(&A.s.head[i], s_head[i]);
    }
    if (threadIdx.x < 2 && s_bad[threadIdx.x]) atomicAdd(&A.s.bad[threadIdx.x], (unsigned long long)s_bad[threadIdx.x]);
}

// One warp: exclusive prefix of the per-position counts cnt[0..nq) (nq <= 256, 8 per lane)
// into off[0..nq], of their chunk counts into cp[0..nq], zeroed cursors; returns the
// largest count (all lanes).  A one-thread loop over the positions took ~10 us (a
// dependent L2 load per position).
__device__ __forceinline__ int64_t sw_plan_warp(const int64_t* cnt, int nq, int chunk, int64_t* off, int32_t* cp,
                                                int32_t* fill) {
    const int lane = threadIdx.x & 31;
    int64_t c[8], sum = 0, mx = 0;
    int32_t sc = 0;
#pragma unroll
    for (int u = 0; u < 8; u++) {
        const int q = lane * 8 + u;
        c[u] = q < nq ? cnt[q] : 0;
        sum += c[u];
        sc += (int32_t)((c[u] + chunk - 1) / chunk);
        mx = c[u] > mx ? c[u] : mx;
    }
    int64_t is = sum;
    int32_t ic = sc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t us = __shfl_up_sync(0xffffffffu, is, o);
        const int32_t uc = __shfl_up_sync(0xffffffffu, ic, o);
        if (lane >= o) { is += us; ic += uc; }
    }
    int64_t bs = is - sum;
    int32_t bc = ic - sc;
#pragma unroll
    for (int u = 0; u < 8; u++) {
        const int q = lane * 8 + u;
        if (q < nq) {
            off[q] = bs;
            cp[q] = bc;
            if (fill) fill[q] = 0;
            bs += c[u];
            bc += (int32_t)((c[u] + chunk - 1) / chunk);
        }
    }
    if (lane == 31) { off[nq] = is; cp[nq] = ic; }
#pragma unroll
    for (int o = 16; o; o >>= 1) { const int64_t v = __shfl_xor_sync(0xffffffffu, mx, o); mx = v > mx ? v : mx; }
    return mx;
}

// K2 (one CTA of 32 threads): record offsets, chunk prefix, head features, reset cursors.
__global__ void sweep_plan_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    __shared__ int s_ids[kMaxSlots], s_pos[kMaxSlots];
    for (int i = threadIdx.x; i < kMaxSlots; i += blockDim.x) { s_ids[i] = A.sorted_ids[i]; s_pos[i] = A.sorted_pos[i]; }
    __syncwarp();
    sw_plan_warp(A.s.qcount, A.nq, A.chunk, A.s.qoff, A.s.cpre, A.s.qfill);
    if (threadIdx.x == 0) *A.s.task_ctr = 0;
    for (int q = threadIdx.x; q < A.nq; q += blockDim.x) {
        float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
        const u64 hk = A.s.head[q];
        if (hk) {
            u64 dummy;
            sw_request(A, s_ids, s_pos, (int64_t)key_gid(hk), &f, &dummy);
        }
        A.s.headf[q] = f;
    }
}

// Contiguous record range of this CTA: [i0, i1) of [0, ntot).
__device__ __forceinline__ void sw_cta_range(int64_t ntot, int64_t* i0, int64_t* i1) {
    const int64_t per = (ntot + gridDim.x - 1) / gridDim.x;
    *i0 = min(ntot, per * (int64_t)blockIdx.x);
    *i1 = min(ntot, *i0 + per);
}

// K3: scatter the valid requests' records grouped by queue position.  Each CTA takes a
// contiguous range of the snapshot: counts per position in shared memory, one global
// cursor reservation per (CTA, position), then the records placed with shared cursors
// (a warp-aggregated global cursor per record batch serialised ~30k atomics on the
// dominant position's cursor, ~60 us at C5).
__global__ void __launch_bounds__(kSwPrepThreads) sweep_scatter_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    __shared__ int s_ids[kMaxSlots], s_pos[kMaxSlots];
    __shared__ unsigned s_cnt[kMaxSlots];
    for (int i = threadIdx.x; i < kMaxSlots; i += blockDim.x) { s_ids[i] = A.sorted_ids[i]; s_pos[i] = A.sorted_pos[i]; s_cnt[i] = 0u; }
    __syncthreads();
    int64_t r0, r1;
    sw_cta_range(A.n, &r0, &r1);
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        float4 f;
        u64 fk;
        const int p = sw_request(A, s_ids, s_pos, r, &f, &fk);
        if (p >= 0) atomicAdd(&s_cnt[p], 1u);
    }
    __syncthreads();
    for (int p = threadIdx.x; p < A.nq; p += blockDim.x)
        if (s_cnt[p]) s_cnt[p] = (unsigned)A.s.qoff[p] + (unsigned)atomicAdd(&A.s.qfill[p], (int)s_cnt[p]);
    __syncthreads();
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        float4 f;
        u64 fk;
        const int p = sw_request(A, s_ids, s_pos, r, &f, &fk);
        if (p >= 0) A.s.rec[atomicAdd(&s_cnt[p], 1u)] = f;
    }
}


// ---------------------------------------------------------------------------
// Θ-independent candidate prefilter (exact up to fp32 near-ties).  Within a
// queue, s' = w_base f0(b) + w_urg f1 + w_fair f2(b) with all weights >= 0
// (S:306), f0 = 1/(b+1) and f2 = ln(b+1)/(b+1) both non-increasing in b for
// b >= 2, and the fp32 evaluation monotone in every feature.  So a record p can
// only be in a queue's top K for some Θ if fewer than K records q dominate it
// (f0, f1, f2 all >=): (i) inside p's own length b only the K best by (f1, id)
// qualify (features f0, f2 are bit-identical there, ties go to the lower id as
// in the key), (ii) across lengths, the K-th best f1 of the candidates of all
// shorter lengths must stay below p's f1 (tracked per block of kSkyBlk lengths:
// dominators in p's own block are ignored, which only keeps more).  A dominated
// record can only displace p at an exact fp32 tie, i.e. a near-tie.  The select
// kernels then run over the survivors (~10^3 of the 10^6 records at C5).
//
// Layout: K3a/K3c sort the grouped records by length (a counting sort: per-CTA
// shared histograms, one global reservation per (CTA, length)) into rec2 (free
// until K3g); K3d keeps per length its K best keys by (f1, id) and its K lowest
// ids (lists zero-padded to 32) and the K-th of each (0: fewer than K, keep all);
// K3e merges the lists per block of kSkyBlk lengths; K3f turns a position's
// blocks into prefix bounds with a Hillis-Steele scan of top-K lists in shared
// memory; K3g keeps a record if it is in its length's lists and above its
// block's prefix bound (or among the queue's K lowest ids).
__device__ __forceinline__ int sky_len(const float4& f) { return (int)rintf(1.0f / f.x - 1.0f); }
__device__ __forceinline__ bool sky_grouped(const SweepArgs& A, int p, int b) {
    return b >= A.qbin_lo[p] && b < A.qbin_hi[p];
}
__device__ __forceinline__ u64 sky_key(const float4& f) {
    return ((u64)__float_as_uint(f.y) << 32) | (u64)(~__float_as_uint(f.w));
}
__device__ __forceinline__ u64 sky_idkey(const float4& f) { return (u64)(~__float_as_uint(f.w)) + 1ull; }   // larger = lower id
// position of record i (qoff staged in shared memory), advanced from the previous one
__device__ __forceinline__ int sky_pos_from(const int64_t* qoff, int nq, int p, int64_t i) {
    while (p + 1 < nq && qoff[p + 1] <= i) p++;
    return p;
}
__device__ __forceinline__ int sky_pos_search(const int64_t* qoff, int nq, int64_t i) {
    int lo = 0, hi = nq;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (qoff[mid] <= i) lo = mid; else hi = mid;
    }
    return lo;
}
constexpr int kSortBins = 32768;    // per-CTA shared histogram of lengths < kSortBins (128 KB)
constexpr int kSortThreads = 1024;
constexpr int kSkyBig = 1024;       // K3d: lengths with more records are reduced by a whole CTA
constexpr size_t kSortSmem = (size_t)kSortBins * 4;

// Warp streaming top-K (K <= 32): lane i holds the (i+1)-th largest key so far
// (descending, 0 = none).  A chunk of 32 keys (one per lane) none of which beats
// the K-th is skipped with one vote; otherwise it is bitonic-sorted and merged
// (the elementwise max of the list and the reversed chunk is bitonic).
__device__ __forceinline__ u64 sw_bitonic_step(u64 v, int lane, int j, bool up) {
    const u64 o = shfl_xor_u64(v, j);
    const bool keep_max = ((lane & j) == 0) == up;
    return keep_max ? (o > v ? o : v) : (o < v ? o : v);
}
__device__ __forceinline__ u64 topk_add(u64 top, u64 v, int K, int lane) {
    u64 kth = __shfl_sync(0xffffffffu, top, K - 1);
    unsigned m = __ballot_sync(0xffffffffu, v > kth);
    if (!m) return top;
    if (__popc(m) <= 4) {
        // a few keys beat the K-th (the common case once the list is full): insert them
        // one at a time -- rank by one vote, shift the tail down one lane
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1u;
            const u64 x = shfl_idx_u64(v, src);
            if (!(x > kth)) continue;
            const int pos = __popc(__ballot_sync(0xffffffffu, top > x));
            const u64 up = shfl_up_u64(top, 1);
            top = lane < pos ? top : (lane == pos ? x : up);
            kth = __shfl_sync(0xffffffffu, top, K - 1);
        }
        return top;
    }
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) v = sw_bitonic_step(v, lane, j, (lane & k) == 0 || k == 32);
    const u64 r = shfl_xor_u64(v, 31);
    top = r > top ? r : top;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) top = sw_bitonic_step(top, lane, j, true);
    return top;
}
// Merge a sorted list v (descending across the lanes, zeros last) into top: the
// elementwise max of top and the reversed v is bitonic, one 5-step merge sorts it.
__device__ __forceinline__ u64 topk_merge_sorted(u64 top, u64 v, int K, int lane) {
    const u64 kth = __shfl_sync(0xffffffffu, top, K - 1);
    if (!__any_sync(0xffffffffu, v > kth)) return top;
    const u64 r = shfl_xor_u64(v, 31);
    top = r > top ? r : top;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) top = sw_bitonic_step(top, lane, j, true);
    return top;
}

// K3a: per-CTA shared histogram of the grouped records' lengths (global atomics on
// the ~200 hot short lengths took ~250 us at C5)
__global__ void __launch_bounds__(kSortThreads) sky_hist_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    extern __shared__ unsigned s_h[];
    __shared__ int64_t s_qoff[kMaxSlots + 1];
    for (int b = threadIdx.x; b < kSortBins; b += blockDim.x) s_h[b] = 0u;
    for (int q = threadIdx.x; q <= A.nq; q += blockDim.x) s_qoff[q] = A.s.qoff[q];
    __syncthreads();
    int64_t i0, i1;
    sw_cta_range(s_qoff[A.nq], &i0, &i1);
    int p = i0 < i1 ? sky_pos_search(s_qoff, A.nq, i0 + threadIdx.x) : 0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        p = sky_pos_from(s_qoff, A.nq, p, i);
        const int b = sky_len(A.s.rec[i]);
        if (!sky_grouped(A, p, b)) continue;
        if (b < kSortBins) atomicAdd(&s_h[b], 1u); else atomicAdd(&A.s.bcnt[b], 1);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kSortBins; b += blockDim.x)
        if (s_h[b]) atomicAdd(&A.s.bcnt[b], (int)s_h[b]);
}
// K3b: one CTA, exclusive scan of the kSkyBins counts in place (bcnt[kSkyBins] = total):
// warp w scans its contiguous 2048 bins in coalesced rows of 32, then the warp totals
__global__ void __launch_bounds__(1024) sky_scan_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    __shared__ int ws[32];
    const int per = A.sky_nbins / 32;                  // bins per warp (sky_nbins: multiple of 1024)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int* bc = A.s.bcnt + warp * per;
    int tot = 0;
    for (int j = lane; j < per; j += 32) { tot += bc[j]; A.s.bfill[warp * per + j] = 0; }
    tot = __reduce_add_sync(0xffffffffu, tot);
    if (lane == 0) ws[warp] = tot;
    __syncthreads();
    int run = 0;
    for (int w = 0; w < warp; w++) run += ws[w];
    for (int j0 = 0; j0 < per; j0 += 32) {
        const int c = bc[j0 + lane];
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        bc[j0 + lane] = run + incl - c;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 1023) A.s.bcnt[A.sky_nbins] = run;
}
// K3c: the grouped records sorted by length into rec2 (same per-CTA ranges as K3a:
// recount, reserve one range per (CTA, length), place with shared cursors)
__global__ void __launch_bounds__(kSortThreads) sky_scatter_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    extern __shared__ unsigned s_h[];
    __shared__ int64_t s_qoff[kMaxSlots + 1];
    for (int b = threadIdx.x; b < kSortBins; b += blockDim.x) s_h[b] = 0u;
    for (int q = threadIdx.x; q <= A.nq; q += blockDim.x) s_qoff[q] = A.s.qoff[q];
    __syncthreads();
    int64_t i0, i1;
    sw_cta_range(s_qoff[A.nq], &i0, &i1);
    const int pstart = i0 < i1 ? sky_pos_search(s_qoff, A.nq, i0 + threadIdx.x) : 0;
    int p = pstart;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        p = sky_pos_from(s_qoff, A.nq, p, i);
        const int b = sky_len(A.s.rec[i]);
        if (sky_grouped(A, p, b) && b < kSortBins) atomicAdd(&s_h[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kSortBins; b += blockDim.x)
        if (s_h[b]) s_h[b] = (unsigned)A.s.bcnt[b] + (unsigned)atomicAdd(&A.s.bfill[b], (int)s_h[b]);
    __syncthreads();
    p = pstart;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        p = sky_pos_from(s_qoff, A.nq, p, i);
        const float4 f = A.s.rec[i];
        const int b = sky_len(f);
        if (!sky_grouped(A, p, b)) continue;
        const unsigned slot = b < kSortBins ? atomicAdd(&s_h[b], 1u)
                                            : (unsigned)A.s.bcnt[b] + (unsigned)atomicAdd(&A.s.bfill[b], 1);
        EWSJF_CHECK(slot >= (unsigned)A.s.bcnt[b] && slot < (unsigned)A.s.bcnt[b + 1]);
        A.s.rec2[slot] = f;
    }
}
// K3d: per length, its K best records by (f1, id) and its K lowest ids (both lists
// zero-padded to 32 per length; unordered) and the K-th of each (0 when the length
// has <= K records: all of them are candidates).  BIG: one CTA per length with more
// than kSkyBig records (16 warps over slices, then one merge per list); else one warp.
template <bool BIG>
__global__ void __launch_bounds__(kSwPrepThreads) sky_group_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    __shared__ u64 s1[kSwPrepThreads / 32][32], s2[kSwPrepThreads / 32][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int K = A.K;
    // top-K of the keys of records [beg, end) of rec2, 4 chunks of 32 loaded at a time
    auto scan = [&](int beg, int end, u64* t1, u64* t2) {
        u64 a = 0ull, c = 0ull;
        for (int j0 = beg; j0 < end; j0 += 128) {
            float4 f[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int j = j0 + 32 * u + lane;
                f[u] = j < end ? A.s.rec2[j] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const bool v = j0 + 32 * u + lane < end;
                a = topk_add(a, v ? sky_key(f[u]) : 0ull, K, lane);
                c = topk_add(c, v ? sky_idkey(f[u]) : 0ull, K, lane);
            }
        }
        *t1 = a; *t2 = c;
    };
    auto emit = [&](int b, int cnt, u64 k1, u64 k2) {   // one warp
        k1 = lane < K ? k1 : 0ull;
        k2 = lane < K ? k2 : 0ull;
        A.s.lentop[(size_t)b * kSkyMaxK + lane] = k1;
        A.s.lenid[(size_t)b * kSkyMaxK + lane] = k2;
        if (lane == K - 1) {
            A.s.lenkth[2 * (size_t)b] = cnt > K ? k1 : 0ull;
            A.s.lenkth[2 * (size_t)b + 1] = cnt > K ? k2 : 0ull;
        }
    };
    if (BIG) {
        const int nbig = *A.s.nbig;
        for (int x = blockIdx.x; x < nbig; x += gridDim.x) {
            const int b = A.s.biglist[x];
            const int beg = A.s.bcnt[b], end = A.s.bcnt[b + 1], c = end - beg;
            const int per = (c + nwarp - 1) / nwarp;
            const int sb = min(end, beg + warp * per), se = min(end, sb + per);
            u64 k1, k2;
            scan(sb, se, &k1, &k2);
            s1[warp][lane] = k1;
            s2[warp][lane] = k2;
            __syncthreads();
            if (warp < 2) {
                u64 (*s)[32] = warp == 0 ? s1 : s2;
                u64 t = s[0][lane];
                for (int w = 1; w < nwarp; w++) t = topk_merge_sorted(t, s[w][lane], K, lane);
                s[0][lane] = t;
            }
            __syncthreads();
            if (warp == 0) emit(b, c, s1[0][lane], s2[0][lane]);
            __syncthreads();
        }
    } else {
        const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
        for (int b = 2 + w0; b < A.sky_nbins; b += nw) {
            const int beg = A.s.bcnt[b], end = A.s.bcnt[b + 1], c = end - beg;
            if (c > kSkyBig && lane == 0) A.s.biglist[atomicAdd(A.s.nbig, 1)] = b;   // the CTA kernel's
            if (c == 0 || c > kSkyBig) continue;
            u64 k1, k2;
            scan(beg, end, &k1, &k2);
            emit(b, c, k1, k2);
        }
    }
}
// K3e: one CTA per block of kSkyBlk lengths of one position: the top K candidate
// keys (by f1) and the K lowest candidate ids of the block, merged from the
// per-length lists (the block's top K by f1 among all its candidates are among
// the lengths' top K by f1, and likewise for the ids).  Warp w merges lengths
// w, w + 16, ... of the block, warps 0 / 1 merge the 16 partial lists.
__global__ void __launch_bounds__(kSwPrepThreads) sky_block_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    __shared__ u64 s1[kSwPrepThreads / 32][32], s2[kSwPrepThreads / 32][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int K = A.K;
    const int nblk = A.qblk[A.nq];
    for (int g = blockIdx.x; g < nblk; g += gridDim.x) {
        int p = 0;
        while (p + 1 < A.nq && A.qblk[p + 1] <= g) p++;
        const int jj = g - A.qblk[p];
        const int blo = A.qbin_lo[p] + jj * kSkyBlk, bhi = min(blo + kSkyBlk, A.qbin_hi[p]);
        u64 t1 = 0ull, t2 = 0ull;
        for (int b = blo + warp; b < bhi; b += nwarp) {
            if (A.s.bcnt[b + 1] == A.s.bcnt[b]) continue;   // no records: its lists are stale
            t1 = topk_merge_sorted(t1, A.s.lentop[(size_t)b * kSkyMaxK + lane], K, lane);
            t2 = topk_merge_sorted(t2, A.s.lenid[(size_t)b * kSkyMaxK + lane], K, lane);
        }
        s1[warp][lane] = t1;
        s2[warp][lane] = t2;
        __syncthreads();
        if (warp < 2) {
            u64 (*sl)[32] = warp == 0 ? s1 : s2;
            u64 t = sl[0][lane];
            for (int w = 1; w < nwarp; w++) t = topk_merge_sorted(t, sl[w][lane], K, lane);
            (warp == 0 ? A.s.blktop : A.s.blkid)[(size_t)g * kSkyMaxK + lane] = lane < K ? t : 0ull;
        }
        __syncthreads();
    }
}
// K3f: one CTA per position.  pref[g] = high word (f1) of the K-th largest candidate
// key of the position's blocks before g (0 while fewer than K): an exclusive scan
// of the blocks' top-K lists (merge = top K of the union) in shared memory --
// per-warp runs, a Hillis-Steele scan over the 32 run totals, a per-block fix-up --
// segments of kSkyScanSeg blocks with a carried prefix.  qidk[p] =
// the queue's K-th lowest candidate id key (all weights 0: every member scores 0
// and the K lowest ids are the answer, R24), 0 while fewer than K.
constexpr int kSkyScanSeg = 256;
constexpr int kSkyPrefThreads = 1024;
__global__ void __launch_bounds__(kSkyPrefThreads) sky_prefix_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    extern __shared__ u64 s_l[];                       // [kSkyScanSeg][32] per-warp inclusive prefixes
    __shared__ u64 s_carry[32], s_id[kSkyPrefThreads / 32][32], s_w[kSkyPrefThreads / 32][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int p = blockIdx.x;
    if (p >= A.nq) return;
    const int K = A.K;
    const int g0 = A.qblk[p], g1 = A.qblk[p + 1];
    auto kth_hi = [&](u64 top) -> u32 {                // high word of the K-th of a list (0: < K keys)
        return (u32)(__shfl_sync(0xffffffffu, top, K - 1) >> 32);
    };
    if (warp == 0) s_carry[lane] = 0ull;
    // the id lists: each warp folds its share of the blocks, then a tree over the warps
    u64 ti = 0ull;
    for (int g = g0 + warp; g < g1; g += nwarp) ti = topk_merge_sorted(ti, A.s.blkid[(size_t)g * kSkyMaxK + lane], K, lane);
    s_id[warp][lane] = ti;
    __syncthreads();
    for (int d = 1; d < nwarp; d <<= 1) {
        if ((warp & (2 * d - 1)) == 0 && warp + d < nwarp)
            s_id[warp][lane] = topk_merge_sorted(s_id[warp][lane], s_id[warp + d][lane], K, lane);
        __syncthreads();
    }
    if (warp == 0) {
        const u64 kid = __shfl_sync(0xffffffffu, s_id[0][lane], K - 1);
        if (lane == 0) A.s.qidk[p] = kid;
    }
    // the block lists' exclusive prefix, per segment: (1) each warp scans its contiguous
    // run of blocks, (2) a Hillis-Steele scan over the 32 run totals, (3) each block's
    // bound = K-th of (carry ∪ earlier runs ∪ its run's blocks before it)
    for (int s0 = g0; s0 < g1; s0 += kSkyScanSeg) {
        const int n = min(kSkyScanSeg, g1 - s0);
        const int per = (n + nwarp - 1) / nwarp;
        const int j0 = min(n, warp * per), j1 = min(n, j0 + per);
        u64 t = 0ull;
        for (int j = j0; j < j1; j++) {
            t = topk_merge_sorted(t, A.s.blktop[(size_t)(s0 + j) * kSkyMaxK + lane], K, lane);
            s_l[j * 32 + lane] = t;
        }
        s_w[warp][lane] = t;
        __syncthreads();
        for (int d = 1; d < nwarp; d <<= 1) {
            const u64 mine = s_w[warp][lane], other = warp >= d ? s_w[warp - d][lane] : 0ull;
            __syncthreads();
            if (warp >= d) s_w[warp][lane] = topk_merge_sorted(other, mine, K, lane);
            __syncthreads();
        }
        u64 ex = s_carry[lane];
        if (warp > 0) ex = topk_merge_sorted(ex, s_w[warp - 1][lane], K, lane);
        for (int j = j0; j < j1; j++) {
            const u64 before = j == j0 ? ex : topk_merge_sorted(ex, s_l[(j - 1) * 32 + lane], K, lane);
            const u32 h = kth_hi(before);
            if (lane == 0) A.s.pref[s0 + j] = h;
        }
        __syncthreads();
        if (warp == 0) s_carry[lane] = topk_merge_sorted(s_carry[lane], s_w[nwarp - 1][lane], K, lane);
        __syncthreads();
    }
}
__device__ __forceinline__ bool sky_keep(const SweepArgs& A, const float4& f, int p) {
    const int b = sky_len(f);
    if (!sky_grouped(A, p, b)) return true;
    const u64 k1 = sky_key(f), k2 = sky_idkey(f);
    if (!(k1 >= A.s.lenkth[2 * (size_t)b] || k2 >= A.s.lenkth[2 * (size_t)b + 1])) return false;   // not in its length's lists
    if (k2 >= A.s.qidk[p]) return true;                    // among the queue's K lowest ids
    const int g = A.qblk[p] + (b - A.qbin_lo[p]) / kSkyBlk;
    return __float_as_uint(f.y) > A.s.pref[g];
}
// K3g: survivors per position, then (plan2, one thread) the compacted layout, then the scatter
__global__ void __launch_bounds__(kSwPrepThreads) sky_count_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    __shared__ int64_t s_qoff[kMaxSlots + 1];
    __shared__ unsigned s_cnt[kMaxSlots];
    for (int q = threadIdx.x; q <= A.nq; q += blockDim.x) s_qoff[q] = A.s.qoff[q];
    for (int q = threadIdx.x; q < kMaxSlots; q += blockDim.x) s_cnt[q] = 0u;
    __syncthreads();
    int64_t i0, i1;
    sw_cta_range(s_qoff[A.nq], &i0, &i1);
    int p = i0 < i1 ? sky_pos_search(s_qoff, A.nq, i0 + threadIdx.x) : 0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        p = sky_pos_from(s_qoff, A.nq, p, i);
        if (sky_keep(A, A.s.rec[i], p)) atomicAdd(&s_cnt[p], 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < A.nq; q += blockDim.x)
        if (s_cnt[q]) atomicAdd((unsigned long long*)&A.s.qcnt2[q], (unsigned long long)s_cnt[q]);
}
__global__ void sky_plan_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    if (threadIdx.x >= 32) return;
    const int64_t mx = sw_plan_warp(A.s.qcnt2, A.nq, A.chunk, A.s.qoff2, A.s.cpre2, A.s.qfill2);
    if (threadIdx.x == 0) *A.s.direct = mx <= kSwDirectMax;
}
__global__ void __launch_bounds__(kSwPrepThreads) sky_compact_kernel(const SweepArgs* __restrict__ Ap) {
    const SweepArgs& A = *Ap;
    __shared__ int64_t s_qoff[kMaxSlots + 1];
    for (int q = threadIdx.x; q <= A.nq; q += blockDim.x) s_qoff[q] = A.s.qoff[q];
    __syncthreads();
    int64_t i0, i1;
    sw_cta_range(s_qoff[A.nq], &i0, &i1);
    int p = i0 < i1 ? sky_pos_search(s_qoff, A.nq, i0 + threadIdx.x) : 0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        p = sky_pos_from(s_qoff, A.nq, p, i);
        const float4 f = A.s.rec[i];
        if (sky_keep(A, f, p)) {
            const int64_t o = A.s.qoff2[p] + atomicAdd(&A.s.qfill2[p], 1);
            EWSJF_CHECK(o < A.s.qoff2[p + 1]);
            A.s.rec2[o] = f;
        }
    }
}

// K4: persistent warps over tasks (Θ block, queue, chunk).
__global__ void __launch_bounds__(kSwWarps * 32) sweep_select_kernel(const SweepArgs* __restrict__ Ap, int phase) {
    const SweepArgs& A = *Ap;
    extern __shared__ __align__(16) unsigned char smem[];
    if (*A.s.direct) return;                      // K5d handles this sweep
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cap = A.cap, K = A.K;
    u64* buf = (u64*)smem + (size_t)warp * kSwT * cap;           // [kSwT][cap]
    // per (warp, Θ): weights + threshold high word as a float, threshold low word, exact threshold, count
    float4* ws = (float4*)((u64*)smem + (size_t)kSwWarps * kSwT * cap) + warp * kSwT;
    u64* th64 = (u64*)((float4*)((u64*)smem + (size_t)kSwWarps * kSwT * cap) + kSwWarps * kSwT) + warp * kSwT;
    uint32_t* thlo = (uint32_t*)((u64*)((float4*)((u64*)smem + (size_t)kSwWarps * kSwT * cap) + kSwWarps * kSwT) +
                                 kSwWarps * kSwT) + warp * kSwT;
    int* cnt = (int*)(thlo - warp * kSwT + kSwWarps * kSwT) + warp * kSwT;
    // raise (Θ t)'s filter to key th (one lane); the float/low-word copies follow the exact key
    auto raise = [&](int t, u64 th) {
        if (th > th64[t]) {
            th64[t] = th;
            ws[t].w = __uint_as_float((uint32_t)(th >> 32));
            thlo[t] = (uint32_t)th;
        }
    };
    const int nchunks = A.s.cpre[A.nq];
    const int nblocks = (A.n_theta + kSwT - 1) / kSwT;
    // Phase 0 processes the first chunk of every (Θ block, queue) so that the
    // exact K-th keys it publishes filter phase 1 from its first record on.
    const int total = phase == 0 ? nblocks * A.nq : nblocks * nchunks;
    unsigned long long d_ins = 0, d_cuts = 0;     // diagnostics, one atomic per warp at the end
    for (;;) {
        int task = 0;
        if (lane == 0) task = (int)atomicAdd(A.s.task_ctr, 1u);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task >= total) break;
        int blk, q, chunk;
        if (phase == 0) {
            // seeding: per Θ of the block, a valid bound of the K-th key among the
            // queue's first 256 records (scores in registers, register selection)
            blk = task / A.nq;
            q = task % A.nq;
            const int64_t b0 = A.s.qoff[q];
            const int n0 = (int)min((int64_t)(32 * kRegSel), A.s.qoff[q + 1] - b0);
            if (n0 < K) continue;
            float4 f[kRegSel];
#pragma unroll
            for (int r = 0; r < kRegSel; r++) {
                const int j = lane + 32 * r;
                f[r] = j < n0 ? __ldg(&A.s.rec[b0 + j]) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll 1
            for (int t = 0; t < kSwT; t++) {
                const int th = blk * kSwT + t;
                if (th >= A.n_theta) break;
                const float* w = A.s.w + ((size_t)th * A.nq + q) * 3;
                const float w0 = w[0], w1 = w[1], w2 = w[2];
                u64 key[kRegSel];
#pragma unroll
                for (int r = 0; r < kRegSel; r++) {
                    const float sc = fmaf(w2, f[r].z, fmaf(w1, f[r].y, w0 * f[r].x));
                    key[r] = lane + 32 * r < n0 ? score_key(sc, __float_as_uint(f[r].w)) : 0ull;
                }
                const u64 kth = warp_kth_regs<kRegSel>(key, K, kApproxBit, 1 << 30);
                if (lane == 0) atomicMax(&A.s.gthr[(size_t)th * kMaxSlots + q], kth);
            }
            continue;
        } else {
            blk = task / nchunks;
            const int rem = task % nchunks;
            int lo = 0, hi = A.nq;      // last q with cpre[q] <= rem
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (A.s.cpre[mid] <= rem) lo = mid; else hi = mid;
            }
            q = lo;
            chunk = rem - A.s.cpre[q];
        }
        // chunk c = records [c*chunk, (c+1)*chunk) of the queue; phase 0 takes the
        // first chunk0 records of chunk 0, phase 1 the rest (chunk 0 resumes from its row)
        const int64_t cbeg = A.s.qoff[q] + (int64_t)chunk * A.chunk;
        const int64_t cend = min(A.s.qoff[q + 1], cbeg + A.chunk);
        const int64_t beg = cbeg, end = cend;
        const int t0 = blk * kSwT;
        // warp-private state in shared memory: weights + fast threshold per Θ
        // (read as broadcasts), candidate counts
        if (lane < kSwT) {
            const int th = min(t0 + lane, A.n_theta - 1);
            const float* w = A.s.w + ((size_t)th * A.nq + q) * 3;
            const u64 g = __ldcg(&A.s.gthr[(size_t)th * kMaxSlots + q]);
            ws[lane] = make_float4(w[0], w[1], w[2], __uint_as_float((uint32_t)(g >> 32)));
            th64[lane] = g;
            thlo[lane] = (uint32_t)g;
            cnt[lane] = 0;
        }
        __syncwarp();
        // 4 records per lane per step (4 independent 16-byte loads in flight)
        int step = 0;
        for (int64_t e0 = beg; e0 < end; e0 += 128) {
            if ((++step & 7) == 0 && lane < kSwT) {   // share thresholds with the other tasks of (Θ, q)
                const u64 g = __ldcg(&A.s.gthr[(size_t)min(t0 + lane, A.n_theta - 1) * kMaxSlots + q]);
                raise(lane, g);
            }
            __syncwarp();
            float4 f[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int64_t e = e0 + lane + 32 * u;
                f[u] = e < end ? __ldg(&A.s.rec[e]) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            unsigned pass[4] = {0u, 0u, 0u, 0u};
            // fast test on the key's high word (s' >= threshold's s'); equal s' (common
            // when a weight clamps to 0) is decided by the id on the rare path
#pragma unroll
            for (int t = 0; t < kSwT; t++) {
                const float4 w = ws[t];         // (w_base, w_urg, w_fair, threshold high word)
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const float sc = fmaf(w.z, f[u].z, fmaf(w.y, f[u].y, w.x * f[u].x));
                    pass[u] |= (unsigned)(sc >= w.w) << t;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (e0 + lane + 32 * u >= end) pass[u] = 0u;
            if (!__any_sync(0xffffffffu, (pass[0] | pass[1] | pass[2] | pass[3]) != 0u)) continue;
#pragma unroll 1
            for (int u = 0; u < 4; u++) {
                // register selects (no dynamic indexing of f / pass: they stay in registers)
                const float4 fu = u == 0 ? f[0] : (u == 1 ? f[1] : (u == 2 ? f[2] : f[3]));
                unsigned pu = u == 0 ? pass[0] : (u == 1 ? pass[1] : (u == 2 ? pass[2] : pass[3]));
                const uint32_t gid = __float_as_uint(fu.w);
                // each lane inserts its own passing Θ (few bits; no warp-wide loop over Θ)
                while (pu) {
                    const int t = __ffs(pu) - 1;
                    pu &= pu - 1u;
                    const float4 w = ws[t];
                    const float sc = fmaf(w.z, fu.z, fmaf(w.y, fu.y, w.x * fu.x));
                    const u64 key = score_key(sc, gid);
                    if (key >= th64[t]) {                                   // exact (s', ~id) test
                        buf[(size_t)t * cap + atomicAdd(&cnt[t], 1)] = key;  // <= 32 per t per step
                        d_ins++;
                    }
                }
                __syncwarp();
                // cut the buffers that crossed cap - 32 (warp-uniform)
                unsigned full = 0;
                if (lane < kSwT) full = cnt[lane] > cap - 32;
                full = __ballot_sync(0xffffffffu, full);
                while (full) {
                    const int t = __ffs(full) - 1;
                    full &= full - 1u;
                    u64* bt = buf + (size_t)t * cap;
                    int c = cnt[t];
                    const u64 kth = warp_kth_arr(bt, c, K, kApproxBit, K + (cap - 32 - K) / 4);
                    d_cuts++;
                    c = warp_keep_ge(bt, c, kth);
                    if (lane == 0) {
                        raise(t, kth);
                        atomicMax(&A.s.gthr[(size_t)min(t0 + t, A.n_theta - 1) * kMaxSlots + q], kth);
                        cnt[t] = c;
                    }
                    __syncwarp();
                }
            }
        }
        // rows of this task: each Θ keeps the keys >= a valid bound of its local K-th
        // key (K real keys above it, at most K + 32 kept; the merge selects exactly)
        __syncwarp();
#pragma unroll 1
        for (int t = 0; t < kSwT; t++) {
            if (t0 + t >= A.n_theta) break;
            u64* bt = buf + (size_t)t * cap;
            int c = cnt[t];
            if (c >= K) {
                const u64 th = c > K ? warp_kth_arr(bt, c, K, kApproxBit, K + 32) : 0ull;
                if (th) c = warp_keep_ge(bt, c, th);
                u64 mn = ~0ull;                  // the smallest kept key: >= K keys are >= it
                for (int j = lane; j < c; j += 32) mn = bt[j] < mn ? bt[j] : mn;
                mn = warp_min_u64(mn);
                if (lane == 0) atomicMax(&A.s.gthr[(size_t)(t0 + t) * kMaxSlots + q], mn);
            }
            u64* dst = A.s.rows + ((size_t)task * kSwT + t) * A.rcap;
            for (int j = lane; j < c; j += 32) dst[j] = bt[j];
            if (lane == 0) A.s.rowcnt[(size_t)task * kSwT + t] = c;
        }
        __syncwarp();
    }
    d_ins = __reduce_add_sync(0xffffffffu, (unsigned)d_ins);     // inserts are per lane
    if (lane == 0 && (d_ins | d_cuts)) {
        atomicAdd(&A.s.bad[2], d_cuts);
        atomicAdd(&A.s.bad[3], d_ins);
    }
}

struct SweepOutArgs {
    SweepScratch s;
    int32_t nq, K, cap, n_theta, rcap;
    ewsjf_select_out outs[kSwBatch];
};

// K5: one warp per (Θ, queue): merge the rows of the queue's chunks.
__global__ void __launch_bounds__(kSwWarps * 32) sweep_merge_kernel(const SweepOutArgs* __restrict__ Ap) {
    const SweepOutArgs& A = *Ap;
    extern __shared__ __align__(16) unsigned char smem[];
    if (*A.s.direct) return;                      // K5d handles this sweep
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cap = A.cap, K = A.K;
    u64* bb = (u64*)smem + (size_t)warp * cap;
    const int nchunks = A.s.cpre[A.nq];
    const int item = blockIdx.x * kSwWarps + warp;
    if (item >= A.n_theta * A.nq) return;
    const int th = item / A.nq, q = item % A.nq;
    const int blk = th / kSwT, t = th % kSwT;
    const u64 g = __ldcg(&A.s.gthr[(size_t)th * kMaxSlots + q]);
    int n = 0;
    const int c_beg = A.s.cpre[q], c_end = A.s.cpre[q + 1];
    for (int cb = c_beg; cb < c_end; cb += 32) {        // 32 rows at a time, one per lane
        const int c = cb + lane;
        const size_t row = (size_t)(blk * nchunks + c) * kSwT + t;
        const int rc = c < c_end ? A.s.rowcnt[row] : 0;
        const u64* src = A.s.rows + row * A.rcap;
        for (int j = 0; j < A.rcap; j++) {
            const u64 v = j < rc ? src[j] : 0ull;
            const bool keep = j < rc && v >= g;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (!m) {
                if (!__any_sync(0xffffffffu, j + 1 < rc)) break;
                continue;
            }
            if (keep) bb[n + __popc(m & ((1u << lane) - 1u))] = v;
            n += __popc(m);
            if (n > cap - 32) {
                __syncwarp();
                const u64 kth = warp_kth_arr(bb, n, K, kApproxBit, K + (cap - 32 - K) / 4);
                n = warp_keep_ge(bb, n, kth);
            }
        }
    }
    __syncwarp();
    if (n > K) {
        const u64 kth = warp_kth_arr(bb, n, K);
        n = warp_keep_ge(bb, n, kth);
    }
    // rank sort (keys unique, n <= K): entry j goes to rank #(keys > it)
    const ewsjf_select_out& o = A.outs[th];
    const float qi = (float)(q + 1);
    for (int j = lane; j < n; j += 32) {
        const u64 v = bb[j];
        int r = 0;
        for (int i = 0; i < n; i++) r += bb[i] > v;
        o.d_topk_id[(size_t)q * K + r] = (int64_t)key_gid(v);
        o.d_topk_score[(size_t)q * K + r] = qi * key_sp(v);
    }
    for (int r = n + lane; r < K; r += 32) { o.d_topk_id[(size_t)q * K + r] = -1; o.d_topk_score[(size_t)q * K + r] = 0.f; }
    if (lane == 0) {
        const int64_t cnt = A.s.qcount[q];
        o.d_count[q] = cnt;
        u64 best = 0;
        for (int j = 0; j < n; j++) best = bb[j] > best ? bb[j] : best;
        if (cnt == 0 || n == 0) {
            o.d_head_id[q] = -1; o.d_head_score[q] = 0.f; o.d_max_score[q] = 0.f;
        } else {
            const float4 hf = A.s.headf[q];
            const float* w = A.s.w + ((size_t)th * A.nq + q) * 3;
            const float hs = fmaf(w[2], hf.z, fmaf(w[1], hf.y, w[0] * hf.x));
            o.d_head_id[q] = (int64_t)key_gid(A.s.head[q]);
            o.d_head_score[q] = qi * hs;
            o.d_max_score[q] = qi * key_sp(best);
        }
    }
}

// K5d (after the prefilter, <= kSwDirectMax survivors per queue, K <= 32): one warp
// per (Θ, queue) scores the queue's survivors 32 at a time, bitonic-sorts each
// chunk across the lanes and merges it into the running top 32 (one key per lane,
// descending: the elementwise max of the list and the reversed chunk is bitonic,
// a 5-step merge sorts it).  Same keys and outputs as K4 + K5.
__global__ void __launch_bounds__(kSwWarps * 32) sweep_direct_kernel(const SweepOutArgs* __restrict__ Ap) {
    const SweepOutArgs& A = *Ap;
    if (!*A.s.direct) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int item = blockIdx.x * kSwWarps + warp;
    if (item >= A.n_theta * A.nq) return;
    const int th = item / A.nq, q = item % A.nq;
    const int K = A.K;
    const float* w = A.s.w + ((size_t)th * A.nq + q) * 3;
    const float w0 = w[0], w1 = w[1], w2 = w[2];
    const int64_t b0 = A.s.qoff[q], b1 = A.s.qoff[q + 1];
    u64 top = 0ull;                                   // lane i: the (i+1)-th best key so far
    for (int64_t e0 = b0; e0 < b1; e0 += 256) {       // 8 chunks of 32 loaded at a time
        float4 f[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int64_t e = e0 + 32 * u + lane;
            f[u] = e < b1 ? __ldg(&A.s.rec[e]) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const bool ok = e0 + 32 * u + lane < b1;
            const u64 v = ok ? score_key(fmaf(w2, f[u].z, fmaf(w1, f[u].y, w0 * f[u].x)), __float_as_uint(f[u].w)) : 0ull;
            top = topk_add(top, v, K, lane);
        }
    }
    const ewsjf_select_out& o = A.outs[th];
    const float qi = (float)(q + 1);
    const int n = __popc(__ballot_sync(0xffffffffu, top != 0ull));
    if (lane < K) {
        const bool has = lane < n;
        o.d_topk_id[(size_t)q * K + lane] = has ? (int64_t)key_gid(top) : -1;
        o.d_topk_score[(size_t)q * K + lane] = has ? qi * key_sp(top) : 0.f;
    }
    if (lane == 0) {
        const int64_t cnt = A.s.qcount[q];
        o.d_count[q] = cnt;
        if (cnt == 0 || n == 0) {
            o.d_head_id[q] = -1; o.d_head_score[q] = 0.f; o.d_max_score[q] = 0.f;
        } else {
            const float4 hf = A.s.headf[q];
            const float hs = fmaf(w2, hf.z, fmaf(w1, hf.y, w0 * hf.x));
            o.d_head_id[q] = (int64_t)key_gid(A.s.head[q]);
            o.d_head_score[q] = qi * hs;
            o.d_max_score[q] = qi * key_sp(top);
        }
    }
}

// K6: one warp per Θ: Alg. 1 ArgMax over non-empty queues (ties -> lowest position, R24).
__global__ void sweep_summary_kernel(const SweepOutArgs* __restrict__ Ap) {
    const SweepOutArgs& A = *Ap;
    const int th = blockIdx.x;
    const int lane = threadIdx.x & 31;
    if (th >= A.n_theta || threadIdx.x >= 32) return;
    const ewsjf_select_out& o = A.outs[th];
    // lane-parallel: key = (ordered head score, ~position), max = highest score, lowest position
    u64 best = 0ull;
    for (int p = lane; p < A.nq; p += 32)
        if (o.d_count[p] > 0) {
            const u64 k = ((u64)ord_f32(o.d_head_score[p]) << 32) | (u64)(~(u32)p);
            best = k > best ? k : best;
        }
    best = warp_max_u64(best);
    if (lane != 0) return;
    const int primary = best ? (int)(~(u32)best) : -1;
    if (o.d_summary) {
        ewsjf_summary sm;
        memset(&sm, 0, sizeof sm);
        sm.n_queues = A.nq;
        sm.primary = primary;
        sm.n_invalid = (int64_t)A.s.bad[0];
        sm.n_excluded = (int64_t)A.s.bad[1];
        sm.status = (sm.n_invalid || sm.n_excluded) ? EWSJF_ERR_DOMAIN : EWSJF_OK;
        *o.d_summary = sm;
    }
}


// Upload one argument block into the next ring slot (stream-ordered); returns its device copy.
template <typename T>
static const T* sw_upload(ewsjf_ctx* ctx, const T& a) {
    SweepScratch* S = ctx->sw;
    const int i = S->arg_next;
    S->arg_next = (i + 1) % SweepScratch::kArgSlots;
    if (cudaEventSynchronize(S->arg_ev[i]) != cudaSuccess) return nullptr;   // its previous copy has run
    unsigned char* h = S->h_args + (size_t)i * S->arg_slot;
    unsigned char* d = S->d_args + (size_t)i * S->arg_slot;
    memcpy(h, &a, sizeof(T));
    if (cudaMemcpyAsync(d, h, sizeof(T), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
        cudaEventRecord(S->arg_ev[i], ctx->stream) != cudaSuccess)
        return nullptr;
    return (const T*)d;
}

// The same, into a fixed device block (the graphs' arguments).
template <typename T>
static const T* sw_upload_to(ewsjf_ctx* ctx, const T& a, T* dst) {
    SweepScratch* S = ctx->sw;
    const int i = S->arg_next;
    S->arg_next = (i + 1) % SweepScratch::kArgSlots;
    if (cudaEventSynchronize(S->arg_ev[i]) != cudaSuccess) return nullptr;
    unsigned char* h = S->h_args + (size_t)i * S->arg_slot;
    memcpy(h, &a, sizeof(T));
    if (cudaMemcpyAsync(dst, h, sizeof(T), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
        cudaEventRecord(S->arg_ev[i], ctx->stream) != cudaSuccess)
        return nullptr;
    return dst;
}

void sweep_free(ewsjf_ctx* ctx) {
    SweepScratch* S = ctx->sw;
    if (!S) return;
    for (auto e : S->arg_ev)
        if (e) cudaEventDestroy(e);
    for (auto e : S->w_ev)
        if (e) cudaEventDestroy(e);
    if (S->g_prep) cudaGraphExecDestroy(S->g_prep);
    if (S->cap_st) cudaStreamDestroy(S->cap_st);
    if (S->g_batch) cudaGraphExecDestroy(S->g_batch);
    if (S->h_w) cudaFreeHost(S->h_w);
    if (S->h_args) cudaFreeHost(S->h_args);
    void* d[] = {S->d_fix, S->d_args, S->direct, S->lentop, S->lenid, S->blkid, S->qidk, S->bcnt, S->bfill, S->lenkth, S->biglist, S->nbig, S->blktop, S->pref, S->rec2, S->qoff2, S->cpre2, S->qfill2,
                 S->qcnt2, S->rec, S->qcount, S->qoff, S->cpre, S->qfill, S->head, S->headf, S->bad, S->task_ctr, S->gthr,
                 S->rows, S->rowcnt, S->w};
    for (void* p : d)
        if (p) cudaFree(p);
    delete S;
    ctx->sw = nullptr;
}

// Diagnostics of the last sweep (cuts, candidate inserts); false if none ran.
bool sweep_diag(ewsjf_ctx* ctx, unsigned long long* ci, long long* records) {
    if (!ctx->sw || !ctx->sw->bad) return false;
    SweepScratch* S = ctx->sw;
    *records = 0;
    if (S->last_nq > 0 &&
        cudaMemcpy(records, (S->last_sky ? S->qoff2 : S->qoff) + S->last_nq, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return false;
    return cudaMemcpy(ci, ctx->sw->bad + 2, 16, cudaMemcpyDeviceToHost) == cudaSuccess;
}

// Scratch for a snapshot of n requests at depth K (grown on demand, kept by the
// ctx: repeated sweeps of the same size allocate nothing).
ewsjf_status sweep_alloc(ewsjf_ctx* ctx, int64_t n, int64_t tasks, int K) {
    SweepScratch* S = ctx->sw;
    if (!S) {
        S = ctx->sw = new SweepScratch();
        bool ok = cudaMalloc(&S->qcount, 8 * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->qoff, 8 * (kMaxSlots + 1)) == cudaSuccess &&
                  cudaMalloc(&S->cpre, 4 * (kMaxSlots + 1)) == cudaSuccess &&
                  cudaMalloc(&S->qfill, 4 * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->head, 8 * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->headf, 16 * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->bad, 32) == cudaSuccess && cudaMalloc(&S->task_ctr, 4) == cudaSuccess &&
                  cudaMalloc(&S->gthr, 8 * (size_t)kSwBatch * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->w, 12 * (size_t)kSwBatch * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->bcnt, 4 * (size_t)(kSkyBins + 1)) == cudaSuccess &&
                  cudaMalloc(&S->bfill, 4 * (size_t)kSkyBins) == cudaSuccess &&
                  cudaMalloc(&S->blktop, 8 * (size_t)kSkyMaxBlocks * kSkyMaxK) == cudaSuccess &&
                  cudaMalloc(&S->blkid, 8 * (size_t)kSkyMaxBlocks * kSkyMaxK) == cudaSuccess &&
                  cudaMalloc(&S->lentop, 8 * (size_t)kSkyBins * kSkyMaxK) == cudaSuccess &&
                  cudaMalloc(&S->lenid, 8 * (size_t)kSkyBins * kSkyMaxK) == cudaSuccess &&
                  cudaMalloc(&S->lenkth, 16 * (size_t)kSkyBins) == cudaSuccess &&
                  cudaMalloc(&S->biglist, 4 * (size_t)kSkyBins) == cudaSuccess &&
                  cudaMalloc(&S->nbig, 4) == cudaSuccess &&
                  cudaMalloc(&S->qidk, 8 * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->pref, 4 * (size_t)kSkyMaxBlocks) == cudaSuccess &&
                  cudaMalloc(&S->qoff2, 8 * (kMaxSlots + 1)) == cudaSuccess &&
                  cudaMalloc(&S->cpre2, 4 * (kMaxSlots + 1)) == cudaSuccess &&
                  cudaMalloc(&S->qfill2, 4 * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->qcnt2, 8 * kMaxSlots) == cudaSuccess &&
                  cudaMalloc(&S->direct, 4) == cudaSuccess;
        S->arg_slot = (std::max(sizeof(SweepArgs), sizeof(SweepOutArgs)) + 255) & ~(size_t)255;
        ok = ok && cudaMallocHost(&S->h_args, S->arg_slot * SweepScratch::kArgSlots) == cudaSuccess &&
             cudaMalloc(&S->d_args, S->arg_slot * SweepScratch::kArgSlots) == cudaSuccess &&
             cudaMalloc(&S->d_fix, S->arg_slot * 3) == cudaSuccess &&
             cudaStreamCreateWithFlags(&S->cap_st, cudaStreamNonBlocking) == cudaSuccess;
        for (auto& e : S->arg_ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
        for (auto& e : S->w_ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaMallocHost(&S->h_w, 2 * sizeof(float) * 3 * (size_t)kSwBatch * kMaxSlots) == cudaSuccess;
        if (!ok) return fail(ctx, EWSJF_ERR_CUDA, "sweep scratch allocation failed");
    }
    if (S->n_cap < n) {
        for (void* x : {(void*)S->rec, (void*)S->rec2})
            if (x) cudaFree(x);
        S->rec = S->rec2 = nullptr;
        S->n_cap = 0;
        const size_t nn = (size_t)std::max<int64_t>(n, 1);
        if (cudaMalloc(&S->rec, 16 * nn) != cudaSuccess || cudaMalloc(&S->rec2, 16 * nn) != cudaSuccess)
            return fail(ctx, EWSJF_ERR_CUDA, "sweep records allocation failed");
        S->n_cap = n;
    }
    const int64_t rows_need = tasks * kSwT * (int64_t)(kSwMaxK + 32);
    if (S->task_cap < rows_need) {
        if (S->rows) cudaFree(S->rows);
        if (S->rowcnt) cudaFree(S->rowcnt);
        S->rows = nullptr; S->rowcnt = nullptr; S->task_cap = 0;
        if (cudaMalloc(&S->rows, 8 * (size_t)rows_need) != cudaSuccess ||
            cudaMalloc(&S->rowcnt, 4 * (size_t)tasks * kSwT) != cudaSuccess)
            return fail(ctx, EWSJF_ERR_CUDA, "sweep rows allocation failed");
        S->task_cap = rows_need;
    }
    (void)K;
    return EWSJF_OK;
}

}  // namespace ewsjf

using namespace ewsjf;

extern "C" ewsjf_status ewsjf_score_select_sweep(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arrival,
                                                 const float* d_cost, const int32_t* d_qid, int64_t n,
                                                 const ewsjf_partition_t* part, const ewsjf_meta* thetas,
                                                 int32_t n_theta, const ewsjf_select_params* params,
                                                 ewsjf_select_out* outs) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (!part || !thetas || !params || !outs || n_theta < 0 || part->n < 0 || part->n > EWSJF_MAX_QUEUES)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad sweep arguments");
    // Θ ranks scoring policies: the sweep selects by score (SCORE mode), as O11 does
    if (params->mode != EWSJF_SELECT_SCORE) return fail(ctx, EWSJF_ERR_INVALID_ARG, "sweep: SCORE mode only");
    if (params->k < 1 || params->k > ctx->max_k) return fail(ctx, EWSJF_ERR_INVALID_ARG, "k out of range");
    if (n < 0 || (n > 0 && (!d_len || !d_arrival || !d_qid)) || n >= 0xffffffffll)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad pool");
    for (int t = 0; t < n_theta; t++)
        if (!outs[t].d_topk_id || !outs[t].d_topk_score || !outs[t].d_count || !outs[t].d_head_id ||
            !outs[t].d_head_score || !outs[t].d_max_score)
            return fail(ctx, EWSJF_ERR_INVALID_ARG, "sweep outputs must be device buffers");
    if (n_theta == 0) return EWSJF_OK;
    const int K = params->k;
    if (K > kSwMaxK || part->n == 0 || n == 0) {
        // deep selections (and degenerate pools) go through n_theta score_select calls
        ewsjf_status worst = EWSJF_OK;
        for (int32_t t = 0; t < n_theta; t++) {
            ewsjf_weights w[EWSJF_MAX_QUEUES];
            ewsjf_status s = ewsjf_weights_from_meta(&thetas[t], part, w);
            if (s != EWSJF_OK) return s;
            ewsjf_select_out o = outs[t];
            o.h_summary = nullptr;
            s = ewsjf_score_select(ctx, d_len, d_arrival, d_cost, d_qid, n, part, w, params, &o);
            if (s != EWSJF_OK && s != EWSJF_ERR_DOMAIN) return s;
            if (s == EWSJF_ERR_DOMAIN) worst = s;
        }
        return worst;
    }
    CU(cudaSetDevice(ctx->device));
    const int nq = part->n;
    const int chunk = (int)std::max<int64_t>(4096, (n + 3999) / 4000);
    const int64_t max_chunks = n / chunk + nq + 1;
    const int64_t tasks = (int64_t)((kSwBatch + kSwT - 1) / kSwT) * max_chunks;
    // scratch is reserved up front (ewsjf_ctx_reserve_sweep): no allocation on this call
    SweepScratch* S = ctx->sw;
    if (!S || S->n_cap < n || S->task_cap < tasks * kSwT * (int64_t)(kSwMaxK + 32))
        return fail(ctx, EWSJF_ERR_CAPACITY, "sweep: snapshot of %lld requests exceeds the ctx reservation "
                    "(ewsjf_ctx_reserve_sweep)", (long long)n);

    static thread_local SweepArgs A;
    memset(&A, 0, sizeof A);
    A.len = d_len; A.arrival = d_arrival; A.cost = d_cost; A.qid = d_qid; A.n = n;
    // candidate buffer per (warp, Θ): K + 64 <= cap <= 256, shrunk until 8 warps x kSwT buffers fit
    int cap = std::min(256, (K + 64 + 31) & ~31);
    const int budget = ctx->smem_optin > 0 ? ctx->smem_optin : 232448;
    while (cap > K + 64 && (size_t)kSwWarps * kSwT * (cap * 8 + 32) > (size_t)budget) cap -= 32;
    if (cap < K + 64 || (size_t)kSwWarps * kSwT * (cap * 8 + 32) > (size_t)budget)
        return fail(ctx, EWSJF_ERR_UNSUPPORTED, "sweep: k=%d does not fit shared memory", K);
    A.nq = nq; A.K = K; A.cap = cap; A.chunk = chunk; A.chunk0 = std::min(chunk, 1024); A.rcap = K + 32;
    A.now = params->now; A.c0 = params->cost.c0; A.c1 = params->cost.c1; A.c2 = params->cost.c2;
    std::vector<std::pair<int, int>> ids;
    for (int i = 0; i < nq; i++) ids.push_back({part->q[i].id, i});
    std::sort(ids.begin(), ids.end());
    A.nids = nq;
    for (int i = 0; i < nq; i++) { A.sorted_ids[i] = ids[i].first; A.sorted_pos[i] = ids[i].second; }
    for (int i = 0; i < nq; i++) A.mean[i] = part->q[i].mean;
    A.s = *S;
    const bool sky = K <= kSkyMaxK && !getenv("EWSJF_NO_SKY");
    int nb = 0;
    if (sky) {
        for (int p = 0; p < nq; p++) {
            int lo = std::max(2, part->q[p].min_len), hi = std::min(part->q[p].max_len, kSkyBins);
            if (lo >= hi) lo = hi = 0;
            A.qbin_lo[p] = lo; A.qbin_hi[p] = hi; A.qblk[p] = nb;
            nb += (hi - lo + kSkyBlk - 1) / kSkyBlk;
        }
        A.qblk[nq] = nb;
        int maxhi = 0;
        for (int p = 0; p < nq; p++) maxhi = std::max(maxhi, A.qbin_hi[p]);
        A.sky_nbins = std::min(kSkyBins, std::max(1024, (maxhi + 1 + 1023) & ~1023));
    }
    cudaStream_t st = ctx->stream;
    const int pgrid = std::max(1, std::min(ctx->num_sms * 4, (int)((n + kSwPrepThreads - 1) / kSwPrepThreads)));
    const int sgrid = ctx->num_sms * 4;
    const size_t pref_smem = (size_t)kSkyScanSeg * 32 * 8;
    if (sky && !S->sky_attr) {   // per ctx (its device)
        CU(cudaFuncSetAttribute(sky_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSortSmem));
        CU(cudaFuncSetAttribute(sky_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSortSmem));
        CU(cudaFuncSetAttribute(sky_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pref_smem));
        S->sky_attr = true;
    }
    const size_t sel_smem = (size_t)kSwWarps * kSwT * (A.cap * 8 + 16 + 8 + 4 + 4);
    const size_t mrg_smem = (size_t)kSwWarps * A.cap * 8;
    // kernel attributes and occupancy are queried once per shared-memory size (host calls)
    if (S->attr_smem != sel_smem) {   // per ctx (its device), not per host thread
        CU(cudaFuncSetAttribute(sweep_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel_smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&S->occ, sweep_select_kernel, kSwWarps * 32, sel_smem);
        S->attr_smem = sel_smem;
    }
    const int occ = S->occ;
    S->last_nq = nq;
    S->last_sky = sky;
    // The launch sequences: the Θ-independent prep (K1-K3, the prefilter K3a-g) and one
    // Θ batch (K4 x 2, K5 / K5d, K6).  Both are replayed as CUDA graphs (one capture per
    // shape, kernel arguments in fixed device buffers refreshed by a stream-ordered copy
    // before each replay): ~20 small kernels per sweep were launch-bound on the host.
    // `scoped` brackets each launch with the ctx's timing events (direct launches only).
    cudaStream_t cs = st;   // the stream the sequences enqueue on (a private one while capturing)
    auto prep_seq = [&](const SweepArgs* dA, bool scoped) -> cudaError_t {
        int nk = 0;
        auto L = [&](auto f) { nk++; if (scoped) { LaunchScope ls(ctx, KIND_SWEEP); f(); } else f(); };
        cudaMemsetAsync(S->qcount, 0, 8 * kMaxSlots, cs);
        cudaMemsetAsync(S->head, 0, 8 * kMaxSlots, cs);
        cudaMemsetAsync(S->bad, 0, 32, cs);
        L([&] { sweep_count_kernel<<<pgrid, kSwPrepThreads, 0, cs>>>(dA); });
        L([&] { sweep_plan_kernel<<<1, 32, 0, cs>>>(dA); });
        L([&] { sweep_scatter_kernel<<<pgrid, kSwPrepThreads, 0, cs>>>(dA); });
        // Θ-independent candidate prefilter (K <= 32): the select kernels run over the
        // records no other K records dominate in every feature
        cudaMemsetAsync(S->direct, 0, 4, cs);      // sky_plan sets it when the survivors are few
        if (sky) {
            cudaMemsetAsync(S->bcnt, 0, 4 * (size_t)(kSkyBins + 1), cs);
            cudaMemsetAsync(S->nbig, 0, 4, cs);
            cudaMemsetAsync(S->qcnt2, 0, 8 * kMaxSlots, cs);
            L([&] { sky_hist_kernel<<<ctx->num_sms, kSortThreads, kSortSmem, cs>>>(dA); });
            L([&] { sky_scan_kernel<<<1, 1024, 0, cs>>>(dA); });
            L([&] { sky_scatter_kernel<<<ctx->num_sms, kSortThreads, kSortSmem, cs>>>(dA); });
            L([&] { sky_group_kernel<false><<<sgrid, kSwPrepThreads, 0, cs>>>(dA); });
            L([&] { sky_group_kernel<true><<<ctx->num_sms * 2, kSwPrepThreads, 0, cs>>>(dA); });
            L([&] { sky_block_kernel<<<std::max(1, std::min(ctx->num_sms * 3, nb)), kSwPrepThreads, 0, cs>>>(dA); });
            L([&] { sky_prefix_kernel<<<nq, kSkyPrefThreads, pref_smem, cs>>>(dA); });
            L([&] { sky_count_kernel<<<pgrid, kSwPrepThreads, 0, cs>>>(dA); });
            L([&] { sky_plan_kernel<<<1, 32, 0, cs>>>(dA); });
            L([&] { sky_compact_kernel<<<pgrid, kSwPrepThreads, 0, cs>>>(dA); });
        }
        if (!scoped) S->g_prep_kernels = nk;
        return cudaGetLastError();
    };
    auto batch_seq = [&](const SweepArgs* dB, const SweepOutArgs* dO, int bn, bool scoped) -> cudaError_t {
        int nk = 0;
        auto L = [&](auto f) { nk++; if (scoped) { LaunchScope ls(ctx, KIND_SWEEP); f(); } else f(); };
        cudaMemsetAsync(S->gthr, 0, 8 * (size_t)kSwBatch * kMaxSlots, cs);
        for (int ph = 0; ph < 2; ph++) {
            cudaMemsetAsync(S->task_ctr, 0, 4, cs);
            L([&] { sweep_select_kernel<<<ctx->num_sms * std::max(occ, 1), kSwWarps * 32, sel_smem, cs>>>(dB, ph); });
        }
        L([&] { sweep_merge_kernel<<<(bn * nq + kSwWarps - 1) / kSwWarps, kSwWarps * 32, mrg_smem, cs>>>(dO); });
        if (sky) L([&] { sweep_direct_kernel<<<(bn * nq + kSwWarps - 1) / kSwWarps, kSwWarps * 32, 0, cs>>>(dO); });
        L([&] { sweep_summary_kernel<<<bn, 32, 0, cs>>>(dO); });
        if (!scoped) S->g_batch_kernels = nk;
        return cudaGetLastError();
    };
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(st, &cap_st));
    const bool graphs = cap_st == cudaStreamCaptureStatusNone && !getenv("EWSJF_SWEEP_NO_GRAPH");
    // capture `seq` into *exec for `key` unless it already holds that shape
    auto ensure_graph = [&](cudaGraphExec_t* exec, int64_t* have, int64_t key, auto seq) -> cudaError_t {
        if (*exec && *have == key) return cudaSuccess;
        if (*exec) { cudaGraphExecDestroy(*exec); *exec = nullptr; }
        cudaGraph_t g = nullptr;
        // captured on the sweep's private stream (the ctx stream may be the legacy default
        // stream, which cannot be captured); replayed on the ctx stream
        cudaError_t e = cudaStreamBeginCapture(S->cap_st, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return e;
        cs = S->cap_st;
        const cudaError_t es = seq();
        cs = st;
        e = cudaStreamEndCapture(S->cap_st, &g);
        if (es != cudaSuccess) e = es;
        if (e == cudaSuccess) e = cudaGraphInstantiate(exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (e == cudaSuccess) *have = key;
        return e;
    };
    if (graphs) {
        const SweepArgs* dA = sw_upload_to(ctx, A, (SweepArgs*)S->d_fix);
        if (!dA) return fail(ctx, EWSJF_ERR_CUDA, "sweep: argument upload failed");
        const int64_t key = (((int64_t)n * 257 + nq) * 4099 + nb) * 64 + K * 2 + (sky ? 1 : 0);
        cudaError_t e = ensure_graph(&S->g_prep, &S->g_prep_key, key, [&] { return prep_seq(dA, false); });
        if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "sweep prep graph: %s", cudaGetErrorString(e));
        LaunchScope ls(ctx, KIND_SWEEP);
        CU(cudaGraphLaunch(S->g_prep, st));
        ctx->launches += S->g_prep_kernels - 1;
    } else {
        const SweepArgs* dA = sw_upload(ctx, A);
        if (!dA) return fail(ctx, EWSJF_ERR_CUDA, "sweep: argument upload failed");
        CU(prep_seq(dA, true));
    }
    if (sky) { A.s.rec = S->rec2; A.s.qoff = S->qoff2; A.s.cpre = S->cpre2; }   // the select / merge kernels read the survivors
    static thread_local SweepOutArgs O;
    for (int32_t b0 = 0; b0 < n_theta; b0 += kSwBatch) {
        const int bn = std::min(kSwBatch, n_theta - b0);
        A.n_theta = bn;
        for (int t = 0; t < bn; t++) {
            const ewsjf_meta& m = thetas[b0 + t];
            A.theta[t][0] = m.a_b; A.theta[t][1] = m.b_b; A.theta[t][2] = m.a_u;
            A.theta[t][3] = m.b_u; A.theta[t][4] = m.a_f; A.theta[t][5] = m.b_f;
        }
        {   // A7 on the host (O(n_theta x nq), the tick's ewsjf_weights_from_meta arithmetic:
            // round(a b̄) + b in fp64 without contraction, clamp, fp32), one stream-ordered copy
            const int slot = S->w_next;
            S->w_next ^= 1;
            CU(cudaEventSynchronize(S->w_ev[slot]));          // its previous copy has run
            float* hw = S->h_w + (size_t)slot * 3 * kSwBatch * kMaxSlots;
            for (int t = 0; t < bn; t++)
                for (int q = 0; q < nq; q++)
                    for (int x = 0; x < 3; x++) {
                        volatile double prod = A.theta[t][2 * x] * A.mean[q];   // rounded once, as __dmul_rn
                        const double v = prod + A.theta[t][2 * x + 1];
                        hw[((size_t)t * nq + q) * 3 + x] = (float)(v > 0.0 ? v : 0.0);
                    }
            CU(cudaMemcpyAsync(S->w, hw, sizeof(float) * 3 * (size_t)bn * nq, cudaMemcpyHostToDevice, st));
            CU(cudaEventRecord(S->w_ev[slot], st));
        }
        O.s = A.s; O.nq = nq; O.K = K; O.cap = A.cap; O.n_theta = bn; O.rcap = A.rcap;
        for (int t = 0; t < bn; t++) {
            O.outs[t] = outs[b0 + t];
            O.outs[t].h_summary = nullptr;
        }
        if (graphs) {
            const SweepArgs* dB = sw_upload_to(ctx, A, (SweepArgs*)(S->d_fix + S->arg_slot));
            const SweepOutArgs* dO = sw_upload_to(ctx, O, (SweepOutArgs*)(S->d_fix + 2 * S->arg_slot));
            if (!dB || !dO) return fail(ctx, EWSJF_ERR_CUDA, "sweep: argument upload failed");
            const int64_t key = ((((int64_t)bn * 257 + nq) * 64 + K) * 64 + occ) * 2 + (sky ? 1 : 0) + ((int64_t)sel_smem << 40);
            cudaError_t e = ensure_graph(&S->g_batch, &S->g_batch_key, key, [&] { return batch_seq(dB, dO, bn, false); });
            if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "sweep batch graph: %s", cudaGetErrorString(e));
            LaunchScope ls(ctx, KIND_SWEEP);
            CU(cudaGraphLaunch(S->g_batch, st));
            ctx->launches += S->g_batch_kernels - 1;
        } else {
            const SweepArgs* dB = sw_upload(ctx, A);
            const SweepOutArgs* dO = sw_upload(ctx, O);
            if (!dB || !dO) return fail(ctx, EWSJF_ERR_CUDA, "sweep: argument upload failed");
            CU(batch_seq(dB, dO, bn, true));
        }
    }
    return EWSJF_OK;
}

// Reserve the sweep's scratch for snapshots of up to max_n requests (records,
// per-task candidate rows; sizes as the call computes them for nq <= 256).
extern "C" ewsjf_status ewsjf_ctx_reserve_sweep(ewsjf_ctx* ctx, int64_t max_n) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (max_n < 0 || max_n >= 0xffffffffll) return fail(ctx, EWSJF_ERR_INVALID_ARG, "reserve_sweep: bad size");
    CU(cudaSetDevice(ctx->device));
    CU(cudaStreamSynchronize(ctx->stream));
    const int chunk = (int)std::max<int64_t>(4096, (max_n + 3999) / 4000);
    const int64_t max_chunks = max_n / chunk + kMaxSlots + 1;
    const int64_t tasks = (int64_t)((kSwBatch + kSwT - 1) / kSwT) * max_chunks;
    return sweep_alloc(ctx, max_n, tasks, kSwMaxK);
}
