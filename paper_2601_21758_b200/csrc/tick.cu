// tick.cu — the fused EWSJF tick on sm_100a.
//
//  partial_kernel  (K6): one persistent 512-thread CTA per SM streams its
//     contiguous share of the SoA pool through a 3-stage TMA bulk-copy ring
//     (cp.async.bulk + mbarrier), routes every request with a shared-memory
//     length->queue LUT (A8), scores it with Eq. 4 (A10),
//     counts members per queue (warp match-any aggregation) and keeps a
//     threshold-filtered per-queue candidate buffer in shared memory (A11).
//     Gap-falling lengths (A9) are appended to a gap list.
//  merge_kernel    (K7+K8): one CTA per queue merges the per-CTA rows into the
//     exact per-queue top-k / head / max score, runs Alg. 2 (App. D) over the
//     sorted gap list when it is non-empty, and the last CTA picks the ArgMax
//     queue of Alg. 1.
#include <cfloat>
#include <climits>
#include "tick.cuh"

namespace ewsjf {

// ------------------------------------------------------------ smem layout ---
struct PartialSmem {
    int64_t stages, bars, lut, minlen, maxlen, sid, wb, wu, wf, ids, islot, wcnt;
    int64_t thr, sec, bcnt, buf, misc, total;
    int narr;
};
__host__ __device__ inline int64_t al16(int64_t x) { return (x + 15) & ~(int64_t)15; }
__host__ __device__ inline PartialSmem partial_layout(bool route, bool has_cost, bool tma, int lut_size,
                                                      int nslots, int nids, int pass0, int ngs, int cap) {
    PartialSmem L;
    L.narr = 2 + (has_cost ? 1 : 0) + (route ? 0 : 1);
    int64_t o = 0;
    L.stages = o; o += tma ? (int64_t)kStages * L.narr * kTile * 4 : 0;
    L.bars = o;   o = al16(o + kStages * 8);
    L.lut = o;    o = al16(o + (route ? lut_size : 0));
    L.minlen = o; o = al16(o + (route && lut_size == 0 ? 4 * nslots : 0));
    L.maxlen = o; o = al16(o + (route && lut_size == 0 ? 4 * nslots : 0));
    L.sid = o;    o = al16(o + 4 * nslots);
    L.wb = o;     o = al16(o + 4 * nslots);
    L.wu = o;     o = al16(o + 4 * nslots);
    L.wf = o;     o = al16(o + 4 * nslots);
    L.ids = o;    o = al16(o + (route ? 0 : 4 * nids));
    L.islot = o;  o = al16(o + (route ? 0 : 4 * nids));
    L.wcnt = o;   o = al16(o + (pass0 ? (int64_t)kWarps * nslots * 4 : 0));
    L.thr = o;    o = al16(o + 8 * (int64_t)ngs);
    L.sec = o;    o = al16(o + 8 * (int64_t)ngs);
    L.bcnt = o;   o = al16(o + 4 * (int64_t)ngs);
    L.buf = o;    o = al16(o + 8 * (int64_t)ngs * cap);
    L.misc = o;   o = al16(o + 128);
    L.total = o;
    return L;
}

struct Misc {                 // small CTA-wide scratch
    unsigned long long maxk;
    int sel;
    int cnt[3];
};

// Block-wide count of candidate keys >= t among (buffer entry held by this
// thread) ∪ (this thread's pending items of group slot gs).  One barrier.
__device__ __forceinline__ int block_count_ge(u64 t, bool hb, u64 bv, const u64 (&pk)[4], const int (&pg)[4],
                                              unsigned pmask, int gs, Misc* M, int it) {
    int c = (hb && bv >= t) ? 1 : 0;
#pragma unroll
    for (int j = 0; j < 4; j++) c += ((pmask >> j) & 1) && pg[j] == gs && pk[j] >= t;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&M->cnt[it % 3], c);
    __syncthreads();
    int total = M->cnt[it % 3];
    if (threadIdx.x == 0) M->cnt[(it + 2) % 3] = 0;
    return total;
}

// Overflow of group slot gs: pick t with K <= #(keys >= t) <= tgt by bisection
// over the 64-bit key space, drop keys < t, insert the pending keys >= t.
__device__ void compact_slot(int gs, const PartialArgs& A, u64* thr, int* bcnt, u64* buf, Misc* M,
                             u64 (&pk)[4], int (&pg)[4], unsigned& pmask) {
    const int tid = threadIdx.x;
    const int cap = A.cap;
    int nb = bcnt[gs];
    nb = nb < cap ? nb : cap;
    bool hb = tid < nb;
    u64 bv = hb ? buf[(size_t)gs * cap + tid] : 0ull;
    u64 lo = thr[gs];
    // max key
    u64 mx = hb ? bv : 0ull;
#pragma unroll
    for (int j = 0; j < 4; j++)
        if (((pmask >> j) & 1) && pg[j] == gs && pk[j] > mx) mx = pk[j];
    mx = warp_max_u64(mx);
    if (tid == 0) { M->maxk = 0; M->cnt[0] = M->cnt[1] = M->cnt[2] = 0; }
    __syncthreads();
    if ((tid & 31) == 0 && mx) atomicMax(&M->maxk, mx);
    __syncthreads();
    u64 hi = M->maxk + 1ull;
    int it = 0;
    int c = block_count_ge(lo, hb, bv, pk, pg, pmask, gs, M, it++);
    if (c > A.tgt) {
        // invariant: count(lo) >= K, count(hi) < K
        while (hi - lo > 1ull) {
            u64 mid = lo + (hi - lo) / 2ull;
            int cm = block_count_ge(mid, hb, bv, pk, pg, pmask, gs, M, it++);
            if (cm >= A.K) {
                lo = mid;
                if (cm <= A.tgt) break;
            } else {
                hi = mid;
            }
        }
    }
    const u64 t = lo;
    __syncthreads();
    if (tid == 0) bcnt[gs] = 0;
    __syncthreads();
    if (hb && bv >= t) buf[(size_t)gs * cap + atomicAdd(&bcnt[gs], 1)] = bv;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (((pmask >> j) & 1) && pg[j] == gs) {
            if (pk[j] >= t) buf[(size_t)gs * cap + atomicAdd(&bcnt[gs], 1)] = pk[j];
            pmask &= ~(1u << j);
        }
    }
    if (tid == 0) {
        if (t > thr[gs]) thr[gs] = t;
        if (t) atomicMax(&A.gthr[A.g_lo + gs], t);
    }
    __syncthreads();
}

__device__ void handle_overflow(const PartialArgs& A, u64* thr, int* bcnt, u64* buf, Misc* M, u64 (&pk)[4],
                                int (&pg)[4], unsigned& pmask) {
    for (;;) {
        if (threadIdx.x == 0) M->sel = INT_MAX;
        __syncthreads();
        if (pmask) {
            int m = INT_MAX;
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (((pmask >> j) & 1) && pg[j] < m) m = pg[j];
            atomicMin(&M->sel, m);
        }
        __syncthreads();
        const int gs = M->sel;
        if (gs == INT_MAX) break;
        compact_slot(gs, A, thr, bcnt, buf, M, pk, pg, pmask);
    }
}

// ---------------------------------------------------------------- partial ---
template <bool ROUTE, bool HAS_COST, bool USE_LUT>
__global__ void __launch_bounds__(kThreads, 1)
    partial_kernel(const __grid_constant__ PartialArgs A, const __grid_constant__ Policy P) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nslots = P.nslots;
    const int ngs = A.g_hi - A.g_lo;
    const PartialSmem L = partial_layout(ROUTE, HAS_COST, A.tma, USE_LUT ? A.lut_size : 0, nslots, A.nids,
                                         A.pass0, ngs, A.cap);
    uint64_t* bars = (uint64_t*)(smem + L.bars);
    unsigned char* lut = smem + L.lut;
    int* s_min = (int*)(smem + L.minlen);
    int* s_max = (int*)(smem + L.maxlen);
    int* s_sid = (int*)(smem + L.sid);
    float* s_wb = (float*)(smem + L.wb);
    float* s_wu = (float*)(smem + L.wu);
    float* s_wf = (float*)(smem + L.wf);
    int* s_ids = (int*)(smem + L.ids);
    int* s_islot = (int*)(smem + L.islot);
    int* s_wcnt = (int*)(smem + L.wcnt);
    u64* s_thr = (u64*)(smem + L.thr);
    u64* s_sec = (u64*)(smem + L.sec);
    int* s_bcnt = (int*)(smem + L.bcnt);
    u64* s_buf = (u64*)(smem + L.buf);
    Misc* M = (Misc*)(smem + L.misc);
    const int narr = L.narr;
    const int G = gridDim.x;

    // ---- tiles of this CTA and TMA prologue (overlaps the table setup below)
    const int64_t full = A.tma ? A.n / kTile : 0;
    const int64_t t0 = full * blockIdx.x / G, t1 = full * (blockIdx.x + 1) / G;
    auto stage_ptr = [&](int st, int arr) -> int* {
        return (int*)(smem + L.stages + ((int64_t)st * narr + arr) * kTile * 4);
    };
    auto issue = [&](int64_t t, int st) {
        mbar_arrive_expect_tx(&bars[st], (uint32_t)(narr * kTile * 4));
        const int64_t off = t * kTile;
        int a = 0;
        tma_load_1d(stage_ptr(st, a++), A.len + off, kTile * 4, &bars[st]);
        tma_load_1d(stage_ptr(st, a++), A.arrival + off, kTile * 4, &bars[st]);
        if (HAS_COST) tma_load_1d(stage_ptr(st, a++), A.cost + off, kTile * 4, &bars[st]);
        if (!ROUTE) tma_load_1d(stage_ptr(st, a++), A.qid_in + off, kTile * 4, &bars[st]);
    };
    if (A.tma && tid == 0) {
        for (int s = 0; s < kStages; s++) mbar_init(&bars[s], 1);
        fence_mbar_init();
        for (int s = 0; s < kStages && t0 + s < t1; s++) issue(t0 + s, s);
    }

    // ---- policy tables -> smem
    for (int i = tid; i < nslots; i += kThreads) {
        s_sid[i] = P.sid[i];
        s_wb[i] = P.wb[i];
        s_wu[i] = P.wu[i];
        s_wf[i] = P.wf[i];
        if (ROUTE && !USE_LUT) { s_min[i] = P.min_len[i]; s_max[i] = P.max_len[i]; }
    }
    if (!ROUTE)
        for (int i = tid; i < A.nids; i += kThreads) { s_ids[i] = A.sorted_ids[i]; s_islot[i] = A.sorted_slot[i]; }
    if (USE_LUT) {
        // lut[b] = position of the queue containing b, kLutGap otherwise
        uint32_t* lw = (uint32_t*)lut;
        const int nw = (A.lut_size + 3) / 4;
        for (int i = tid; i < nw; i += kThreads) lw[i] = 0x01010101u * kLutGap;
        __syncthreads();
        for (int q = 0; q < nslots; q++) {
            const int lo = P.min_len[q];
            const int hi = min(P.max_len[q], A.lut_size);
            for (int b = lo + tid; b < hi; b += kThreads) lut[b] = (unsigned char)q;
        }
    }
    if (A.pass0 && A.select)
        for (int i = tid; i < kWarps * nslots; i += kThreads) s_wcnt[i] = 0;
    for (int i = tid; i < ngs; i += kThreads) { s_thr[i] = 0ull; s_sec[i] = 0ull; s_bcnt[i] = 0; }
    if (tid == 0) { M->cnt[0] = M->cnt[1] = M->cnt[2] = 0; }
    __syncthreads();

    unsigned long long inv = 0, exc = 0;
    u64 pk[4] = {0, 0, 0, 0};
    int pg[4] = {0, 0, 0, 0};
    unsigned pmask = 0;
    const bool is_score = (A.sp.mode == EWSJF_SELECT_SCORE);

    // Process the 4 consecutive requests [idx0, idx0+nv) held by this thread.
    auto process4 = [&](int64_t idx0, int nv, const int (&b)[4], const float (&ar)[4], const float (&co)[4],
                        const int (&qi)[4]) {
        int slot[4];
        int qo[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int s = (int)kBadSlot;
            if (j < nv) {
                if (ROUTE) {
                    if (b[j] >= 1) {
                        if (USE_LUT) {
                            const int e = (b[j] < A.lut_size) ? (int)lut[b[j]] : (int)kLutGap;
                            s = (e == (int)kLutGap) ? (int)kGapSlot : e;
                        } else {
                            int lo = 0, hi = nslots;
                            while (lo < hi) {
                                int mid = (lo + hi) >> 1;
                                if (s_min[mid] <= b[j]) lo = mid + 1; else hi = mid;
                            }
                            s = (lo > 0 && b[j] < s_max[lo - 1]) ? lo - 1 : (int)kGapSlot;
                        }
                    }
                } else {
                    if (b[j] >= 1) {
                        int lo = 0, hi = A.nids;
                        while (lo < hi) {
                            int mid = (lo + hi) >> 1;
                            if (s_ids[mid] < qi[j]) lo = mid + 1; else hi = mid;
                        }
                        if (lo < A.nids && s_ids[lo] == qi[j]) s = s_islot[lo];
                    }
                }
            }
            slot[j] = (j < nv) ? s : -1;
            qo[j] = (s < nslots) ? s_sid[s] : (s == (int)kGapSlot ? -2 : -1);
        }
        if (ROUTE && A.pass0 && A.qid_out) {
            if (nv == 4 && A.tma) {
                *(int4*)(A.qid_out + idx0) = make_int4(qo[0], qo[1], qo[2], qo[3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (j < nv) A.qid_out[idx0 + j] = qo[j];
            }
        }
        if (A.pass0) {
#pragma unroll
            for (int j = 0; j < 4; j++) inv += (slot[j] == (int)kBadSlot);
            if (ROUTE) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const bool g = slot[j] == (int)kGapSlot;
                    const unsigned m = __ballot_sync(0xffffffffu, g);
                    if (m) {
                        unsigned long long base = 0;
                        const int leader = __ffs(m) - 1;
                        if (lane == leader) base = atomicAdd(&A.ctr->gap_count, (unsigned long long)__popc(m));
                        base = __shfl_sync(0xffffffffu, base, leader);
                        if (g) {
                            const unsigned long long p = base + __popc(m & ((1u << lane) - 1u));
                            if (p < (unsigned long long)A.gap_cap) {
                                GapEntry e;
                                e.gid = A.gbase + (uint32_t)(idx0 + j);
                                e.len = b[j];
                                e.arrival = ar[j];
                                e.cost = HAS_COST ? co[j] : __int_as_float(0x7fc00000);
                                A.gap[p] = e;
                            }
                        }
                    }
                }
            }
        }
        if (!A.select) return;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int s = slot[j];
            bool counted = false;
            u64 k1 = 0, k2 = 0;
            if (s >= 0 && s < nslots) {
                float sp;
                const bool ok = score_sp(b[j], ar[j], HAS_COST ? co[j] : 0.0f, HAS_COST, A.sp, s_wb[s], s_wu[s],
                                         s_wf[s], &sp);
                if (ok) {
                    counted = true;
                    const uint32_t gid = A.gbase + (uint32_t)(idx0 + j);
                    const u64 ks = score_key(sp, gid), kf = fifo_key(ar[j], gid);
                    k1 = is_score ? ks : kf;
                    k2 = is_score ? kf : ks;
                } else if (A.pass0) {
                    exc++;
                }
            }
            if (A.pass0) {
                const unsigned v = counted ? (unsigned)s : 0xffffffffu;
                const unsigned peers = __match_any_sync(0xffffffffu, v);
                if (counted && lane == __ffs(peers) - 1) s_wcnt[warp * nslots + s] += __popc(peers);
            }
            if (counted && s >= A.g_lo && s < A.g_hi) {
                const int gs = s - A.g_lo;
                const u64 th = *(volatile u64*)&s_thr[gs];
                if (k1 >= th) {
                    const int pos = atomicAdd(&s_bcnt[gs], 1);
                    if (pos < A.cap) {
                        s_buf[(size_t)gs * A.cap + pos] = k1;
                    } else {
                        pk[j] = k1;
                        pg[j] = gs;
                        pmask |= 1u << j;
                    }
                }
                if (k2 > *(volatile u64*)&s_sec[gs]) atomicMax(&s_sec[gs], k2);
            }
        }
    };

    // cross-CTA threshold refresh: loads issued at tile start, applied at tile end
    int rr = 0;
    auto gthr_prefetch = [&](u64& g, int& gs) {
        gs = -1;
        g = 0;
        if (warp == 0 && ngs > 0) {
            gs = lane + 32 * rr;
            if (gs < ngs) g = __ldcg(&A.gthr[A.g_lo + gs]); else gs = -1;
        }
    };
    auto gthr_apply = [&](u64 g, int gs) {
        if (gs >= 0 && g > *(volatile u64*)&s_thr[gs]) *(volatile u64*)&s_thr[gs] = g;
        if (warp == 0) { rr++; if (32 * rr >= ngs) rr = 0; }
    };

    if (A.tma) {
        int64_t it = 0;
        for (int64_t t = t0; t < t1; ++t, ++it) {
            const int st = (int)(it % kStages);
            u64 g; int ggs;
            gthr_prefetch(g, ggs);
            mbar_wait(&bars[st], (uint32_t)((it / kStages) & 1));
            const int4 bv = ((const int4*)stage_ptr(st, 0))[tid];
            const float4 av = ((const float4*)stage_ptr(st, 1))[tid];
            float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
            int4 qv = make_int4(0, 0, 0, 0);
            int a = 2;
            if (HAS_COST) cv = ((const float4*)stage_ptr(st, a++))[tid];
            if (!ROUTE) qv = ((const int4*)stage_ptr(st, a++))[tid];
            const int b4[4] = {bv.x, bv.y, bv.z, bv.w};
            const float a4[4] = {av.x, av.y, av.z, av.w};
            const float c4[4] = {cv.x, cv.y, cv.z, cv.w};
            const int q4[4] = {qv.x, qv.y, qv.z, qv.w};
            process4(t * kTile + 4 * tid, 4, b4, a4, c4, q4);
            gthr_apply(g, ggs);
            const int any = __syncthreads_or(pmask != 0);
            if (tid == 0 && t + kStages < t1) {
                fence_proxy_async();
                issue(t + kStages, st);
            }
            if (any) handle_overflow(A, s_thr, s_bcnt, s_buf, M, pk, pg, pmask);
        }
    }
    // direct-load path: the whole pool (no TMA) or the tail after the full tiles
    {
        const int64_t start = full * kTile;
        const int64_t rem = A.n - start;
        const int64_t ntl = (rem + kTile - 1) / kTile;
        const int64_t d0 = A.tma ? (blockIdx.x == G - 1 ? 0 : ntl) : ntl * blockIdx.x / G;
        const int64_t d1 = A.tma ? ntl : ntl * (blockIdx.x + 1) / G;
        for (int64_t t = d0; t < d1; ++t) {
            const int64_t i0 = start + t * kTile + 4 * tid;
            const int nv = (int)max((int64_t)0, min((int64_t)4, A.n - i0));
            int b4[4], q4[4];
            float a4[4], c4[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const bool v = j < nv;
                b4[j] = v ? __ldg(A.len + i0 + j) : 0;
                a4[j] = v ? __ldg(A.arrival + i0 + j) : 0.f;
                c4[j] = (HAS_COST && v) ? __ldg(A.cost + i0 + j) : 0.f;
                q4[j] = (!ROUTE && v) ? __ldg(A.qid_in + i0 + j) : 0;
            }
            process4(i0, nv, b4, a4, c4, q4);
            const int any = __syncthreads_or(pmask != 0);
            if (any) handle_overflow(A, s_thr, s_bcnt, s_buf, M, pk, pg, pmask);
        }
    }
    __syncthreads();

    // ---- rows out: keys >= max(local, global) threshold, secondary, members
    const Rows& R = A.rows;
    for (int gs = warp; gs < ngs; gs += kWarps) {
        const int slot = A.g_lo + gs;
        int nb = s_bcnt[gs];
        nb = nb < A.cap ? nb : A.cap;
        u64 tf = s_thr[gs];
        const u64 gg = __ldcg(&A.gthr[slot]);
        tf = gg > tf ? gg : tf;
        u64* dst = R.keys + ((size_t)slot * G + blockIdx.x) * R.cap;
        int outc = 0;
        for (int j0 = 0; j0 < nb; j0 += 32) {
            const int j = j0 + lane;
            const u64 v = j < nb ? s_buf[(size_t)gs * A.cap + j] : 0ull;
            const bool keep = j < nb && v >= tf;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) dst[outc + __popc(m & ((1u << lane) - 1u))] = v;
            outc += __popc(m);
        }
        if (lane == 0) {
            R.cnt[(size_t)slot * G + blockIdx.x] = outc;
            R.sec[(size_t)slot * G + blockIdx.x] = s_sec[gs];
        }
    }
    if (A.pass0 && A.select) {
        for (int s = tid; s < nslots; s += kThreads) {
            long long m = 0;
            for (int w = 0; w < kWarps; w++) m += s_wcnt[w * nslots + s];
            R.members[(size_t)s * G + blockIdx.x] = m;
        }
    }
    if (A.pass0) {
        inv = __reduce_add_sync(0xffffffffu, (unsigned)inv);
        exc = __reduce_add_sync(0xffffffffu, (unsigned)exc);
        if (lane == 0) {
            if (inv) atomicAdd(&A.ctr->n_invalid, inv);
            if (exc) atomicAdd(&A.ctr->n_excluded, exc);
        }
    }
}

// ------------------------------------------------------------------ merge ---
constexpr int kMThreads = 512;
constexpr int kGapSort = 8192;        // gap entries handled by Alg. 2 per call
constexpr int kRankMax = 512;         // survivors rank-sorted at the end

struct MergeSmem {
    int64_t uni, psp, gslot, mygap, myslot, tables, rowoff, surv, ssp, misc, total;
    int esmem;
};
__host__ __device__ inline MergeSmem merge_layout(int in_mode) {
    MergeSmem L;
    const int64_t uni_bytes = 131072;   // gap-phase sort keys | select-phase candidate pool
    L.esmem = in_mode == MERGE_IN_ROWS ? 16384 : 10240;
    int64_t o = 0;
    L.uni = o;    o += uni_bytes;
    L.psp = in_mode == MERGE_IN_ROWS ? 0 : 8 * (int64_t)L.esmem;   // payloads after the keys (exchange)
    L.gslot = o;  o = al16(o + 2 * kGapSort);
    L.mygap = o;  o = al16(o + 4 * kGapSort);
    L.myslot = o; o = al16(o + 2 * kGapSort);
    L.tables = o; o = al16(o + 4 * 6 * kMaxSlots);
    L.rowoff = o; o = al16(o + 4 * 1025);
    L.surv = o;   o = al16(o + 8 * kRankMax);
    L.ssp = o;    o = al16(o + 4 * kRankMax);
    L.misc = o;   o = al16(o + 256);
    L.total = o;
    return L;
}

struct MMisc {
    unsigned long long maxk;
    unsigned long long sec;
    unsigned long long members;
    int cnt[3];
    int nfinal, nbub, ndrop, nmine, pn, nsurv, is_last, gexc;
    float sec_sp;
};

// A7 for a bubble (device side, same canonical fp64 expression as the host).
__device__ __forceinline__ void bubble_weights(const double* th, double L, float* wb, float* wu, float* wf) {
    const double b = __dadd_rn(__dmul_rn(th[0], L), th[1]);
    const double u = __dadd_rn(__dmul_rn(th[2], L), th[3]);
    const double f = __dadd_rn(__dmul_rn(th[4], L), th[5]);
    *wb = (float)(b > 0.0 ? b : 0.0);
    *wu = (float)(u > 0.0 ? u : 0.0);
    const float f32 = (float)(f > 0.0 ? f : 0.0);
    *wf = (float)__dmul_rn((double)f32, 0.69314718055994530942);
}

// CTA-wide count of pool keys >= t (one barrier; rotating counters).
__device__ __forceinline__ int pool_count_ge(const u64* pool, int n, u64 t, MMisc* M, int it) {
    int c = 0;
    for (int i = threadIdx.x; i < n; i += kMThreads) c += pool[i] >= t;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&M->cnt[it % 3], c);
    __syncthreads();
    const int total = M->cnt[it % 3];
    if (threadIdx.x == 0) M->cnt[(it + 2) % 3] = 0;
    return total;
}

// Shrink the pool to the keys >= t where K <= #(>= t) <= kRankMax (bisection,
// requires #(>= lo) >= K); survivors are moved to the front.
__device__ void pool_shrink(u64* pool, float* psp, int& pn, u64& lo, int K, u64* surv, float* ssp, MMisc* M) {
    const int tid = threadIdx.x;
    u64 mx = 0;
    for (int i = tid; i < pn; i += kMThreads) mx = pool[i] > mx ? pool[i] : mx;
    mx = warp_max_u64(mx);
    __syncthreads();
    if (tid == 0) { M->maxk = 0; M->cnt[0] = M->cnt[1] = M->cnt[2] = 0; M->nsurv = 0; }
    __syncthreads();
    if ((tid & 31) == 0 && mx) atomicMax(&M->maxk, mx);
    __syncthreads();
    u64 hi = M->maxk + 1ull;
    int it = 0;
    while (hi - lo > 1ull) {
        const u64 mid = lo + (hi - lo) / 2ull;
        const int c = pool_count_ge(pool, pn, mid, M, it++);
        if (c >= K) {
            lo = mid;
            if (c <= kRankMax) break;
        } else {
            hi = mid;
        }
    }
    for (int i = tid; i < pn; i += kMThreads) {
        if (pool[i] >= lo) {
            const int p = atomicAdd(&M->nsurv, 1);
            surv[p] = pool[i];
            if (psp) ssp[p] = psp[i];
        }
    }
    __syncthreads();
    pn = M->nsurv;
    for (int i = tid; i < pn; i += kMThreads) {
        pool[i] = surv[i];
        if (psp) psp[i] = ssp[i];
    }
    __syncthreads();
}

template <int IN, int OUT, bool HAS_COST>
__global__ void __launch_bounds__(kMThreads, 1)
    merge_kernel(const __grid_constant__ MergeArgs A, const __grid_constant__ Policy P) {
    extern __shared__ __align__(128) unsigned char smem[];
    const MergeSmem L = merge_layout(IN);
    const int tid = threadIdx.x, lane = tid & 31;
    u64* uni = (u64*)(smem + L.uni);
    float* psp = IN == MERGE_IN_EXCHANGE ? (float*)(smem + L.uni + L.psp) : nullptr;
    int16_t* gslot = (int16_t*)(smem + L.gslot);
    uint32_t* mygap = (uint32_t*)(smem + L.mygap);
    int16_t* myslot = (int16_t*)(smem + L.myslot);
    int* t_lo = (int*)(smem + L.tables);
    int* t_hi = t_lo + kMaxSlots;
    int* t_slot = t_hi + kMaxSlots;   // position -> internal slot
    int* t_pos = t_slot + kMaxSlots;  // internal slot -> position
    int* t_L = t_pos + kMaxSlots;     // bubble creating length (internal slot >= nq)
    int* t_id = t_L + kMaxSlots;      // internal slot -> stable id
    int* rowoff = (int*)(smem + L.rowoff);
    u64* surv = (u64*)(smem + L.surv);
    float* ssp = (float*)(smem + L.ssp);
    MMisc* M = (MMisc*)(smem + L.misc);
    const int nq = A.nq, K = A.K;
    const ExLayout X = ex_layout(nq, K);
    const bool is_score = A.sp.mode == EWSJF_SELECT_SCORE;

    // ---------------- gap list size
    long long graw = 0, gcount = 0;
    if (IN == MERGE_IN_ROWS) {
        graw = (long long)__ldcg(&A.ctr->gap_count);
        gcount = graw < A.gap_cap ? graw : A.gap_cap;
    } else {
        for (int r = 0; r < A.world; r++) {
            const long long c = ((const ExHeader*)(A.ex_in + (int64_t)r * A.ex_bytes))->gap_count;
            graw += c;
            gcount += c < kExGap ? c : kExGap;
        }
    }
    if (gcount > kGapSort) gcount = kGapSort;
    const bool gap_overflow = graw > gcount;
    auto gap_entry = [&](uint32_t src) -> GapEntry {
        if (IN == MERGE_IN_ROWS) return A.gap[src];
        return ((const GapEntry*)(A.ex_in + (int64_t)(src / kExGap) * A.ex_bytes + X.gaps))[src % kExGap];
    };

    // ---------------- final partition: Alg. 2 over the gap list in global index order (R22)
    for (int i = tid; i < nq; i += kMThreads) {
        t_lo[i] = P.min_len[i]; t_hi[i] = P.max_len[i];
        t_slot[i] = i; t_pos[i] = i; t_id[i] = P.sid[i];
    }
    if (tid == 0) { M->nfinal = nq; M->nbub = 0; M->ndrop = 0; M->nmine = 0; M->gexc = 0; }
    __syncthreads();
    const bool do_gaps = gcount > 0 && OUT != MERGE_OUT_EXCHANGE;
    if (do_gaps) {
        int np2 = 1;
        while (np2 < gcount) np2 <<= 1;
        for (int i = tid; i < np2; i += kMThreads) {
            u64 k = ~0ull;
            if (i < gcount) {
                uint32_t src = (uint32_t)i;
                if (IN == MERGE_IN_EXCHANGE) {
                    long long acc = 0;
                    int r = 0;
                    for (; r < A.world; r++) {
                        long long c = ((const ExHeader*)(A.ex_in + (int64_t)r * A.ex_bytes))->gap_count;
                        c = c < kExGap ? c : kExGap;
                        if (i < acc + c) break;
                        acc += c;
                    }
                    src = (uint32_t)(r * kExGap + (i - acc));
                }
                k = ((u64)gap_entry(src).gid << 32) | src;
            }
            uni[i] = k;
        }
        __syncthreads();
        for (int k2 = 2; k2 <= np2; k2 <<= 1) {           // bitonic sort, ascending
            for (int j = k2 >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < np2; i += kMThreads) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const u64 a = uni[i], b = uni[ixj];
                        if ((a > b) == ((i & k2) == 0)) { uni[i] = b; uni[ixj] = a; }
                    }
                }
                __syncthreads();
            }
        }
        if (tid == 0) {   // Alg. 2 with the integer tests of R19/R20
            int n = nq, nb = 0, nd = 0;
            for (int e = 0; e < gcount; e++) {
                const GapEntry g = gap_entry((uint32_t)(uni[e] & 0xffffffffu));
                const int Lq = g.len;
                int lo = 0, hi = n;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (t_lo[mid] <= Lq) lo = mid + 1; else hi = mid;
                }
                const int i = lo - 1;
                int as;
                if (i >= 0 && Lq < t_hi[i]) {
                    as = t_slot[i];
                } else {
                    const bool hl = i >= 0, hr = i + 1 < n;
                    const long long L64 = Lq;
                    if (hl && 10 * L64 <= 11 * (long long)t_hi[i]) {
                        as = t_slot[i];
                    } else if (hr && 10 * L64 >= 9 * (long long)t_lo[i + 1]) {
                        as = t_slot[i + 1];
                    } else if (n >= kMaxSlots) {
                        as = -1;
                        nd++;
                    } else {
                        const long long lb = hl ? t_hi[i] : 1;
                        const long long rb = hr ? t_lo[i + 1] : (1ll << 40);
                        const long long avail = rb - lb;
                        const long long rg = (long long)A.bubble_width < avail ? (long long)A.bubble_width : avail;
                        long long nlo = L64 - rg / 2;
                        if (nlo < lb) nlo = lb;
                        long long nhi = L64 + (rg + 1) / 2;
                        if (nhi > rb) nhi = rb;
                        if (nhi > INT_MAX) nhi = INT_MAX;
                        for (int p = n; p > i + 1; p--) {
                            t_lo[p] = t_lo[p - 1]; t_hi[p] = t_hi[p - 1]; t_slot[p] = t_slot[p - 1];
                        }
                        const int ns = nq + nb;
                        t_lo[i + 1] = (int)nlo; t_hi[i + 1] = (int)nhi; t_slot[i + 1] = ns;
                        t_L[ns] = Lq;
                        t_id[ns] = A.next_id + nb;
                        if (A.blog && blockIdx.x == 0) {
                            A.blog->pos[nb] = i + 1; A.blog->lo[nb] = (int)nlo;
                            A.blog->hi[nb] = (int)nhi; A.blog->L[nb] = Lq;
                        }
                        n++; nb++;
                        as = ns;
                    }
                }
                gslot[e] = (int16_t)as;
            }
            M->nfinal = n; M->nbub = nb; M->ndrop = nd;
        }
        __syncthreads();
        for (int p = tid; p < M->nfinal; p += kMThreads) t_pos[t_slot[p]] = p;
        if (blockIdx.x == 0 && A.qid) {   // qid write-back of this rank's gap requests
            for (int e = tid; e < gcount; e += kMThreads) {
                const GapEntry g = gap_entry((uint32_t)(uni[e] & 0xffffffffu));
                const long long li = (long long)g.gid - (long long)A.gbase;
                if (li >= 0 && li < A.n_local) { const int as = gslot[e]; A.qid[li] = as >= 0 ? t_id[as] : -1; }
            }
        }
        // keep the gap requests of the slots this CTA will merge (uni is reused below)
        for (int e = tid; e < gcount; e += kMThreads) {
            const int as = gslot[e];
            if (as >= 0 && as % (int)gridDim.x == (int)blockIdx.x) {
                const int p = atomicAdd(&M->nmine, 1);
                mygap[p] = (uint32_t)(uni[e] & 0xffffffffu);
                myslot[p] = (int16_t)as;
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && A.blog && tid == 0) A.blog->n = M->nbub;
    const int nfinal = M->nfinal;
    const int nmine_all = M->nmine;
    const int nloop = OUT == MERGE_OUT_ROUTE ? 0 : (OUT == MERGE_OUT_EXCHANGE ? nq : nfinal);

    for (int s = blockIdx.x; s < nloop; s += gridDim.x) {
        float wb, wu, wf;
        if (s < nq) { wb = P.wb[s]; wu = P.wu[s]; wf = P.wf[s]; }
        else bubble_weights(A.theta, (double)t_L[s], &wb, &wu, &wf);
        // payload s' of a local-pool request (rows input)
        auto recompute = [&](uint32_t gid) -> float {
            const long long li = (long long)gid - (long long)A.gbase;
            float sp = 0.f;
            if (li >= 0 && li < A.n_local)
                score_sp(__ldg(A.len + li), __ldg(A.arrival + li), HAS_COST ? __ldg(A.cost + li) : 0.f, HAS_COST,
                         A.sp, wb, wu, wf, &sp);
            return sp;
        };
        auto gap_keys = [&](const GapEntry& g, u64& k1, u64& k2, float& sp) -> bool {
            const bool hc = !(g.cost != g.cost);
            const bool ok = score_sp(g.len, g.arrival, hc ? g.cost : 0.f, hc, A.sp, wb, wu, wf, &sp);
            const u64 ks = score_key(sp, g.gid), kf = fifo_key(g.arrival, g.gid);
            k1 = is_score ? ks : kf;
            k2 = is_score ? kf : ks;
            return ok;
        };
        __syncthreads();
        if (tid == 0) { M->members = 0; M->sec = 0; M->sec_sp = 0.f; M->gexc = 0; M->pn = 0; }
        // ---- rows: prefix of counts
        const int nrows = IN == MERGE_IN_ROWS ? A.rows.G : A.world;
        if (tid == 0) {
            int acc = 0;
            for (int r = 0; r < nrows; r++) {
                rowoff[r] = acc;
                if (s < nq) {
                    acc += IN == MERGE_IN_ROWS ? A.rows.cnt[(size_t)s * A.rows.G + r]
                                               : ((const int*)(A.ex_in + (int64_t)r * A.ex_bytes + X.cnt))[s];
                }
            }
            rowoff[nrows] = acc;
        }
        __syncthreads();
        // ---- members and secondary (rows + this slot's gap requests)
        {
            unsigned long long m = 0;
            u64 sk = 0;
            float ssk = 0.f;
            int gex = 0;
            if (s < nq) {
                for (int r = tid; r < nrows; r += kMThreads) {
                    u64 k;
                    float kp = 0.f;
                    if (IN == MERGE_IN_ROWS) {
                        m += (unsigned long long)A.rows.members[(size_t)s * A.rows.G + r];
                        k = A.rows.sec[(size_t)s * A.rows.G + r];
                    } else {
                        const unsigned char* rec = A.ex_in + (int64_t)r * A.ex_bytes;
                        m += (unsigned long long)((const int64_t*)(rec + X.members))[s];
                        k = ((const u64*)(rec + X.sec))[s];
                        kp = ((const float*)(rec + X.sec_sp))[s];
                    }
                    if (k > sk) { sk = k; ssk = kp; }
                }
            }
            for (int e = tid; e < nmine_all; e += kMThreads) {
                if (myslot[e] != s) continue;
                u64 k1, k2;
                float sp;
                if (gap_keys(gap_entry(mygap[e]), k1, k2, sp)) {
                    m++;
                    if (k2 > sk) { sk = k2; ssk = sp; }
                } else {
                    gex++;
                }
            }
            for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
            gex = __reduce_add_sync(0xffffffffu, gex);
            const u64 wm = warp_max_u64(sk);
            const unsigned holder = __ballot_sync(0xffffffffu, sk == wm && wm != 0);
            const float wsp = __shfl_sync(0xffffffffu, ssk, holder ? __ffs(holder) - 1 : 0);
            if (lane == 0) {
                if (m) atomicAdd(&M->members, m);
                if (gex) atomicAdd(&M->gexc, gex);
                if (wm) atomicMax(&M->sec, wm);
            }
            __syncthreads();
            if (lane == 0 && wm && wm == M->sec) M->sec_sp = wsp;   // keys are unique: one writer
            __syncthreads();
        }

        // ---- candidate pool: rows entries then this slot's gap requests
        u64 thr = 0;
        int pn = 0;
        const int total_rows = rowoff[nrows];
        const int total = total_rows + nmine_all;
        int e0 = 0;
        while (e0 < total) {
            const int space = L.esmem - pn;
            if (space < kMThreads && pn > kRankMax) {
                pool_shrink(uni, psp, pn, thr, K, surv, ssp, M);
                continue;
            }
            const int take = min(total - e0, space);
            if (tid == 0) M->pn = pn;
            __syncthreads();
            for (int i = tid; i < take; i += kMThreads) {
                const int e = e0 + i;
                u64 key = 0;
                float sp = 0.f;
                bool ok = false;
                if (e < total_rows) {
                    int lo = 0, hi = nrows;       // row r with rowoff[r] <= e < rowoff[r+1]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (rowoff[mid] <= e) lo = mid; else hi = mid;
                    }
                    const int j = e - rowoff[lo];
                    if (IN == MERGE_IN_ROWS) {
                        key = A.rows.keys[((size_t)s * A.rows.G + lo) * A.rows.cap + j];
                    } else {
                        const unsigned char* rec = A.ex_in + (int64_t)lo * A.ex_bytes;
                        key = ((const u64*)(rec + X.keys))[(size_t)s * K + j];
                        sp = ((const float*)(rec + X.sp))[(size_t)s * K + j];
                    }
                    ok = true;
                } else if (myslot[e - total_rows] == s) {
                    u64 k2;
                    ok = gap_keys(gap_entry(mygap[e - total_rows]), key, k2, sp);
                }
                if (ok && key >= thr) {
                    const int p = atomicAdd(&M->pn, 1);
                    uni[p] = key;
                    if (psp) psp[p] = sp;
                }
            }
            __syncthreads();
            pn = M->pn;
            e0 += take;
        }
        if (pn > kRankMax) pool_shrink(uni, psp, pn, thr, K, surv, ssp, M);
        // rank sort (keys unique) -> surv[0..pn) descending
        for (int i = tid; i < pn; i += kMThreads) {
            const u64 k = uni[i];
            int r = 0;
            for (int j = 0; j < pn; j++) r += uni[j] > k;
            surv[r] = k;
            if (psp) ssp[r] = psp[i];
        }
        __syncthreads();
        const int nout = pn < K ? pn : K;
        auto payload = [&](int r) -> float {     // s' of ranked entry r
            const u64 k = surv[r];
            if (is_score) return key_sp(k);
            if (IN == MERGE_IN_EXCHANGE) return ssp[r];
            return recompute(key_gid(k));
        };
        const unsigned long long members = M->members;
        const u64 sec = M->sec;
        float sec_payload = 0.f;
        if (sec) {
            if (!is_score) sec_payload = key_sp(sec);                 // SCORE-keyed: s' is the key
            else if (IN == MERGE_IN_EXCHANGE) sec_payload = M->sec_sp;  // carried by the records
            else sec_payload = recompute(key_gid(sec));               // local pool
        }

        if (OUT == MERGE_OUT_FINAL) {
            const int pos = t_pos[s];
            const float qi = (float)(pos + 1);
            for (int r = tid; r < K; r += kMThreads) {
                const size_t o = (size_t)pos * K + r;
                if (r < nout) {
                    A.topk_id[o] = (int64_t)key_gid(surv[r]);
                    A.topk_score[o] = qi * payload(r);
                } else {
                    A.topk_id[o] = -1;
                    A.topk_score[o] = 0.f;
                }
            }
            if (tid == 0) {
                A.count[pos] = (int64_t)members;
                if (members == 0 || nout == 0) {
                    A.head_id[pos] = -1; A.head_score[pos] = 0.f; A.max_score[pos] = 0.f;
                } else if (is_score) {
                    A.head_id[pos] = (int64_t)key_gid(sec);
                    A.head_score[pos] = qi * sec_payload;
                    A.max_score[pos] = qi * key_sp(surv[0]);
                } else {
                    A.head_id[pos] = (int64_t)key_gid(surv[0]);
                    A.head_score[pos] = qi * payload(0);
                    A.max_score[pos] = qi * key_sp(sec);
                }
            }
        } else {   // MERGE_OUT_EXCHANGE: this rank's record
            unsigned char* rec = A.ex_out;
            for (int r = tid; r < nout; r += kMThreads) {
                ((u64*)(rec + X.keys))[(size_t)s * K + r] = surv[r];
                ((float*)(rec + X.sp))[(size_t)s * K + r] = payload(r);
            }
            if (tid == 0) {
                ((int*)(rec + X.cnt))[s] = nout;
                ((int64_t*)(rec + X.members))[s] = (int64_t)members;
                ((u64*)(rec + X.sec))[s] = sec;
                ((float*)(rec + X.sec_sp))[s] = sec_payload;
            }
        }
        if (IN == MERGE_IN_ROWS && s < nq && tid == 0) A.gthr[s] = 0ull;
        if (tid == 0 && M->gexc) atomicAdd(&A.ctr->n_excluded, (unsigned long long)M->gexc);
    }
    if (IN == MERGE_IN_ROWS && OUT == MERGE_OUT_ROUTE)
        for (int i = blockIdx.x * kMThreads + tid; i < nq; i += gridDim.x * kMThreads) A.gthr[i] = 0ull;
    if (OUT == MERGE_OUT_EXCHANGE && blockIdx.x == 0) {   // header + gap entries of this rank
        const int ng = (int)(graw < kExGap ? graw : kExGap);
        for (int i = tid; i < ng; i += kMThreads) ((GapEntry*)(A.ex_out + X.gaps))[i] = A.gap[i];
        if (tid == 0) {
            ExHeader* h = (ExHeader*)(A.ex_out + X.hdr);
            h->gap_count = graw;
            h->n_invalid = (int64_t)__ldcg(&A.ctr->n_invalid);
            h->n_excluded = (int64_t)__ldcg(&A.ctr->n_excluded);
        }
    }

    // ---------------- last CTA: Alg. 1 ArgMax (ties -> lowest index R24), summary, reset
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const unsigned t = atomicAdd(&A.ctr->ticket, 1u);
        M->is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!M->is_last || tid != 0) return;
    __threadfence();
    long long inv = (long long)__ldcg(&A.ctr->n_invalid) + M->ndrop;
    long long exc = (long long)__ldcg(&A.ctr->n_excluded);
    if (IN == MERGE_IN_EXCHANGE) {
        for (int r = 0; r < A.world; r++) {
            const ExHeader* h = (const ExHeader*)(A.ex_in + (int64_t)r * A.ex_bytes);
            inv += h->n_invalid;
            exc += h->n_excluded;
        }
    }
    if (OUT != MERGE_OUT_EXCHANGE && A.summary) {
        int primary = -1;
        float best = 0.f;
        if (OUT == MERGE_OUT_FINAL) {
            for (int p = 0; p < nfinal; p++) {
                if (__ldcg(&A.count[p]) > 0) {
                    const float h = __ldcg(&A.head_score[p]);
                    if (primary < 0 || h > best) { primary = p; best = h; }
                }
            }
        }
        ewsjf_summary sm;
        sm.n_queues = nfinal;
        sm.primary = primary;
        sm.n_invalid = inv;
        sm.n_excluded = exc;
        sm.n_gap = graw;
        sm.n_bubbles = M->nbub;
        sm.n_dropped = M->ndrop;
        sm.status = (gap_overflow || M->ndrop) ? EWSJF_ERR_CAPACITY : ((inv || exc) ? EWSJF_ERR_DOMAIN : EWSJF_OK);
        sm.pad = 0;
        *A.summary = sm;
    }
    A.ctr->n_invalid = 0;
    A.ctr->n_excluded = 0;
    A.ctr->gap_count = 0;
    A.ctr->ticket = 0;
}

// ---------------------------------------------------------------- launch ---
template <bool R, bool C, bool U>
static cudaError_t launch_partial_t(const PartialArgs& A, const Policy& P, int grid, cudaStream_t st) {
    const PartialSmem L = partial_layout(R, C, A.tma, U ? A.lut_size : 0, P.nslots, A.nids, A.pass0,
                                         A.g_hi - A.g_lo, A.cap);
    auto k = partial_kernel<R, C, U>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    k<<<grid, kThreads, L.total, st>>>(A, P);
    return cudaGetLastError();
}

cudaError_t launch_partial(const PartialArgs& A, const Policy& P, bool route, bool has_cost, bool use_lut, int grid,
                           cudaStream_t st) {
    if (route) {
        if (has_cost) return use_lut ? launch_partial_t<true, true, true>(A, P, grid, st)
                                     : launch_partial_t<true, true, false>(A, P, grid, st);
        return use_lut ? launch_partial_t<true, false, true>(A, P, grid, st)
                       : launch_partial_t<true, false, false>(A, P, grid, st);
    }
    return has_cost ? launch_partial_t<false, true, false>(A, P, grid, st)
                    : launch_partial_t<false, false, false>(A, P, grid, st);
}

int64_t partial_smem_bytes(bool route, bool has_cost, bool tma, int lut_size, int nslots, int nids, int pass0, int ngs,
                           int cap) {
    return partial_layout(route, has_cost, tma, lut_size, nslots, nids, pass0, ngs, cap).total;
}

template <int I, int O, bool C>
static cudaError_t launch_merge_t(const MergeArgs& A, const Policy& P, int grid, cudaStream_t st) {
    const MergeSmem L = merge_layout(I);
    auto k = merge_kernel<I, O, C>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    k<<<grid, kMThreads, L.total, st>>>(A, P);
    return cudaGetLastError();
}

cudaError_t launch_merge(const MergeArgs& A, const Policy& P, bool has_cost, int grid, cudaStream_t st) {
    if (A.in_mode == MERGE_IN_ROWS) {
        if (A.out_mode == MERGE_OUT_FINAL)
            return has_cost ? launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_FINAL, true>(A, P, grid, st)
                            : launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_FINAL, false>(A, P, grid, st);
        if (A.out_mode == MERGE_OUT_EXCHANGE)
            return has_cost ? launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_EXCHANGE, true>(A, P, grid, st)
                            : launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_EXCHANGE, false>(A, P, grid, st);
        return launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_ROUTE, false>(A, P, grid, st);
    }
    return launch_merge_t<MERGE_IN_EXCHANGE, MERGE_OUT_FINAL, false>(A, P, grid, st);
}

}  // namespace ewsjf
