// partial.cu — the streaming pass of the EWSJF tick (K6) and the fused tick
// kernel (K6 + grid barrier + K7/K8 merge) on sm_100a.
//
// One persistent 512-thread CTA per SM streams a contiguous share of the SoA
// pool (len, arrival, cost[, qid]) through a 3-stage ring of 1-D TMA bulk
// copies (cp.async.bulk + mbarrier, 8 KB per array per stage).  Per request,
// with no per-request atomics and almost no branches:
//   A8  route: length -> queue position through a shared-memory byte LUT
//       (P:162); gap-falling lengths go to a gap list for Alg. 2 (App. D);
//   A10 score: s' = Φ/q_i of Eq. 4 with the queue's weights
//       (float4 per queue in shared memory, MUFU lg2 + rcp);
//   A11 count the member (per-thread u16 counters) and compare its key's high
//       word with the queue's running threshold; the rare survivors enter a
//       per-queue shared-memory candidate buffer, the rarer buffer overflows an
//       overflow list, resolved once per tile by a warp-per-queue compaction
//       (exact 64-bit threshold by quickselect on the candidates).
// Thresholds are shared across CTAs through global memory (atomicMax), so a
// CTA holding only newer / lower-scored requests stops inserting early.
// The fused kernel (cooperative launch, all CTAs co-resident) then crosses a
// grid barrier and runs the merge phase (merge.cuh) on the L2-resident rows.
#include <climits>
#include <cstdlib>
#include "merge.cuh"

namespace ewsjf {

__host__ __device__ inline int64_t al16(int64_t x) { return (x + 15) & ~(int64_t)15; }

constexpr int kCodeGap = 0xFE;     // LUT / route code: gap-falling length
constexpr int kCodeBad = 0xFF;     // len < 1 or unknown qid
constexpr int kCodeNone = 0x1FF;   // no request (ragged tail)
constexpr int kW4 = 256;           // weight table entries (codes index it directly)

struct PartialSmem {
    int64_t stages, bars, lut, minlen, maxlen, sid, w4, ids, islot, cnt;
    int64_t thr64, thrhi, sec, bcnt, ovfcnt, exact, bstage, buf, ovfk, ovfs, misc, total;
    int narr;
};
__host__ __device__ inline PartialSmem partial_layout(bool route, bool has_cost, bool tma, int lut_size, int nslots,
                                                      int nids, int pass0, int cnt_thread, int ngs, int cap) {
    PartialSmem L;
    L.narr = 2 + (has_cost ? 1 : 0) + (route ? 0 : 1);
    int64_t o = 0;
    L.stages = o; o += tma ? (int64_t)kStages * L.narr * kTile * 4 : 0;
    L.bars = o;   o = al16(o + kStages * 8);
    L.lut = o;    o = al16(o + (route ? lut_size : 0));
    L.minlen = o; o = al16(o + (route && lut_size == 0 ? 4 * nslots : 0));
    L.maxlen = o; o = al16(o + (route && lut_size == 0 ? 4 * nslots : 0));
    L.sid = o;    o = al16(o + 4 * kW4);
    L.w4 = o;     o = al16(o + 16 * kW4);
    L.ids = o;    o = al16(o + (route ? 0 : 4 * nids));
    L.islot = o;  o = al16(o + (route ? 0 : 4 * nids));
    L.cnt = o;    o = al16(o + (pass0 ? (cnt_thread ? 2LL * kThreads * nslots : 4LL * kWarps * nslots) : 0));
    L.thr64 = o;  o = al16(o + 8 * (int64_t)ngs);
    L.thrhi = o;  o = al16(o + 4 * (int64_t)ngs);
    L.sec = o;    o = al16(o + 8 * (int64_t)ngs);
    L.bcnt = o;   o = al16(o + 4 * (int64_t)ngs);
    L.ovfcnt = o; o = al16(o + 4 * (int64_t)ngs);
    L.exact = o;  o = al16(o + 4 * (int64_t)ngs);
    L.bstage = o; o = al16(o + 8 * 320);
    L.buf = o;    o = al16(o + 8 * (int64_t)ngs * cap);
    L.ovfk = o;   o = al16(o + 8 * kTile);
    L.ovfs = o;   o = al16(o + 2 * kTile);
    L.misc = o;   o = al16(o + 128);
    L.total = o;
    return L;
}

struct PMisc {
    int novf;       // overflow list fill (this tile)
    int want;       // some buffer crossed its high-water mark
    long long tile[kStages];   // dynamic scheduling: tile held by each stage (>= full: end / tail)
};

// Warp-level quickselect over a queue's candidates (buffer keys + its overflow
// keys): returns t with K <= #(keys >= t) <= tgt, given #(keys >= lo) > tgt.
// Pivots are candidate keys strictly inside (lo, hi); keys are unique.
template <typename CountFn, typename PickFn>
__device__ __forceinline__ u64 warp_select(u64 lo, int K, int tgt, CountFn count_ge, PickFn pick_in) {
    const int lane = threadIdx.x & 31;
    u64 hi = ~0ull;
    for (int it = 0; it < 128; it++) {
        u64 p;
        const bool has = pick_in(lo, hi, p);
        const unsigned m = __ballot_sync(0xffffffffu, has);
        if (!m) break;                              // no candidate strictly between: t = lo
        const int nset = __popc(m);
        const int src = __fns(m, 0, 1 + (int)((it * 0x9E3779B9u + 17u) % (unsigned)nset));
        const u64 piv = ((u64)__shfl_sync(0xffffffffu, (u32)(p >> 32), src) << 32) |
                        (u64)__shfl_sync(0xffffffffu, (u32)p, src);
        const int c = count_ge(piv);
        if (c >= K) {
            lo = piv;
            if (c <= tgt) break;
        } else {
            hi = piv;
        }
        (void)lane;
    }
    return lo;
}

// ---------------------------------------------------------------- phase ---
// FAST: the fused single-pass tick — all queues in one group, member counts in
// per-thread u16 counters, TMA with dynamic tile scheduling; the per-request
// path has no runtime flag checks and no per-request counters besides the
// member count (invalid requests are derived from the totals at the end).
template <int MODE, bool ROUTE, bool HAS_COST, bool USE_LUT, bool FAST>
__device__ __forceinline__ void partial_phase(const PartialArgs& A, const Policy& P, unsigned char* smem) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nslots = P.nslots;
    const int ngs = FAST ? nslots : A.g_hi - A.g_lo;
    const int g_lo = FAST ? 0 : A.g_lo;
    const int cap = A.cap;
    const PartialSmem L = partial_layout(ROUTE, HAS_COST, A.tma, USE_LUT ? A.lut_size : 0, nslots, A.nids, A.pass0,
                                         A.cnt_thread, ngs, cap);
    uint64_t* bars = (uint64_t*)(smem + L.bars);
    unsigned char* lut = smem + L.lut;
    int* s_min = (int*)(smem + L.minlen);
    int* s_max = (int*)(smem + L.maxlen);
    int* s_sid = (int*)(smem + L.sid);
    float4* s_w4 = (float4*)(smem + L.w4);
    int* s_ids = (int*)(smem + L.ids);
    int* s_islot = (int*)(smem + L.islot);
    uint16_t* s_cnt16 = (uint16_t*)(smem + L.cnt);
    int* s_cntw = (int*)(smem + L.cnt);
    u64* s_thr64 = (u64*)(smem + L.thr64);
    u32* s_thrhi = (u32*)(smem + L.thrhi);
    u64* s_sec = (u64*)(smem + L.sec);
    int* s_bcnt = (int*)(smem + L.bcnt);
    int* s_ovfcnt = (int*)(smem + L.ovfcnt);
    int* s_exact = (int*)(smem + L.exact);      // an exact local K-th threshold was computed
    u64* s_bstage = (u64*)(smem + L.bstage);
    u64* s_buf = (u64*)(smem + L.buf);
    u64* s_ovfk = (u64*)(smem + L.ovfk);
    uint16_t* s_ovfs = (uint16_t*)(smem + L.ovfs);
    PMisc* M = (PMisc*)(smem + L.misc);
    const int narr = L.narr;
    const int G = gridDim.x;
    const bool pass0 = FAST || A.pass0 != 0;
    const bool select = FAST || A.select != 0;
    const bool count_members = FAST || (pass0 && select);
    const bool cnt_thread = FAST || A.cnt_thread != 0;
    const bool write_qid = ROUTE && pass0 && A.qid_out != nullptr;
    const bool identity = A.ids_identity != 0;
    const int lutsz = USE_LUT ? A.lut_size : 0;
    const uint32_t gbase = A.gbase;
    const bool tma = FAST || A.tma != 0;
    const bool dyn = FAST || A.dyn != 0;

    // ---- tiles: full TMA tiles [0, full); the ragged tail (if any) is tile `full`
    const int64_t full = tma ? A.n / kTile : 0;
    const bool has_tail = tma && (A.n % kTile) != 0;
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
    // producer state (thread 0): next tile to issue
    // Tile order: contiguous range per CTA, or (dyn) round-robin strided tiles
    // blockIdx.x + i*G, so that all CTAs sweep the pool front to back together
    // (the oldest requests first: thresholds become global-quality early).
    long long next_tile = 0;
    bool prod_done = false;
    // issue the next tile into stage st, or mark the stage as end / tail
    auto produce = [&](int st) {
        if (prod_done) return;
        long long t;
        if (dyn) {
            t = next_tile;
            next_tile += G;
        } else {
            t = next_tile < t1 ? next_tile++ : LLONG_MAX;
        }
        M->tile[st] = t;
        if (t < full) {
            issue(t, st);
        } else {
            prod_done = true;
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[st])) : "memory");
        }
    };
    if (tma && tid == 0) {
        for (int s = 0; s < kStages; s++) mbar_init(&bars[s], 1);
        fence_mbar_init();
        next_tile = dyn ? (long long)blockIdx.x : t0;
        for (int s = 0; s < kStages; s++) produce(s);
    }

    // ---- policy tables -> smem (codes >= nslots see zero weights)
    for (int i = tid; i < kW4; i += kThreads) {
        const bool v = i < nslots;
        s_sid[i] = v ? P.sid[i] : -1;
        s_w4[i] = v ? make_float4(P.wb[i], P.wu[i], P.wf[i], 0.f) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (ROUTE && !USE_LUT && v) { s_min[i] = P.min_len[i]; s_max[i] = P.max_len[i]; }
    }
    if (!ROUTE)
        for (int i = tid; i < A.nids; i += kThreads) { s_ids[i] = A.sorted_ids[i]; s_islot[i] = A.sorted_slot[i]; }
    if (USE_LUT) {
        uint32_t* lw = (uint32_t*)lut;
        const int nw = (lutsz + 3) / 4;
        for (int i = tid; i < nw; i += kThreads) lw[i] = 0x01010101u * kCodeGap;
        __syncthreads();
        for (int q = 0; q < nslots; q++) {
            const int lo = P.min_len[q];
            const int hi = min(P.max_len[q], lutsz);
            for (int b = lo + tid; b < hi; b += kThreads) lut[b] = (unsigned char)q;
        }
        __syncthreads();
        if (tid == 0) lut[0] = (unsigned char)kCodeBad;   // b <= 0 reads lut[0]
    }
    if (count_members) {
        if (cnt_thread) {
            uint32_t* c32 = (uint32_t*)s_cnt16;
            for (int i = tid; i < kThreads * nslots / 2; i += kThreads) c32[i] = 0u;
        } else {
            for (int i = tid; i < kWarps * nslots; i += kThreads) s_cntw[i] = 0;
        }
    }
    for (int i = tid; i < ngs; i += kThreads) {
        s_thr64[i] = 0ull; s_thrhi[i] = 0u; s_sec[i] = 0ull; s_bcnt[i] = 0; s_ovfcnt[i] = 0; s_exact[i] = 0;
    }
    if (tid == 0) { M->novf = 0; M->want = 0; }
    __syncthreads();

    unsigned inv = 0, exc = 0, nins = 0, ngap = 0;
    long long processed = 0;          // requests seen by this thread (FAST: derives the invalid count)
    bool my_ovf = false;       // this thread overflowed a buffer (tile-local)
    bool my_want = false;      // this thread crossed a compaction trigger (tile-local)

    // rare path: a candidate passed the filter
    auto insert = [&](int gs, u64 key) {
        nins++;
        const int pos = atomicAdd(&s_bcnt[gs], 1);
        if (pos < cap) {
            s_buf[(size_t)gs * cap + pos] = key;
            if (pos == A.hwm || (pos == A.K && !s_exact[gs])) my_want = true;
        } else {
            const int o = atomicAdd(&M->novf, 1);
            EWSJF_CHECK(o < kTile);
            s_ovfk[o] = key;
            s_ovfs[o] = (uint16_t)gs;
            atomicAdd(&s_ovfcnt[gs], 1);
            my_ovf = true;
        }
    };

    // the 4 consecutive requests [idx0, idx0 + nv) of this thread
    auto process4 = [&](int64_t idx0, int nv, const int (&b)[4], const float (&ar)[4], const float (&co)[4],
                        const int (&qi)[4]) {
        int code[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int bj = b[j];
            int c;
            if (ROUTE) {
                if (USE_LUT) {
                    const int ix = bj < lutsz ? max(bj, 0) : 0;
                    c = lut[ix];
                    c = bj >= lutsz ? kCodeGap : c;
                } else {
                    int lo = 0, hi = nslots;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (s_min[mid] <= bj) lo = mid + 1; else hi = mid;
                    }
                    c = (lo > 0 && bj < s_max[lo - 1]) ? lo - 1 : kCodeGap;
                    c = bj >= 1 ? c : kCodeBad;
                }
            } else {
                int lo = 0, hi = A.nids;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (s_ids[mid] < qi[j]) lo = mid + 1; else hi = mid;
                }
                c = (lo < A.nids && s_ids[lo] == qi[j] && bj >= 1) ? s_islot[lo] : kCodeBad;
            }
            code[j] = j < nv ? c : kCodeNone;
        }
        processed += nv;
        if (write_qid) {
            int qo[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int c = code[j];
                qo[j] = c < kCodeGap ? (identity ? c : s_sid[c]) : c - 0x100;   // 0xFE -> -2, 0xFF -> -1
            }
            if (nv == 4 && tma) {
                __stcs((int4*)(A.qid_out + idx0), make_int4(qo[0], qo[1], qo[2], qo[3]));
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (j < nv) A.qid_out[idx0 + j] = qo[j];
            }
        }
        if (pass0) {
            unsigned gm = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (!FAST) inv += code[j] == kCodeBad;
                gm |= (unsigned)(code[j] == kCodeGap) << j;
            }
            if (ROUTE && __any_sync(0xffffffffu, gm != 0)) {   // rare: append gap requests
                ngap += __popc(gm);
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const bool g = (gm >> j) & 1u;
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
                                e.gid = gbase + (uint32_t)(idx0 + j);
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
        if (!select) return;
        // Phase 1 (independent across the 4 requests -> ILP): weights, score, validity
        float sp[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int c = code[j];
            const float4 w = s_w4[c & 0xFF];
            const bool ok0 = score_sp(b[j], ar[j], HAS_COST ? co[j] : 0.0f, HAS_COST, A.sp, w.x, w.y, w.z, &sp[j]);
            const bool valid = c < kCodeGap;
            ok[j] = valid && ok0;
            exc += (valid && !ok0) ? 1u : 0u;
        }
        // Phase 2: member counts
        if (count_members) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int c = code[j];
                if (cnt_thread) {
                    if (ok[j]) s_cnt16[c * kThreads + tid]++;
                } else {   // > 64 queues: warp match-any aggregation
                    const unsigned v = ok[j] ? (unsigned)c : 0xffffffffu;
                    const unsigned peers = __match_any_sync(0xffffffffu, v);
                    if (ok[j] && lane == __ffs(peers) - 1) s_cntw[warp * nslots + c] += __popc(peers);
                    __syncwarp();      // the next slot's leader may update the same counter
                }
            }
        }
        // Phase 3: filter tests on the key high words (no branches)
        u32 k1h[4], k2h[4], lo[4];
        unsigned pass1 = 0, pass2 = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int gs = code[j] - g_lo;
            const bool in = ok[j] && (FAST || (unsigned)gs < (unsigned)ngs);
            const int gsi = in ? gs : 0;
            lo[j] = ~(gbase + (uint32_t)(idx0 + j));
            const u32 fh = ~ord_f32(ar[j]);
            const u32 sh = __float_as_uint(sp[j]);
            k1h[j] = MODE == EWSJF_SELECT_SCORE ? sh : fh;
            k2h[j] = MODE == EWSJF_SELECT_SCORE ? fh : sh;
            const u32 th = s_thrhi[gsi];
            const u32 sc = (u32)(s_sec[gsi] >> 32);
            pass1 |= (unsigned)(in && k1h[j] >= th) << j;
            pass2 |= (unsigned)(in && k2h[j] >= sc) << j;
        }
        // Phase 4 (rare): exact 64-bit checks, inserts, secondary atomicMax
        if (pass1 | pass2) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int gs = code[j] - g_lo;
                if ((pass1 >> j) & 1u) {
                    const u64 k1 = ((u64)k1h[j] << 32) | lo[j];
                    if (k1 >= *(volatile u64*)&s_thr64[gs]) insert(gs, k1);
                }
                if ((pass2 >> j) & 1u) {
                    const u64 k2 = ((u64)k2h[j] << 32) | lo[j];
                    if (k2 > *(volatile u64*)&s_sec[gs]) atomicMax(&s_sec[gs], k2);
                }
            }
        }
    };

    // Warp-per-queue selection over a queue's buffer (+ its overflow-list keys):
    // returns t with K <= #(>= t) <= tgt (t = current threshold if already so).
    auto select_t = [&](int gs, int nb, int no, int no_all, int tgt) -> u64 {
        u64* bb = s_buf + (size_t)gs * cap;
        auto count_ge = [&](u64 t) -> int {
            int c = 0;
            for (int j = lane; j < nb; j += 32) c += bb[j] >= t;
            if (no)
                for (int j = lane; j < no_all; j += 32) c += (s_ovfs[j] == gs) && (s_ovfk[j] >= t);
            return __reduce_add_sync(0xffffffffu, c);
        };
        auto pick_in = [&](u64 lo, u64 hi, u64& p) -> bool {
            for (int j = lane; j < nb; j += 32) {
                const u64 v = bb[j];
                if (v > lo && v < hi) { p = v; return true; }
            }
            if (no)
                for (int j = lane; j < no_all; j += 32)
                    if (s_ovfs[j] == gs) {
                        const u64 v = s_ovfk[j];
                        if (v > lo && v < hi) { p = v; return true; }
                    }
            return false;
        };
        u64 t = s_thr64[gs];
        if (count_ge(t) > tgt) t = warp_select(t, A.K, tgt, count_ge, pick_in);
        return t;
    };
    // keep buffer keys >= t (in place, stable: writes never pass reads), append overflow keys >= t
    auto compact_to = [&](int gs, int nb, int no, int no_all, u64 t) -> int {
        u64* bb = s_buf + (size_t)gs * cap;
        int outc = 0;
        for (int j0 = 0; j0 < nb; j0 += 32) {
            const int j = j0 + lane;
            const u64 v = j < nb ? bb[j] : 0ull;
            const bool keep = j < nb && v >= t;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            __syncwarp();
            if (keep) bb[outc + __popc(m & ((1u << lane) - 1u))] = v;
            outc += __popc(m);
            __syncwarp();
        }
        if (no) {
            for (int j0 = 0; j0 < no_all; j0 += 32) {
                const int j = j0 + lane;
                const bool keep = j < no_all && s_ovfs[j] == gs && s_ovfk[j] >= t;
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (keep) bb[outc + __popc(m & ((1u << lane) - 1u))] = s_ovfk[j];
                outc += __popc(m);
            }
        }
        __syncwarp();
        return outc;
    };
    auto publish = [&](int gs, u64 t) {
        if (t > s_thr64[gs]) { s_thr64[gs] = t; s_thrhi[gs] = (u32)(t >> 32); }
        if (t) atomicMax(&A.gthr[g_lo + gs], t);
    };

    // Batched compaction, one warp per queue.  Two CTA barriers per event.
    unsigned ncomp = 0;
    auto compact_all = [&]() {
        const int no_all = M->novf;
        for (int gs = warp; gs < ngs; gs += kWarps) {
            const int nb = min(s_bcnt[gs], cap);
            const int no = s_ovfcnt[gs];
            const bool first = !s_exact[gs] && nb > A.K;   // establish an exact local threshold early
            if (no == 0 && nb < A.hwm && !first) continue;
            const u64 t = select_t(gs, nb, no, no_all, first && no == 0 ? A.K : A.tgt);
            const int outc = compact_to(gs, nb, no, no_all, t);
            ncomp++;
            if (lane == 0) { s_bcnt[gs] = outc; s_ovfcnt[gs] = 0; s_exact[gs] = 1; publish(gs, t); }
        }
        __syncthreads();
        if (tid == 0) M->novf = 0;
        my_ovf = false;
        my_want = false;
        __syncthreads();
    };

    // cross-CTA threshold refresh: loads issued at tile start, applied at tile end
    int rr = 0;
    u64 g_pre = 0;
    int g_gs = -1;
    auto gthr_prefetch = [&]() {
        g_gs = -1;
        if (select && warp == 0 && ngs > 0) {
            const int gs = lane + 32 * rr;
            if (gs < ngs) { g_gs = gs; g_pre = __ldcg(&A.gthr[g_lo + gs]); }
            rr = (32 * (rr + 1) >= ngs) ? 0 : rr + 1;
        }
    };
    auto gthr_apply = [&]() {
        if (g_gs >= 0 && g_pre > *(volatile u64*)&s_thr64[g_gs]) {
            *(volatile u64*)&s_thr64[g_gs] = g_pre;
            *(volatile u32*)&s_thrhi[g_gs] = (u32)(g_pre >> 32);
        }
    };
    auto direct_tile = [&](int64_t i_base) {   // one tile of direct (non-TMA) loads
        const int64_t i0 = i_base + 4 * tid;
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
        gthr_prefetch();
        process4(i0, nv, b4, a4, c4, q4);
        gthr_apply();
        if (__syncthreads_or(my_ovf || my_want)) compact_all();
    };

    // ---- cross-CTA threshold board (FAST only).  After its first tile a CTA
    // writes its per-queue top-m keys to board[q][cta][*]; the K-th largest
    // board key of a queue is a key of K distinct real requests, hence a valid
    // lower bound of the queue's global K-th key.  One warp per tile (rotating)
    // recomputes it for one queue from registers prefetched at tile start.
    const int bm = FAST ? A.board_m : 0;
    const int bn = bm * G;                       // board keys per queue (<= 320)
    auto board_write = [&]() {
        for (int gs = warp; gs < ngs; gs += kWarps) {
            const int nb = min(s_bcnt[gs], cap);
            u64 prev = ~0ull;
            for (int i = 0; i < bm; i++) {
                u64 mx = 0;
                for (int j = lane; j < nb; j += 32) {
                    const u64 v = s_buf[(size_t)gs * cap + j];
                    if (v < prev && v > mx) mx = v;
                }
                mx = warp_max_u64(mx);
                if (lane == 0) A.board[((size_t)(g_lo + gs) * G + blockIdx.x) * bm + i] = mx;
                prev = mx;
                if (!mx) break;
            }
        }
    };
    int b_slot = -1;
    int it_count = 0;
    auto board_prefetch = [&]() {   // cp.async the queue's board row into smem (no registers held)
        b_slot = -1;
        if (bm && it_count >= 2 && (it_count & 1) == 0 && warp == 1 + ((it_count >> 1) % (kWarps - 1))) {
            b_slot = (int)((blockIdx.x + (it_count >> 1)) % ngs);
            const u64* row = A.board + (size_t)(g_lo + b_slot) * G * bm;
            for (int j = lane; j < bn; j += 32)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s_bstage + j)), "l"(row + j)
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    };
    auto board_apply = [&]() {
        if (b_slot < 0) return;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        auto count_ge = [&](u64 t) -> int {
            int c = 0;
            for (int j = lane; j < bn; j += 32) { const u64 v = s_bstage[j]; c += (v != 0ull) && v >= t; }
            return __reduce_add_sync(0xffffffffu, c);
        };
        auto pick_in = [&](u64 lo, u64 hi, u64& p) -> bool {
            for (int j = lane; j < bn; j += 32) {
                const u64 v = s_bstage[j];
                if (v > lo && v < hi) { p = v; return true; }
            }
            return false;
        };
        const u64 t = warp_select(0ull, A.K, A.K, count_ge, pick_in);
        if (lane == 0 && t) {
            atomicMax(&A.gthr[g_lo + b_slot], t);
            if (t > *(volatile u64*)&s_thr64[b_slot]) {
                *(volatile u64*)&s_thr64[b_slot] = t;
                *(volatile u32*)&s_thrhi[b_slot] = (u32)(t >> 32);
            }
        }
    };

    if (tma) {
        int st = 0;
        uint32_t par = 0;
        for (;;) {
            gthr_prefetch();
            board_prefetch();
            mbar_wait(&bars[st], par);
            const long long t = M->tile[st];
            if (t >= full) {                      // end of this CTA's work (maybe the tail first)
                if (t == full && has_tail) {
                    g_gs = -1;
                    direct_tile(full * kTile);
                }
                break;
            }
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
            gthr_apply();
            board_apply();
            const int any = __syncthreads_or(my_ovf || my_want);
            if (tid == 0) {
                fence_proxy_async();
                produce(st);
            }
            if (any) compact_all();
            if (bm && it_count == 0) {   // once: publish the first tile's top-m keys
                board_write();
                __syncthreads();
            }
            it_count++;
            if (++st == kStages) { st = 0; par ^= 1u; }
        }
        // static scheduling: the last CTA also owns the tail
        if (!dyn && has_tail && blockIdx.x == G - 1) direct_tile(full * kTile);
    } else {   // direct-load path over the whole pool, static tiles
        const int64_t ntl = (A.n + kTile - 1) / kTile;
        const int64_t d0 = ntl * blockIdx.x / G, d1 = ntl * (blockIdx.x + 1) / G;
        for (int64_t t = d0; t < d1; ++t) direct_tile(t * kTile);
    }
    __syncthreads();

    // ---- final trim: every queue keeps at most its exact local top-K, whose K-th
    // key is published (a valid lower bound of the global K-th key)
    if (select) {
        for (int gs = warp; gs < ngs; gs += kWarps) {
            const int nb = min(s_bcnt[gs], cap);
            if (nb <= A.K) continue;
            const u64 t = select_t(gs, nb, 0, 0, A.K);
            const int outc = compact_to(gs, nb, 0, 0, t);
            if (lane == 0) { s_bcnt[gs] = outc; publish(gs, t); }
        }
        __syncthreads();
    }

    // ---- rows out: keys >= max(local, global) threshold, secondary, members
    const Rows& R = A.rows;
    long long counted = 0;
    for (int gs = warp; gs < ngs; gs += kWarps) {
        const int slot = g_lo + gs;
        const int nb = min(s_bcnt[gs], cap);
        u64 tf = s_thr64[gs];
        const u64 gg = __ldcg(&A.gthr[slot]);
        tf = gg > tf ? gg : tf;
        u64* dst = R.keys + ((size_t)slot * G + blockIdx.x) * R.cap;
        int outc = 0;
        for (int j0 = 0; j0 < nb; j0 += 32) {
            const int j = j0 + lane;
            const u64 v = j < nb ? s_buf[(size_t)gs * cap + j] : 0ull;
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
    if (count_members) {
        for (int s = warp; s < nslots; s += kWarps) {
            long long m = 0;
            if (cnt_thread) {
                const uint32_t* c32 = (const uint32_t*)(s_cnt16 + (size_t)s * kThreads);
                for (int i = lane; i < kThreads / 2; i += 32) { const uint32_t v = c32[i]; m += (v & 0xffffu) + (v >> 16); }
            } else {
                for (int w = lane; w < kWarps; w += 32) m += s_cntw[w * nslots + s];
            }
            for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
            if (lane == 0) R.members[(size_t)s * G + blockIdx.x] = m;
            counted += m;   // lane 0 of each warp holds its queues' totals
        }
    }
    // FAST: invalid = processed - counted - excluded - gap (per warp, lane-summed below)
    long long invl = FAST ? processed - (long long)exc - (long long)ngap : (long long)inv;
    for (int o = 16; o; o >>= 1) {
        invl += __shfl_xor_sync(0xffffffffu, invl, o);
        exc += __shfl_xor_sync(0xffffffffu, exc, o);
        nins += __shfl_xor_sync(0xffffffffu, nins, o);
    }
    if (lane == 0) {
        if (FAST) invl -= counted;
        if (pass0 && invl) atomicAdd(&A.ctr->n_invalid, (unsigned long long)invl);
        if (pass0 && exc) atomicAdd(&A.ctr->n_excluded, (unsigned long long)exc);
        if (nins) atomicAdd(&A.ctr->dbg_inserted, (unsigned long long)nins);
        if (ncomp) atomicAdd(&A.ctr->dbg_compactions, (unsigned long long)ncomp);
    }
}

// ---------------------------------------------------------------- kernels --
template <int MODE, bool ROUTE, bool HAS_COST, bool USE_LUT>
__global__ void __launch_bounds__(kThreads, 1)
    partial_kernel(const __grid_constant__ PartialArgs A, const __grid_constant__ Policy P) {
    extern __shared__ __align__(128) unsigned char smem[];
    partial_phase<MODE, ROUTE, HAS_COST, USE_LUT, false>(A, P, smem);
}

// Grid-wide barrier of a cooperative launch (every CTA co-resident).
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v < target) __nanosleep(64);
        } while (v < target);
    }
    __syncthreads();
}

// Fused single-pass tick: partial phase -> grid barrier -> merge phase.
template <int MODE, bool ROUTE, bool HAS_COST, bool USE_LUT, bool FAST>
__global__ void __launch_bounds__(kThreads, 1)
    tick_kernel(const __grid_constant__ PartialArgs A, const __grid_constant__ Policy P,
                const __grid_constant__ MergeArgs MA) {
    extern __shared__ __align__(128) unsigned char smem[];
    partial_phase<MODE, ROUTE, HAS_COST, USE_LUT, FAST>(A, P, smem);
    grid_barrier(&A.ctr->barrier, gridDim.x);
    if (FAST && A.board_m) {   // nobody reads the board any more: clear this CTA's rows
        for (int i = threadIdx.x; i < P.nslots * A.board_m; i += kThreads) {
            const int s = i / A.board_m, j = i % A.board_m;
            A.board[((size_t)s * gridDim.x + blockIdx.x) * A.board_m + j] = 0ull;
        }
    }
    merge_phase<MERGE_IN_ROWS, MERGE_OUT_FINAL, HAS_COST>(MA, P, smem);
}

// ---------------------------------------------------------------- launch ---
int64_t merge_smem_total(int in_mode);

template <int MO, bool R, bool C, bool U>
static cudaError_t launch_t(const PartialArgs& A, const Policy& P, const MergeArgs* MA, int grid, cudaStream_t st) {
    const PartialSmem L = partial_layout(R, C, A.tma, U ? A.lut_size : 0, P.nslots, A.nids, A.pass0, A.cnt_thread,
                                         A.g_hi - A.g_lo, A.cap);
    if (!MA) {
        auto k = partial_kernel<MO, R, C, U>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
        if (e != cudaSuccess) return e;
        k<<<grid, kThreads, L.total, st>>>(A, P);
        return cudaGetLastError();
    }
    const int64_t smem = L.total > merge_smem_total(MERGE_IN_ROWS) ? L.total : merge_smem_total(MERGE_IN_ROWS);
    const bool fast = A.tma && A.cnt_thread && A.pass0 && A.select && A.g_lo == 0 && A.g_hi == P.nslots &&
                      !getenv("EWSJF_NO_FAST");
    auto k = fast ? tick_kernel<MO, R, C, U, true> : tick_kernel<MO, R, C, U, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void* args[] = {(void*)&A, (void*)&P, (void*)MA};
    return cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kThreads), args, (size_t)smem, st);
}

template <int MO>
static cudaError_t launch_m(const PartialArgs& A, const Policy& P, const MergeArgs* MA, bool route, bool has_cost,
                            bool use_lut, int grid, cudaStream_t st) {
    if (route) {
        if (has_cost) return use_lut ? launch_t<MO, true, true, true>(A, P, MA, grid, st)
                                     : launch_t<MO, true, true, false>(A, P, MA, grid, st);
        return use_lut ? launch_t<MO, true, false, true>(A, P, MA, grid, st)
                       : launch_t<MO, true, false, false>(A, P, MA, grid, st);
    }
    return has_cost ? launch_t<MO, false, true, false>(A, P, MA, grid, st)
                    : launch_t<MO, false, false, false>(A, P, MA, grid, st);
}

// MA == nullptr: partial pass only; otherwise the fused cooperative tick kernel.
cudaError_t launch_partial(const PartialArgs& A, const Policy& P, const MergeArgs* MA, bool route, bool has_cost,
                           bool use_lut, int grid, cudaStream_t st) {
    if (A.sp.mode == EWSJF_SELECT_FIFO)
        return launch_m<EWSJF_SELECT_FIFO>(A, P, MA, route, has_cost, use_lut, grid, st);
    return launch_m<EWSJF_SELECT_SCORE>(A, P, MA, route, has_cost, use_lut, grid, st);
}

int64_t partial_smem_bytes(bool route, bool has_cost, bool tma, int lut_size, int nslots, int nids, int pass0,
                           int cnt_thread, int ngs, int cap) {
    return partial_layout(route, has_cost, tma, lut_size, nslots, nids, pass0, cnt_thread, ngs, cap).total;
}

}  // namespace ewsjf
