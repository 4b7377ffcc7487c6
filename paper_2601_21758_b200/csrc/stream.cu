// stream.cu — the streaming pass of the EWSJF tick on sm_100a (route A8 +
// Eq. 4 score A10 + per-queue filter A11) and its fusion with the per-queue
// merge (merge.cuh) behind one grid barrier.
//
// (The round-1 tick, kept behind EWSJF_NO_FTICK / EWSJF_OLD_TICK; the default tick
// is ftick.cu.)  Every warp owns a private ring of A.stages stages (128 requests x
// {len, arrival, cost} per stage), filled by per-lane 16-byte cp.async copies
// (LDGSTS; a ring of 1-D TMA bulk copies per warp behind EWSJF_TMA_RING measured
// slower: ~90 cycles per 512-byte bulk copy), and walks its own warp tiles.  Per request the common path is: byte-LUT
// route, qid store, weights (float4) + Eq. 4 (one MUFU.LG2, one MUFU.RCP), a
// per-thread u16 member counter and two 32-bit threshold compares.
//
// The rare requests that beat their queue's threshold reserve a slot in the
// queue's shared candidate buffer with one warp-aggregated atomicAdd per
// distinct queue (no locks); past the buffer they spill into a CTA overflow
// list.  When a buffer crosses its high-water mark the CTA meets in a
// collective (named barrier, entered by each warp after its current tile, so
// it happens a few times per launch, not per tile): one warp per queue cuts
// buffer + overflow to the exact K-th key (warp quickselect), which raises the
// queue's filter threshold and is published to the other CTAs (atomicMax on
// gthr) together with the queue's top keys on a cross-CTA board; a few times
// per launch each warp turns the board into a valid global threshold (the
// K-th largest of distinct real keys).
//
// Paper: route = Dispatcher, score = Eq. 4, selection =
// Alg. 1's per-queue scores + ArgMax; readings R1-R27.
#include <climits>
#include <cstdlib>
#include "merge.cuh"
#include "select.cuh"

namespace ewsjf {

constexpr int kSThreads = 512;
constexpr int kSWarps = kSThreads / 32;
constexpr int kWT = 128;          // requests per warp tile (4 per lane)
constexpr int kSStagesMax = 8;    // TMA ring depth per warp: runtime A.stages (<= 8)
constexpr int kSTab = 256;        // per-code tables (codes 0..255 index them unmasked)
constexpr int kOvfCap = kSWarps * kWT;   // overflow bound: one tile per warp after a flag
constexpr int kBoardRegs = 10;    // board keys per lane in the board selection (G*m <= 320)
constexpr int kSCodeGap = 0xFE;
constexpr int kSCodeBad = 0xFF;

__host__ __device__ inline int64_t sal16(int64_t x) { return (x + 15) & ~(int64_t)15; }

struct SMisc {
    int flag;       // some buffer crossed its high-water mark: collective wanted
    int novf;       // overflow list fill
    int ndone;      // warps done streaming
    int pad;
};

struct StreamSmem {
    int64_t ring, bars, w4, thr64, sec, thrhi, sechi, thrf, secf, sid, bcnt, misc, cnt, buf, ovfk, ovfq, lut, total;
    int narr;
};
__host__ __device__ inline StreamSmem stream_layout(bool has_cost, int lut_size, int nslots, int cap, int stages) {
    StreamSmem L;
    L.narr = has_cost ? 3 : 2;
    int64_t o = 0;
    L.ring = o;  o += (int64_t)kSWarps * stages * L.narr * kWT * 4;
    L.bars = o;  o = sal16(o + 8LL * kSWarps * stages);
    L.w4 = o;    o = sal16(o + 32LL * kSTab);    // per-code record {wb, wu, wf, thrf, secf, qid, -, -}
    L.thr64 = o; o = sal16(o + 8LL * kSTab);
    L.sec = o;   o = sal16(o + 8LL * kSTab);
    L.thrhi = o; o = sal16(o + 4LL * kSTab);
    L.sechi = o; o = sal16(o + 4LL * kSTab);
    L.thrf = o;  o = sal16(o + 4LL * kSTab);
    L.secf = o;  o = sal16(o + 4LL * kSTab);
    L.sid = o;   o = sal16(o + 20LL * kSTab);   // sid, round-1 counts, offsets, CTA bounds
    L.bcnt = o;  o = sal16(o + 4LL * kSTab);
    L.misc = o;  o = sal16(o + sizeof(SMisc));
    L.cnt = o;   o = sal16(o + 2LL * kSThreads * (nslots + 2));   // + rows: excluded, other
    L.buf = o;   o = sal16(o + (8LL * nslots * cap > (int64_t)sizeof(Policy) ? 8LL * nslots * cap : (int64_t)sizeof(Policy)));
    L.ovfk = o;  o = sal16(o + 8LL * kOvfCap);
    L.ovfq = o;  o = sal16(o + kOvfCap);
    L.lut = o;   o = sal16(o + lut_size + 1);                      // lut[lut_size] = gap
    L.total = o;
    return L;
}

int64_t stream_smem_bytes(bool has_cost, int lut_size, int nslots, int cap, int stages) {
    return stream_layout(has_cost, lut_size, nslots, cap, stages).total;
}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// phase timestamps (EWSJF_PHASES diagnostics): slot s of this CTA's row
__device__ __forceinline__ void dbg_max(const PartialArgs& A, int s, unsigned long long v) {
    if (A.dbg) atomicMax(&A.dbg[blockIdx.x * kDbgStride + s], v);
}

// cp.async (LDGSTS) of 16 bytes global -> shared, L2 only; groups per thread.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most n of this thread's groups are pending (n = ring depth - 1)
__device__ __forceinline__ void cp_async_wait(int n) {
    switch (n) {
        case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
        case 6: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
    }
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Warp sort of one u64 per lane, descending (lane 0 = largest); bitonic network.
__device__ __forceinline__ u64 warp_sort_desc(u64 v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const u64 o = shfl_xor_u64(v, j);
            const bool first = (lane & j) == 0;          // lower lane of the pair
            const bool desc = (lane & k) == 0;           // block direction (last stage: all descending)
            v = (first == desc) ? (o > v ? o : v) : (o < v ? o : v);
        }
    }
    return v;
}

// Warp selection over a set of unique nonzero keys given by for_each(f)
// (f(key) for every key, lane-strided).  Returns t with K <= #(>= t) <= tgt
// (tgt == K: t is the exact K-th largest key).  Requires #keys >= K.
// Each round draws one min-hash sample per lane among the keys strictly
// inside the current bracket (lo, hi) (an unbiased sample whatever the key
// order), sorts the 32 samples and takes the one whose rank estimates the
// target count; the bracket shrinks strictly every round.
template <typename ForEach>
__device__ __forceinline__ u64 warp_select(ForEach for_each, int K, int tgt) {
    const int lane = threadIdx.x & 31;
    u64 lo = 0ull, hi = ~0ull;   // invariant: #(>= lo) >= K, #(>= hi) < K
    int c_hi = 0;                // #(>= hi)
    for (unsigned it = 0;; it++) {
        int m = 0;
        u64 s = 0ull;
        u32 best = 0u;
        const u32 salt = 0x9E3779B9u * (it + 1u);
        for_each([&](u64 v) {
            if (v > lo && v < hi) {
                m++;
                const u32 h = ((u32)v ^ salt) * 0x85EBCA77u ^ (u32)(v >> 32) * 0xC2B2AE3Du;
                if (h >= best) { best = h; s = v; }
            }
        });
        m = __reduce_add_sync(0xffffffffu, m);
        if (m == 0) break;               // lo is a key with #(>= lo) == K (or the only bound left)
        const int ns = __popc(__ballot_sync(0xffffffffu, s != 0ull));
        s = warp_sort_desc(s);
        // sample rank r (0 = largest) estimates #(>= s_r) ~ c_hi + (r + 1) m / ns
        const int want = (K + tgt) / 2 - c_hi;
        int r = (int)ceilf((float)want * (float)ns / (float)m) - 1;
        r = r < 0 ? 0 : (r >= ns ? ns - 1 : r);
        const u64 piv = ((u64)__shfl_sync(0xffffffffu, (u32)(s >> 32), r) << 32) |
                        (u64)__shfl_sync(0xffffffffu, (u32)s, r);
        int c = 0;
        for_each([&](u64 v) { c += v >= piv; });
        c = __reduce_add_sync(0xffffffffu, c);
        if (c >= K) {
            lo = piv;
            if (c <= tgt) break;
        } else {
            hi = piv;
            c_hi = c;
        }
    }
    return lo;
}

// warp_select over a contiguous array a[0..n): samples are drawn by random
// index (4 probes per lane, the first inside the bracket wins); when fewer than
// 8 lanes find one, the round falls back to the min-hash scan.  One count scan
// per round.  Same contract as warp_select.
__device__ __forceinline__ u64 warp_select_arr(const u64* a, int n, int K, int tgt) {
    const int lane = threadIdx.x & 31;
    u64 lo = 0ull, hi = ~0ull;
    int c_hi = 0, m = n;         // m ~ #keys strictly inside (lo, hi)
    for (unsigned it = 0;; it++) {
        u64 s = 0ull;
        u32 h = (lane * 0x9E3779B9u) ^ (it * 0x85EBCA77u) ^ 0x27D4EB2Fu;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            h = h * 1664525u + 1013904223u;
            const u64 v = a[(int)(((unsigned long long)(h >> 8) * (unsigned)n) >> 24)];
            if (s == 0ull && v > lo && v < hi) s = v;
        }
        int ns = __popc(__ballot_sync(0xffffffffu, s != 0ull));
        if (ns < 8) {                  // sparse bracket: min-hash sample over a scan
            int mm = 0;
            u32 best = 0u;
            s = 0ull;
            const u32 salt = 0x9E3779B9u * (it + 1u);
            for (int j = lane; j < n; j += 32) {
                const u64 v = a[j];
                if (v > lo && v < hi) {
                    mm++;
                    const u32 hh = ((u32)v ^ salt) * 0x85EBCA77u ^ (u32)(v >> 32) * 0xC2B2AE3Du;
                    if (hh >= best) { best = hh; s = v; }
                }
            }
            m = __reduce_add_sync(0xffffffffu, mm);
            if (m == 0) break;
            ns = __popc(__ballot_sync(0xffffffffu, s != 0ull));
        }
        s = warp_sort_desc(s);
        const int want = (K + tgt) / 2 - c_hi;
        int r = (int)ceilf((float)want * (float)ns / (float)max(m, 1)) - 1;
        r = r < 0 ? 0 : (r >= ns ? ns - 1 : r);
        const u64 piv = ((u64)__shfl_sync(0xffffffffu, (u32)(s >> 32), r) << 32) |
                        (u64)__shfl_sync(0xffffffffu, (u32)s, r);
        int c = 0;
        for (int j = lane; j < n; j += 32) c += a[j] >= piv;
        c = __reduce_add_sync(0xffffffffu, c);
        if (c >= K) {
            m = c - c_hi - 1;          // keys strictly inside (piv, hi)... approx. for the next estimate
            lo = piv;
            if (c <= tgt) break;
        } else {
            m = m - (c - c_hi);
            hi = piv;
            c_hi = c;
        }
        if (m < 1) m = 1;
    }
    return lo;
}

template <int MODE, bool HAS_COST>
__device__ __forceinline__ void stream_phase(const PartialArgs& A, const Policy& P, unsigned char* smem) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nslots = P.nslots;
    const int cap = A.cap, K = A.K, hwm = A.hwm;
    const int lutsz = A.lut_size;
    const int S = A.stages;
    const StreamSmem L = stream_layout(HAS_COST, lutsz, nslots, cap, S);
    constexpr int narr = HAS_COST ? 3 : 2;
    unsigned char* lut = smem + L.lut;
    uint16_t* s_cnt16 = (uint16_t*)(smem + L.cnt);
    int* s_sid = (int*)(smem + L.sid);
    // per-code record read with two 16-byte loads on the common path:
    // .x/.y/.z = w_base, w_urg, w_fair·ln2; .w = fast filter; [+1].x = fast secondary, [+1].y = qid bits
    float4* s_rec = (float4*)(smem + L.w4);
    u64* s_thr64 = (u64*)(smem + L.thr64);
    u32* s_thrhi = (u32*)(smem + L.thrhi);
    u64* s_sec = (u64*)(smem + L.sec);
    u32* s_sechi = (u32*)(smem + L.sechi);
    // fast filter (SCORE s' >= thrf, FIFO arrival <= thrf) and secondary (SCORE arrival <= secf,
    // FIFO s' >= secf) live in the per-code record
    auto thrf_at = [&](int q) -> float* { return (float*)(s_rec + 2 * q) + 3; };
    auto secf_at = [&](int q) -> float* { return (float*)(s_rec + 2 * q + 1); };
    int* s_bcnt = (int*)(smem + L.bcnt);
    u64* s_buf = (u64*)(smem + L.buf);
    u64* s_ovfk = (u64*)(smem + L.ovfk);
    unsigned char* s_ovfq = smem + L.ovfq;
    SMisc* M = (SMisc*)(smem + L.misc);
    uint64_t* bars = (uint64_t*)(smem + L.bars) + warp * S;
    unsigned char* ring = smem + L.ring + (int64_t)warp * S * narr * kWT * 4;
    const uint32_t gbase = A.gbase;
    const bool identity = A.ids_identity != 0;
    const bool write_qid = A.qid_out != nullptr;
    const int G = gridDim.x;
    const int bm = A.board_m;            // board keys per (queue, CTA); 0 = off

    // ---- warp tiles: tile t covers requests [t*kWT, (t+1)*kWT); warp gw of the
    // grid takes tiles gw, gw + GW, ...: all warps sweep the pool front to back
    // together (the oldest requests first, so thresholds settle early).
    const int64_t nfull = A.n / kWT;
    const int64_t GW = (int64_t)G * kSWarps;
    const int64_t gw = (int64_t)blockIdx.x * kSWarps + warp;
    auto stage = [&](int st, int a) -> unsigned char* { return ring + (st * narr + a) * kWT * 4; };
    // per-lane ring (A.tma == 0): every lane copies and later reads back its own
    // 16 bytes per array with cp.async; one commit group per tile (empty past the end)
    const bool lane_ring = A.tma == 0;
    auto issue_lane = [&](int64_t t, int st) {
        if (t < nfull) {
            const int64_t off = t * kWT + 4 * lane;
            cp_async16(stage(st, 0) + 16 * lane, A.len + off);
            cp_async16(stage(st, 1) + 16 * lane, A.arrival + off);
            if (HAS_COST) cp_async16(stage(st, 2) + 16 * lane, A.cost + off);
        }
        cp_async_commit();
    };
    auto issue = [&](int64_t t, int st) {   // lane 0
        mbar_arrive_expect_tx(&bars[st], (uint32_t)(narr * kWT * 4));
        const int64_t off = t * kWT;
        tma_load_1d(stage(st, 0), A.len + off, kWT * 4, &bars[st]);
        tma_load_1d(stage(st, 1), A.arrival + off, kWT * 4, &bars[st]);
        if (HAS_COST) tma_load_1d(stage(st, 2), A.cost + off, kWT * 4, &bars[st]);
    };
    if (tid == 0 && A.dbg) { for (int s = 0; s < kDbgStride; s++) A.dbg[blockIdx.x * kDbgStride + s] = 0ull; dbg_max(A, 0, gtime()); }
    if (lane_ring) {
        if (A.pass0 != 4)
            for (int s = 0; s < S; s++) issue_lane(gw + s * GW, s);
    } else if (lane == 0) {
        for (int s = 0; s < S; s++) mbar_init(&bars[s], 1);
        fence_mbar_init();
        for (int s = 0; s < S; s++) {
            const int64_t t = gw + s * GW;
            if (t < nfull) issue(t, s);
        }
    }

    // ---- policy tables -> smem while the first tiles are in flight.  Only the
    // fields the stream reads are loaded from the Policy parameter (one code per
    // thread); the whole Policy is staged in shared memory only when the LUT has
    // to be built here (no prebuilt LUT).
    const Policy* Ps = (const Policy*)s_buf;
    {
        if (!A.lut_dev) {
            const int n16 = (int)((sizeof(Policy) + 15) / 16);
            const int4* src = reinterpret_cast<const int4*>(&P);
            for (int i = tid; i < n16; i += kSThreads) ((int4*)s_buf)[i] = src[i];
        }
        uint32_t* c32 = (uint32_t*)s_cnt16;
        for (int i = tid; i < kSThreads * (nslots + 2) / 2; i += kSThreads) c32[i] = 0u;
    }
    if (tid == 0) { M->flag = 0; M->novf = 0; M->ndone = 0; }
    for (int i = tid; i < kSTab; i += kSThreads) {
        const bool v = i < nslots;
        const float inf0 = __int_as_float(0x7f800000);
        const int sid = v ? P.sid[i] : (i == kSCodeGap ? -2 : -1);   // qid table: gap -> -2, bad/none -> -1
        // codes >= nslots never pass the filters
        s_rec[2 * i] = make_float4(v ? P.wb[i] : 0.f, v ? P.wu[i] : 0.f, v ? P.wf[i] : 0.f,
                                   MODE == EWSJF_SELECT_SCORE ? (v ? 0.f : inf0) : (v ? inf0 : -inf0));
        s_rec[2 * i + 1] = make_float4(MODE == EWSJF_SELECT_SCORE ? (v ? inf0 : -inf0) : (v ? 0.f : inf0),
                                       __int_as_float(sid), 0.f, 0.f);
        s_thr64[i] = 0ull; s_thrhi[i] = 0u; s_sec[i] = 0ull; s_sechi[i] = 0u; s_bcnt[i] = 0;
        s_sid[i] = sid;
    }
    __syncthreads();
    if (tid == 0) dbg_max(A, 12, A.dbg ? gtime() : 0ull);
    if (A.lut_dev) {
        // the prebuilt LUT (ctx cache, 16-byte padded): four 16-byte loads per thread
        const int n16 = (lutsz + 1 + 15) / 16;
        const int4* src = reinterpret_cast<const int4*>(A.lut_dev);
        for (int i = tid; i < n16; i += kSThreads) ((int4*)lut)[i] = __ldg(src + i);
    } else {
        // byte LUT length -> queue position, built a word (4 lengths) at a time:
        // each thread walks a contiguous run of words through the sorted,
        // disjoint [min_len, max_len) intervals.
        const int nw = (lutsz + 1 + 3) / 4;   // lut[0..lutsz], lut[lutsz] = gap
        const int wpt = (nw + kSThreads - 1) / kSThreads;
        const int w0 = tid * wpt, w1 = min(nw, w0 + wpt);
        if (w0 < w1) {
            int qi = 0, hi = nslots;                 // first queue with max_len > 4*w0
            while (qi < hi) {
                const int mid = (qi + hi) >> 1;
                if (Ps->max_len[mid] <= 4 * w0) qi = mid + 1; else hi = mid;
            }
            int qmin = qi < nslots ? Ps->min_len[qi] : INT_MAX, qmax = qi < nslots ? Ps->max_len[qi] : INT_MAX;
            uint32_t* lw = (uint32_t*)lut;
            for (int w = w0; w < w1; w++) {
                const int L0 = 4 * w;
                while (L0 >= qmax) {
                    qi++;
                    qmin = qi < nslots ? Ps->min_len[qi] : INT_MAX;
                    qmax = qi < nslots ? Ps->max_len[qi] : INT_MAX;
                }
                if (L0 > 0 && L0 >= qmin && L0 + 3 < qmax && L0 + 3 < lutsz) {   // the common case
                    lw[w] = 0x01010101u * (uint32_t)qi;
                    continue;
                }
                uint32_t word = 0;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const int Lk = 4 * w + k;
                    while (Lk >= qmax) {
                        qi++;
                        qmin = qi < nslots ? Ps->min_len[qi] : INT_MAX;
                        qmax = qi < nslots ? Ps->max_len[qi] : INT_MAX;
                    }
                    const uint32_t code = Lk == 0 ? (uint32_t)kSCodeBad
                                                  : (Lk >= qmin && Lk < lutsz ? (uint32_t)qi : (uint32_t)kSCodeGap);
                    word |= code << (8 * k);
                }
                lw[w] = word;
            }
        }
    }

    if (tid == 0) dbg_max(A, 13, A.dbg ? gtime() : 0ull);
    __syncthreads();
    if (tid == 0) dbg_max(A, 1, gtime());

    unsigned exc = 0, nins = 0, ngap = 0, ncomp = 0, ndrop = 0, excl_total = 0;
    long long cyc_wait = 0, cyc_proc = 0, cyc_loop0 = 0, cyc_ref = 0, cyc_board = 0, cyc_flag = 0, cyc_tile = 0;   // EWSJF_PHASES cycle accounting
    long long processed = 0;

    // key high word -> the fast-test float (SCORE: s'; FIFO: the arrival a with ~ord(a) == hi)
    auto hi_to_f = [](u32 hi) -> float {
        if (MODE == EWSJF_SELECT_SCORE) return __uint_as_float(hi);
        const u32 u = ~hi;
        return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
    };
    auto raise_thr = [&](int q, u64 t) {   // one lane
        if (t > *(volatile u64*)&s_thr64[q]) {
            atomicMax(&s_thr64[q], t);
            const u32 old = atomicMax(&s_thrhi[q], (u32)(t >> 32));
            const u32 hi = old > (u32)(t >> 32) ? old : (u32)(t >> 32);
            *(volatile float*)thrf_at(q) = hi_to_f(hi);
        }
    };

    // ---- collective: cut every queue holding more than K candidates to its
    // exact K-th key (buffer + overflow), publish thresholds and board rows.
    auto collective = [&]() {
        const unsigned long long tc0 = A.dbg ? gtime() : 0ull;
        named_sync(1, kSThreads);            // every warp finished its tile: no insert in flight
        const int no_all = min(*(volatile int*)&M->novf, kOvfCap);
        for (int q = warp; q < nslots; q += kSWarps) {
            u64* bb = s_buf + (size_t)q * cap;
            int nb = min(s_bcnt[q], cap);
            int no = 0;
            for (int j = lane; j < no_all; j += 32) no += s_ovfq[j] == q;
            no = __reduce_add_sync(0xffffffffu, no);
            u64 t = 0ull;
            auto keep_buf = [&](u64 th) {    // keep buffer keys >= th (stable, in place)
                int outc = 0;
                for (int j0 = 0; j0 < nb; j0 += 32) {
                    const int j = j0 + lane;
                    const u64 v = j < nb ? bb[j] : 0ull;
                    const bool keep = j < nb && v >= th;
                    const unsigned m = __ballot_sync(0xffffffffu, keep);
                    __syncwarp();
                    if (keep) bb[outc + __popc(m & ((1u << lane) - 1u))] = v;
                    outc += __popc(m);
                    __syncwarp();
                }
                nb = outc;
            };
            if (nb + no > cap) {             // window over buffer + overflow: <= cap-64 survive
                t = warp_select(
                    [&](auto f) {
                        for (int j = lane; j < nb; j += 32) f(bb[j]);
                        for (int j = lane; j < no_all; j += 32)
                            if (s_ovfq[j] == q) f(s_ovfk[j]);
                    },
                    K, cap - 64);
                keep_buf(t);
            }
            if (no) {                        // append overflow keys >= t
                for (int j0 = 0; j0 < no_all; j0 += 32) {
                    const int j = j0 + lane;
                    const bool keep = j < no_all && s_ovfq[j] == q && s_ovfk[j] >= t;
                    const unsigned m = __ballot_sync(0xffffffffu, keep);
                    if (keep) bb[nb + __popc(m & ((1u << lane) - 1u))] = s_ovfk[j];
                    nb += __popc(m);
                }
                __syncwarp();
            }
            if (nb > K) {                    // exact K-th of the (<= cap) candidates
                t = warp_kth_arr(bb, nb, K, kApproxBit, cap - 64);
                keep_buf(t);
                ncomp++;
            }
            __syncwarp();
            if (lane == 0) {
                s_bcnt[q] = nb;
                if (t) { raise_thr(q, t); atomicMax(&A.gthr[q], t); }
            }
            if (bm) {                        // board row: this CTA's top-bm keys of q
                u64 prev = ~0ull;
                for (int i = 0; i < bm; i++) {
                    u64 mx = 0;
                    for (int j = lane; j < nb; j += 32) {
                        const u64 v = bb[j];
                        if (v < prev && v > mx) mx = v;
                    }
                    mx = warp_max_u64(mx);
                    if (lane == 0) A.board[((size_t)q * G + blockIdx.x) * bm + i] = mx;
                    prev = mx;
                }
            }
        }
        named_sync(1, kSThreads);
        if (tid == 0) { M->novf = 0; M->flag = 0; }
        named_sync(1, kSThreads);
        if (A.dbg && tid == 0) {
            atomicAdd(&A.dbg[blockIdx.x * kDbgStride + 5], 1ull);
            atomicAdd(&A.dbg[blockIdx.x * kDbgStride + 6], gtime() - tc0);
        }
    };

    // ---- board -> global threshold of queue q (one warp): the K-th largest of
    // the published keys (distinct real requests of distinct CTAs) bounds the
    // global K-th from below.
    auto board_refresh = [&](int q) {
        const int nbk = G * bm;
        const u64* row = A.board + (size_t)q * G * bm;
        u64 v[kBoardRegs];
        int nz = 0;
#pragma unroll
        for (int r = 0; r < kBoardRegs; r++) {
            const int j = lane + 32 * r;
            v[r] = j < nbk ? __ldcg(row + j) : 0ull;
            nz += v[r] != 0ull;
        }
        nz = __reduce_add_sync(0xffffffffu, nz);
        if (nz < K) return;
        const u64 t = warp_kth_regs<kBoardRegs>(v, K, kApproxBit, 1 << 30);
        if (lane == 0 && t) { raise_thr(q, t); atomicMax(&A.gthr[q], t); }
    };

    // ---- the 4 consecutive requests [idx0, idx0 + nv) of this lane
    // r1k != nullptr (round 1): no filter; the lane's scored keys go to r1k/r1q
    auto process4 = [&](int64_t idx0, int nv, const int (&b)[4], const float (&ar)[4], const float (&co)[4],
                        u64* r1k, int* r1q) {
        int code[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int c = lut[min(max(b[j], 0), lutsz)];   // lut[0]: bad; lut[lutsz]: gap
            code[j] = j < nv ? c : 0x1FF;
        }
        processed += nv;
        float4 rw[4], rs[4];                      // per-code records (weights+filter, secondary+qid)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            rw[j] = s_rec[2 * (code[j] & 0xFF)];
            rs[j] = s_rec[2 * (code[j] & 0xFF) + 1];
        }
        if (write_qid) {
            int qo[4];
#pragma unroll
            for (int j = 0; j < 4; j++) qo[j] = __float_as_int(rs[j].y);
            if (nv == 4) {
                __stcs((int4*)(A.qid_out + idx0), make_int4(qo[0], qo[1], qo[2], qo[3]));
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (j < nv) A.qid_out[idx0 + j] = qo[j];
            }
        }
        // gap-falling lengths (rare): append to the gap list for Alg. 2 (App. D)
        {
            unsigned gm = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) gm |= (unsigned)(code[j] == kSCodeGap) << j;
            if (__any_sync(0xffffffffu, gm != 0)) {
                ngap += __popc(gm);
#pragma unroll 1
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
                                e.len = j == 0 ? b[0] : (j == 1 ? b[1] : (j == 2 ? b[2] : b[3]));
                                e.arrival = j == 0 ? ar[0] : (j == 1 ? ar[1] : (j == 2 ? ar[2] : ar[3]));
                                e.cost = HAS_COST ? (j == 0 ? co[0] : (j == 1 ? co[1] : (j == 2 ? co[2] : co[3])))
                                                  : __int_as_float(0x7fc00000);
                                A.gap[p] = e;
                            }
                        }
                    }
                }
            }
        }
        // Eq. 4 score, member counter (branch-free: rows nslots / nslots+1 take
        // the excluded / other requests), fast float filter tests
        float sp[4];
        unsigned okm = 0, pass1 = 0, pass2 = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int c = code[j];
            const int ci = c & 0xFF;
            const float4 w = rw[j];
            const bool ok0 = score_sp(b[j], ar[j], HAS_COST ? co[j] : 0.0f, HAS_COST, A.sp, w.x, w.y, w.z, &sp[j]);
            const bool valid = c < kSCodeGap;
            const bool ok = valid && ok0;
            const int row = ok ? ci : (valid ? nslots : nslots + 1);
            s_cnt16[row * kSThreads + tid]++;
            okm |= (unsigned)ok << j;
            const float f1 = MODE == EWSJF_SELECT_SCORE ? sp[j] : ar[j];
            const float f2 = MODE == EWSJF_SELECT_SCORE ? ar[j] : sp[j];
            const bool p1 = MODE == EWSJF_SELECT_SCORE ? f1 >= w.w : f1 <= w.w;
            const bool p2 = MODE == EWSJF_SELECT_SCORE ? f2 <= rs[j].x : f2 >= rs[j].x;
            pass1 |= (unsigned)(ok && p1) << j;
            pass2 |= (unsigned)(ok && p2) << j;
        }
        if (r1k) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const u32 fh = ~ord_f32(ar[j]);
                const u32 sh = __float_as_uint(sp[j]);
                r1k[j] = ((u64)(MODE == EWSJF_SELECT_SCORE ? sh : fh) << 32) | ~(gbase + (uint32_t)(idx0 + j));
                r1q[j] = ((okm >> j) & 1u) ? (code[j] & 0xFF) : -1;
            }
            pass1 = 0;
        }
        // rare: exact 64-bit keys, slot reservations, secondary max (per lane)
        if (__any_sync(0xffffffffu, (pass1 | pass2) != 0)) {
#pragma unroll 1
            for (int j = 0; j < 4; j++) {
                if (!(((pass1 | pass2) >> j) & 1u)) continue;
                // register selects (a rolled loop must not index the arrays dynamically)
                const float arj = j == 0 ? ar[0] : (j == 1 ? ar[1] : (j == 2 ? ar[2] : ar[3]));
                const float spj = j == 0 ? sp[0] : (j == 1 ? sp[1] : (j == 2 ? sp[2] : sp[3]));
                const int cj = j == 0 ? code[0] : (j == 1 ? code[1] : (j == 2 ? code[2] : code[3]));
                const u32 lo = ~(gbase + (uint32_t)(idx0 + j));
                const int q = cj & 0xFF;
                const u32 fh = ~ord_f32(arj);
                const u32 sh = __float_as_uint(spj);
                const u32 k1h = MODE == EWSJF_SELECT_SCORE ? sh : fh;
                const u32 k2h = MODE == EWSJF_SELECT_SCORE ? fh : sh;
                const u64 k1 = ((u64)k1h << 32) | lo;
                if (((pass1 >> j) & 1u) && k1 >= *(volatile u64*)&s_thr64[q]) {
                    const int pos = atomicAdd(&s_bcnt[q], 1);
                    if (pos < cap) {
                        s_buf[(size_t)q * cap + pos] = k1;
                    } else {
                        const int o = atomicAdd(&M->novf, 1);
                        if (o < kOvfCap) { s_ovfk[o] = k1; s_ovfq[o] = (unsigned char)q; }
                        else ndrop++;
                    }
                    if (pos + 1 >= hwm) *(volatile int*)&M->flag = 1;
                    nins++;
                }
                if ((pass2 >> j) & 1u) {
                    // native 32-bit max on the high word first; only a lane that
                    // may hold the maximum runs the 64-bit (CAS) max
                    const u32 old = atomicMax(&s_sechi[q], k2h);
                    if (k2h >= old) {
                        atomicMax(&s_sec[q], ((u64)k2h << 32) | lo);
                        // the fast copy may lag (looser), never pass a tie by mistake: ties go to the exact max
                        *(volatile float*)secf_at(q) = MODE == EWSJF_SELECT_SCORE ? arj : spj;
                    }
                }
            }
        }
    };

    auto flag_set = [&]() -> bool {
        int f = 0;
        if (lane == 0) f = *(volatile int*)&M->flag;
        return __shfl_sync(0xffffffffu, f, 0) != 0;
    };

    // ---- one warp tile: index t = gw + i*GW; t < nfull: TMA ring stage; t ==
    // nfull: the ragged tail (direct loads).  Returns false past the end.
    const bool has_tail = (A.n % kWT) != 0;
    auto tile = [&](int64_t t, int st, uint32_t par, u64* r1k, int* r1q) -> bool {
        const bool full = t < nfull;
        if (!full && !(t == nfull && has_tail)) return false;
        int b4[4];
        float a4[4], c4[4];
        int nv = 4;
        const int64_t i0 = t * kWT + 4 * lane;
        if (full) {
            if (lane_ring) cp_async_wait(S - 1);
            else mbar_wait(&bars[st], par);
            const int4 bv = ((const int4*)stage(st, 0))[lane];
            const float4 av = ((const float4*)stage(st, 1))[lane];
            float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (HAS_COST) cv = ((const float4*)stage(st, 2))[lane];
            b4[0] = bv.x; b4[1] = bv.y; b4[2] = bv.z; b4[3] = bv.w;
            a4[0] = av.x; a4[1] = av.y; a4[2] = av.z; a4[3] = av.w;
            c4[0] = cv.x; c4[1] = cv.y; c4[2] = cv.z; c4[3] = cv.w;
        } else {                                  // the ragged tail: direct loads
            nv = (int)max((int64_t)0, min((int64_t)4, A.n - i0));
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const bool v = j < nv;
                b4[j] = v ? __ldg(A.len + i0 + j) : 0;
                a4[j] = v ? __ldg(A.arrival + i0 + j) : 0.f;
                c4[j] = (HAS_COST && v) ? __ldg(A.cost + i0 + j) : 0.f;
            }
        }
        process4(i0, nv, b4, a4, c4, r1k, r1q);
        if (!full) return false;
        // every lane has consumed the stage (its values fed the stores above)
        if (lane_ring) {
            issue_lane(t + S * GW, st);
        } else {
            __syncwarp();
            if (lane == 0 && t + S * GW < nfull) issue(t + S * GW, st);
        }
        return true;
    };

    // ---- round 1 (every warp's first tile), one structured CTA pass: the
    // scored keys are bucketed by queue into contiguous slices of the overflow
    // area (per-thread offsets = exclusive prefix of the per-thread member
    // counters), each queue's exact K-th key becomes its threshold, and only
    // the keys >= it enter the queue's buffer.  So the stream starts filtered.
    int* s_r1n = (int*)s_sid + kSTab;      // see layout: r1n / r1off follow sid
    int* s_r1off = s_r1n + kSTab;
    u64* s_r1t = (u64*)(s_r1off + kSTab);   // round-1 CTA-wide bounds (0 = none)

    // ---- one loop: round 1 at i == 0, then the private ring; CTA barriers only
    // in collectives.  A warp out of tiles keeps serving collectives until every
    // warp is done (a flag raised by this warp is visible before its ndone
    // increment, and ndone is read before the flag, so no warp leaves while one
    // is pending).  One call site each for tile() and collective() (code size:
    // the cold paths are not duplicated in the instruction stream).
    u64 r1k[4] = {0ull, 0ull, 0ull, 0ull};
    int r1q[4] = {-1, -1, -1, -1};
    u64 g_pre = 0ull;
    int rq = warp % max(nslots, 1);
    int st = 0;
    uint32_t par = 0u;
    int64_t t = gw;
    bool streaming = true;
    for (int i = 0;; ++i) {
        if (streaming) {
            if ((i & 7) == 1 && lane == 0 && nslots > 0) g_pre = __ldcg(&A.gthr[rq]);
            const bool first = i == 0;
            const bool more = tile(t, st, par, first ? r1k : nullptr, first ? r1q : nullptr);
            if (first) {
            __syncthreads();
            if (tid == 0) dbg_max(A, 13, A.dbg ? gtime() : 0ull);   // all first tiles done
            // per-queue totals and per-thread exclusive prefixes (lane l: threads 16l..16l+15)
            for (int q = warp; q < nslots; q += kSWarps) {
                uint32_t* col = (uint32_t*)(s_cnt16 + (size_t)q * kSThreads) + 8 * lane;
                uint32_t w[8];
                int sum = 0;
    #pragma unroll
                for (int k = 0; k < 8; k++) { w[k] = col[k]; sum += (int)(w[k] & 0xffffu) + (int)(w[k] >> 16); }
                int incl = sum;
    #pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += u;
                }
                int run = incl - sum;
    #pragma unroll
                for (int k = 0; k < 8; k++) {
                    const uint32_t a0 = (uint32_t)run; run += (int)(w[k] & 0xffffu);
                    const uint32_t a1 = (uint32_t)run; run += (int)(w[k] >> 16);
                    col[k] = a0 | (a1 << 16);
                }
                if (lane == 31) s_r1n[q] = incl;
            }
            __syncthreads();
            if (tid == 0) dbg_max(A, 14, A.dbg ? gtime() : 0ull);   // prefix done
            if (warp == 0) {
                int carry = 0;
                for (int q0 = 0; q0 < nslots; q0 += 32) {
                    const int q = q0 + lane;
                    const int v = q < nslots ? s_r1n[q] : 0;
                    int incl = v;
    #pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int u = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += u;
                    }
                    if (q < nslots) s_r1off[q] = carry + incl - v;
                    carry += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
            __syncthreads();
    #pragma unroll
            for (int j = 0; j < 4; j++) {
                const int q = r1q[j];
                if (q >= 0) {
                    int k = 0;
    #pragma unroll
                    for (int jj = 0; jj < j; jj++) k += r1q[jj] == q;
                    s_ovfk[s_r1off[q] + s_cnt16[(size_t)q * kSThreads + tid] + k] = r1k[j];
                }
            }
            __syncthreads();
            if (tid == 0) dbg_max(A, 15, A.dbg ? gtime() : 0ull);   // scatter done
            // slices larger than a warp's register selection (typically one dominant
            // queue): one CTA-wide 256-bucket histogram over the keys' high words gives
            // a valid bound — the lower edge of the highest bucket at which at least K
            // keys lie above — in four barriers; a bucket too full (ties) falls back to
            // the warp selection below.
            {
                // s_h: [256] buckets, [256] max, [257] min, [258..263] pass state (buffers still empty)
                unsigned* s_h = (unsigned*)s_buf;
                for (int q = 0; q < nslots; q++) {
                    const int n = s_r1n[q];
                    if (n <= 32 * kRegSel) continue;
                    const u64* sl = s_ovfk + s_r1off[q];
                    u32 hv[kOvfCap / kSThreads];
                    u32 mx = 0u, mn = 0xffffffffu;
    #pragma unroll
                    for (int r = 0; r < kOvfCap / kSThreads; r++) {
                        const int j = tid + kSThreads * r;
                        hv[r] = j < n ? (u32)(sl[j] >> 32) : 0u;
                        if (j < n) { mx = max(mx, hv[r]); mn = min(mn, hv[r]); }
                    }
                    mx = __reduce_max_sync(0xffffffffu, mx);
                    mn = __reduce_min_sync(0xffffffffu, mn);
                    if (tid == 0) { s_h[256] = 0u; s_h[257] = 0xffffffffu; }
                    __syncthreads();
                    if (lane == 0) { atomicMax(&s_h[256], mx); atomicMin(&s_h[257], mn); }
                    __syncthreads();
                    u32 lo_h = s_h[257], hi_h = s_h[256];    // high-word range still open
                    unsigned above = 0;                      // keys with high word > hi_h
                    u64 res = 0ull;
                    for (int pass = 0; pass < 4; pass++) {
                        __syncthreads();
                        if (tid < 256) s_h[tid] = 0u;
                        __syncthreads();
                        const unsigned long long R = (unsigned long long)(hi_h - lo_h) + 1ull;
    #pragma unroll
                        for (int r = 0; r < kOvfCap / kSThreads; r++)
                            if (tid + kSThreads * r < n && hv[r] >= lo_h && hv[r] <= hi_h)
                                atomicAdd(&s_h[(unsigned)(((unsigned long long)(hv[r] - lo_h) * 256ull) / R)], 1u);
                        __syncthreads();
                        if (warp == 0) {                     // highest bucket b with above + #(>= b) >= K
                            unsigned c[8], tot = 0;
    #pragma unroll
                            for (int k = 0; k < 8; k++) { c[k] = s_h[255 - (8 * lane + k)]; tot += c[k]; }
                            unsigned incl = tot;
    #pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                                if (lane >= o) incl += u;
                            }
                            unsigned run = above + incl - tot;
                            int bsel = -1;
                            unsigned csel = 0, cb = 0;
    #pragma unroll
                            for (int k = 0; k < 8; k++) {
                                run += c[k];
                                if (bsel < 0 && run >= (unsigned)K) { bsel = 255 - (8 * lane + k); csel = run; cb = c[k]; }
                            }
                            const unsigned hit = __ballot_sync(0xffffffffu, bsel >= 0);
                            const int src = hit ? __ffs(hit) - 1 : 0;
                            bsel = __shfl_sync(0xffffffffu, bsel, src);
                            csel = __shfl_sync(0xffffffffu, csel, src);
                            cb = __shfl_sync(0xffffffffu, cb, src);
                            if (lane == 0) {
                                // bucket b holds high words [e_b, e_{b+1}), e_b = lo + ceil(b R / 256)
                                const unsigned long long eb = (unsigned long long)lo_h + ((unsigned long long)bsel * R + 255ull) / 256ull;
                                const unsigned long long eb1 = (unsigned long long)lo_h + ((unsigned long long)(bsel + 1) * R + 255ull) / 256ull;
                                unsigned st = 0;                  // 0: continue, 1: done, 2: give up
                                if (bsel < 0) st = 2;
                                else if (csel <= (unsigned)(cap - 64)) { st = 1; s_h[258] = (unsigned)eb; }
                                else if (eb1 - eb <= 1) st = 2;   // one high word: ties, the warp path decides
                                else { s_h[259] = (unsigned)eb; s_h[260] = (unsigned)(eb1 - 1); s_h[261] = csel - cb; }
                                s_h[262] = st;
                            }
                        }
                        __syncthreads();
                        const unsigned st = s_h[262];
                        if (st == 1) { res = (u64)s_h[258] << 32; break; }
                        if (st == 2) break;
                        lo_h = s_h[259]; hi_h = s_h[260]; above = s_h[261];
                    }
                    if (tid == 0) s_r1t[q] = res;           // 0: none, the warp selection decides
                    // the CTA copies the keys >= the bound straight into the buffer (<= cap - 64 of them)
                    if (res) {
    #pragma unroll
                        for (int r = 0; r < kOvfCap / kSThreads; r++) {
                            const int j = tid + kSThreads * r;
                            if (j < n && sl[j] >= res) s_buf[(size_t)q * cap + atomicAdd(&s_bcnt[q], 1)] = sl[j];
                        }
                    }
                    __syncthreads();
                }
            }
            if (tid == 0) dbg_max(A, 12, A.dbg ? gtime() : 0ull);   // CTA histogram bounds done
            for (int q = warp; q < nslots; q += kSWarps) {
                const int n = s_r1n[q];
                const u64* sl = s_ovfk + s_r1off[q];
                u64 t = 0ull;
                const bool copied = n > 32 * kRegSel && s_r1t[q] != 0ull;     // done CTA-wide above
                if (n > 32 * kRegSel) {
                    t = s_r1t[q];
                    if (!t) t = warp_select_arr(sl, n, K, cap - 64);   // window: <= cap-64 survive
                }
                else if (n > K) t = warp_kth_arr(sl, n, K, kApproxBit, cap - 64);
                if (lane == 0) dbg_max(A, 10, A.dbg ? gtime() : 0ull);
                u64* bb = s_buf + (size_t)q * cap;
                int nb = copied ? s_bcnt[q] : 0;
                for (int j0 = 0; j0 < (copied ? 0 : n); j0 += 32) {
                    const int j = j0 + lane;
                    const u64 v = j < n ? sl[j] : 0ull;
                    const bool keep = j < n && v >= t;
                    const unsigned m = __ballot_sync(0xffffffffu, keep);
                    if (keep) bb[nb + __popc(m & ((1u << lane) - 1u))] = v;
                    nb += __popc(m);
                }
                __syncwarp();
                if (nb > K && !copied) {         // window survivors -> a tighter bound
                    t = warp_kth_arr(bb, nb, K, kApproxBit, cap - 64);
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
                    nb = outc;
                }
                if (lane == 0) dbg_max(A, 11, A.dbg ? gtime() : 0ull);
                uint32_t* col = (uint32_t*)(s_cnt16 + (size_t)q * kSThreads) + 8 * lane;
    #pragma unroll
                for (int k = 0; k < 8; k++) col[k] = 0u;
                if (lane == 0) {
                    s_bcnt[q] = nb;
                    if (t) { raise_thr(q, t); atomicMax(&A.gthr[q], t); }
                }
                if (bm) {                        // board row: this CTA's top-bm keys of q
                    u64 prev = ~0ull;
                    for (int i = 0; i < bm; i++) {
                        u64 mx = 0;
                        for (int j = lane; j < nb; j += 32) {
                            const u64 v = bb[j];
                            if (v < prev && v > mx) mx = v;
                        }
                        mx = warp_max_u64(mx);
                        if (lane == 0) A.board[((size_t)q * G + blockIdx.x) * bm + i] = mx;
                        prev = mx;
                    }
                }
            }
            __syncthreads();
                if (A.dbg && lane == 0 && warp == 0) dbg_max(A, 7, gtime());
            }
            if (more) {
                t += GW;
                if (++st == S) { st = 0; par ^= 1u; }
                if ((i & 7) == 6 && lane == 0 && nslots > 0) {
                    if (g_pre) raise_thr(rq, g_pre);
                    rq += kSWarps;
                    if (rq >= nslots) rq -= nslots * (rq / nslots);
                }
                if (bm && i == 3)
                    for (int q = warp; q < nslots; q += kSWarps) board_refresh(q);
            } else {
                streaming = false;
                if (lane == 0) dbg_max(A, 2, A.dbg ? gtime() : 0ull);
                __threadfence_block();
                __syncwarp();
                if (lane == 0) atomicAdd(&M->ndone, 1);
            }
        } else {
            int f = 0, dn = 0;
            if (lane == 0) {
                dn = *(volatile int*)&M->ndone;
                __threadfence_block();
                f = *(volatile int*)&M->flag;
            }
            f = __shfl_sync(0xffffffffu, f, 0);
            dn = __shfl_sync(0xffffffffu, dn, 0);
            if (!f) {
                if (dn == kSWarps) break;
                __nanosleep(64);
                continue;
            }
        }
        if (flag_set()) collective();
    }
    __syncthreads();
    if (tid == 0) dbg_max(A, 3, A.dbg ? gtime() : 0ull);

    // ---- final trim: every queue keeps exactly its local top-K (no overflow is
    // pending: an overflow always raised the flag first)
    for (int q = warp; q < nslots; q += kSWarps) {
        u64* bb = s_buf + (size_t)q * cap;
        const int nb = min(s_bcnt[q], cap);
        if (nb > K) {
            const u64 t = warp_kth_arr(bb, nb, K);
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
            ncomp++;
            if (lane == 0) { s_bcnt[q] = outc; raise_thr(q, t); atomicMax(&A.gthr[q], t); }
        }
    }
    __syncthreads();

    // ---- rows out: keys >= max(local, global) threshold, secondary, members
    const Rows& R = A.rows;
    long long counted = 0;
    for (int q = warp; q < nslots; q += kSWarps) {
        const int nb = min(s_bcnt[q], cap);
        u64 tf = s_thr64[q];
        const u64 gg = __ldcg(&A.gthr[q]);
        tf = gg > tf ? gg : tf;
        u64* dst = R.keys + ((size_t)q * G + blockIdx.x) * R.cap;
        int outc = 0;
        for (int j0 = 0; j0 < nb; j0 += 32) {
            const int j = j0 + lane;
            const u64 v = j < nb ? s_buf[(size_t)q * cap + j] : 0ull;
            const bool keep = j < nb && v >= tf;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) dst[outc + __popc(m & ((1u << lane) - 1u))] = v;
            outc += __popc(m);
        }
        long long mm = 0;
        const uint32_t* c32 = (const uint32_t*)(s_cnt16 + (size_t)q * kSThreads);
        for (int k = lane; k < kSThreads / 2; k += 32) { const uint32_t v = c32[k]; mm += (v & 0xffffu) + (v >> 16); }
        for (int o = 16; o; o >>= 1) mm += __shfl_xor_sync(0xffffffffu, mm, o);
        mm += s_r1n[q];
        if (lane == 0) {
            R.cnt[(size_t)q * G + blockIdx.x] = outc;
            R.sec[(size_t)q * G + blockIdx.x] = s_sec[q];
            R.members[(size_t)q * G + blockIdx.x] = mm;
        }
        counted += mm;   // lane-uniform
    }
    if (lane == 0) dbg_max(A, 4, A.dbg ? gtime() : 0ull);
    // excluded = the dummy row nslots; invalid = processed - counted - excluded - gap
    {
        const uint32_t* c32 = (const uint32_t*)(s_cnt16 + (size_t)nslots * kSThreads);
        unsigned e = 0;
        if (warp == 0)
            for (int k = lane; k < kSThreads / 2; k += 32) { const uint32_t v = c32[k]; e += (v & 0xffffu) + (v >> 16); }
        exc = warp == 0 ? e : 0u;   // reduced below with the other per-lane counters
        if (warp == 0) {
            unsigned ee = e;
            for (int o = 16; o; o >>= 1) ee += __shfl_xor_sync(0xffffffffu, ee, o);
            excl_total = ee;
        }
    }
    long long invl = processed - (long long)ngap;
    for (int o = 16; o; o >>= 1) {
        invl += __shfl_xor_sync(0xffffffffu, invl, o);
        exc += __shfl_xor_sync(0xffffffffu, exc, o);
        nins += __shfl_xor_sync(0xffffffffu, nins, o);
        ndrop += __shfl_xor_sync(0xffffffffu, ndrop, o);
    }
    if (lane == 0) {
        invl -= counted;
        if (warp == 0) invl -= (long long)excl_total;
        if (invl) atomicAdd(&A.ctr->n_invalid, (unsigned long long)invl);
        if (exc) atomicAdd(&A.ctr->n_excluded, (unsigned long long)exc);
        if (nins) atomicAdd(&A.ctr->dbg_inserted, (unsigned long long)nins);
        if (ncomp) atomicAdd(&A.ctr->dbg_compactions, (unsigned long long)ncomp);
        if (ndrop) atomicAdd(&A.ctr->dbg_overflow, (unsigned long long)ndrop);
    }
}

// Clear this CTA's board rows (nobody reads them any more).
__device__ __forceinline__ void board_clear(const PartialArgs& A, int nslots) {
    if (!A.board_m) return;
    for (int i = threadIdx.x; i < nslots * A.board_m; i += blockDim.x) {
        const int s = i / A.board_m, j = i % A.board_m;
        A.board[((size_t)s * gridDim.x + blockIdx.x) * A.board_m + j] = 0ull;
    }
}

// Streaming pass alone (the merge is a separate launch).
template <int MODE, bool HAS_COST>
__global__ void __launch_bounds__(kSThreads, 1)
    stream_kernel(const __grid_constant__ PartialArgs A, const __grid_constant__ Policy P) {
    extern __shared__ __align__(128) unsigned char smem[];
    stream_phase<MODE, HAS_COST>(A, P, smem);
    board_clear(A, P.nslots);
}

__device__ __forceinline__ void sgrid_barrier(unsigned int* ctr, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v < target) __nanosleep(32);
        } while (v < target);
    }
    __syncthreads();
}

// Fused tick: streaming pass -> grid barrier -> per-queue merge.
template <int MODE, bool HAS_COST>
__global__ void __launch_bounds__(kSThreads, 1)
    stream_tick_kernel(const __grid_constant__ PartialArgs A, const __grid_constant__ Policy P,
                       const __grid_constant__ MergeArgs MA) {
    extern __shared__ __align__(128) unsigned char smem[];
    stream_phase<MODE, HAS_COST>(A, P, smem);
    sgrid_barrier(&A.ctr->barrier, gridDim.x);
    if (threadIdx.x == 0) dbg_max(A, 8, A.dbg ? gtime() : 0ull);
    board_clear(A, P.nslots);
    merge_phase<MERGE_IN_ROWS, MERGE_OUT_FINAL, HAS_COST>(MA, P, smem);
    if (threadIdx.x == 0) dbg_max(A, 9, A.dbg ? gtime() : 0ull);
}

int64_t merge_smem_total(int in_mode);

template <int MO, bool C>
static cudaError_t launch_s(const PartialArgs& A, const Policy& P, const MergeArgs* MA, int grid, cudaStream_t st) {
    const int64_t ls = stream_layout(C, A.lut_size, P.nslots, A.cap, A.stages).total;
    if (!MA) {
        auto k = stream_kernel<MO, C>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ls);
        if (e != cudaSuccess) return e;
        k<<<grid, kSThreads, ls, st>>>(A, P);
        return cudaGetLastError();
    }
    const int64_t lm = merge_smem_total(MERGE_IN_ROWS);
    const int64_t smem = ls > lm ? ls : lm;
    auto k = stream_tick_kernel<MO, C>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void* args[] = {(void*)&A, (void*)&P, (void*)MA};
    return cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kSThreads), args, (size_t)smem, st);
}

// Route + score + select over an aligned pool with a LUT-routable partition of
// <= 64 queues; MA == nullptr: streaming pass only.
cudaError_t launch_stream(const PartialArgs& A, const Policy& P, const MergeArgs* MA, bool has_cost, int grid,
                          cudaStream_t st) {
    if (A.sp.mode == EWSJF_SELECT_FIFO)
        return has_cost ? launch_s<EWSJF_SELECT_FIFO, true>(A, P, MA, grid, st)
                        : launch_s<EWSJF_SELECT_FIFO, false>(A, P, MA, grid, st);
    return has_cost ? launch_s<EWSJF_SELECT_SCORE, true>(A, P, MA, grid, st)
                    : launch_s<EWSJF_SELECT_SCORE, false>(A, P, MA, grid, st);
}

}  // namespace ewsjf
