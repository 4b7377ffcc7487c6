// ftick.cu — the fused EWSJF scheduling tick on sm_100a: route (A8) + Eq. 4
// score (A10) + per-queue count / head / top-k filter (A11) in one HBM pass
// over the pending pool, then a grid barrier and the per-queue merge + Alg. 1
// ArgMax.  Paper: Dispatcher P:162, Eq. 4, Alg. 1 P:167-196;
// readings R1-R27 in DESIGN.md §3.  Gap-falling lengths (App. D, Alg. 2) are
// collected here and resolved by merge_phase (merge.cuh).
//
// Design:
//  * one 512-thread CTA per SM (cooperative launch).  Warp (b, w) owns the
//    contiguous tile block w*G + b of the pool (128 requests per tile), so the
//    first tile of every warp — together the "sample", 16 tiles per CTA spread
//    over the whole pool — is representative whatever the pool order;
//  * every warp streams its block through a private ring of 1-D TMA bulk
//    copies (cp.async.bulk, one elected lane, mbarrier per stage);
//  * per request: byte-LUT route, one 32-byte per-code record (weights, fast
//    thresholds, stable id, member-counter offset), Eq. 4 with one MUFU.LG2 +
//    one MUFU.RCP, a per-thread u16 member counter, two float compares; the
//    qid goes out as one 16-byte streaming store per 4 requests;
//  * sample bound: after its sample tile every CTA publishes its top board_m
//    keys per queue; the last CTA to publish turns the G*board_m keys of each
//    queue into a valid bound on the queue's K-th key (K-th largest of
//    distinct real keys) and releases the others; the sample keys are then
//    filtered against it.  So the stream starts with near-final thresholds
//    and only ~K*(N/S) keys per queue are ever inserted;
//  * survivors go to per-(queue, CTA) rows in global memory (L2); a full row
//    triggers a CTA collective that cuts it to its exact K-th key (CTA radix
//    select) and raises the queue's thresholds here and in gthr;
//  * after a grid barrier (monotone ticket) CTA q merges queue q's rows:
//    candidates >= gthr into shared memory, CTA radix select of the exact
//    K-th key, rank sort of the K survivors, outputs; the last CTA takes
//    Alg. 1's ArgMax.
#include <climits>
#include <type_traits>
#include "merge.cuh"
#include "select.cuh"

namespace ewsjf {

constexpr int kFT = 768;            // threads per CTA (24 warps: latency hiding for the smem/MUFU chains)
constexpr int kFW = kFT / 32;       // warps
constexpr int kFTile = 128;         // requests per warp tile (4 per lane)
constexpr int kFCodeFar = 0xFD;     // length beyond the LUT: binary search in the rare path
constexpr int kFCodeGap = 0xFE;     // length between queues (App. D)
constexpr int kFCodeBad = 0xFF;     // len < 1
constexpr int kFCodeNone = 0xFC;    // padding of a ragged lane
constexpr int kFMaxSlots = 64;
constexpr int kFBoardMax = 2;       // board keys per (queue, CTA); G * m <= 32 * kFBoardRegs
constexpr int kFBoardRegs = 10;
constexpr int kFMaxStages = 8;      // ring depth cap (EWSJF_STAGES)
constexpr int kFCntRow = kFT / 4;   // words per u8 counter row

__host__ __device__ inline int64_t fal(int64_t x) { return (x + 127) & ~(int64_t)127; }

struct FMisc {
    int flag;           // some row crossed its high-water mark: collective wanted
    int novf;           // overflow list fill
    int ndone;          // warps done streaming
    int last;           // this CTA published the last sample board
    int ncoll;
    int sel_d, sel_cd;
    int pn;             // merge: candidate pool fill
    unsigned sel_above;
    int maxnc;          // merge: longest candidate row
    unsigned long long members, sec;
    unsigned long long tcoll;
    unsigned long long agg[3];   // end of stream: invalid, excluded, inserted (CTA totals)
};

struct FSmem {
    int64_t rec, lut, ring, bars, thr64, sec64, bmax, rcnt, misc, hist, surv, ctot, cnt, total;
};
// the per-code records and the LUT sit at fixed offsets (immediate addressing on the hot path)
constexpr int kFRecOff = 0;
constexpr int kFLutOff = 32 * 256;
__host__ __device__ inline FSmem fsmem_layout(bool has_cost, int lut_size, int nslots, int stages) {
    FSmem L;
    const int narr = has_cost ? 3 : 2;
    int64_t o = 0;
    L.rec = kFRecOff;
    L.lut = kFLutOff;
    o = fal(kFLutOff + lut_size + 1);
    L.ring = o;  o = fal(o + (int64_t)kFW * stages * narr * kFTile * 4);
    L.bars = o;  o = fal(o + 20LL * kFMaxStages);   // mbarriers, release counters, stage chunk ids
    L.thr64 = o; o = fal(o + 8LL * kFMaxSlots);
    L.sec64 = o; o = fal(o + 8LL * kFMaxSlots);
    L.bmax = o;  o = fal(o + 8LL * kFMaxSlots * kFBoardMax);
    L.rcnt = o;  o = fal(o + 4LL * kFMaxSlots);
    L.misc = o;  o = fal(o + sizeof(FMisc));
    L.hist = o;  o = fal(o + 4LL * 256);
    L.surv = o;  o = fal(o + 8LL * EWSJF_MAX_K);
    L.ctot = o;  o = fal(o + 4LL * (kFMaxSlots + 1));     // flushed member counts per row
    L.cnt = o;   o = fal(o + 1LL * kFT * (nslots + 1));   // u8 rows: members 0..nslots-1, other codes
    L.total = o;
    return L;
}
int64_t ftick_smem_bytes(bool has_cost, int lut_size, int nslots, int stages) {
    return fsmem_layout(has_cost, lut_size, nslots, stages).total;
}

__device__ __forceinline__ unsigned long long fgtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// wait until at most n of this thread's cp.async groups are pending
__device__ __forceinline__ void cp_async_wait_n(int n) {
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
// 1-D bulk copy with an L2 cache-policy hint (evict-first for the pool, read exactly once:
// the streamed 120 MB then stop evicting the kernel's code, LUT, boards and rows from L2)
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// non-aligned barrier: warps arrive from different call sites (the collective is entered from the
// streaming loop and from the idle loop), which the .aligned form (bar.sync) does not allow
__device__ __forceinline__ void fbar(int id) { asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(kFT) : "memory"); }

// key high word -> fast-test float.  SCORE keys: the bits of s' (>= +0).
// FIFO keys: hi = ~ord(arrival), inverted here.
__device__ __forceinline__ float fifo_hi_to_f(u32 hi) {
    const u32 u = ~hi;
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// CTA-wide exact K-th largest key (512 threads, all must call).  for_each(f)
// calls f(key) for this thread's share of the candidate keys (0 = none);
// requires >= K nonzero keys.  MSB-first 8-bit radix select over a 256-bin
// shared histogram; returns early with a threshold t such that exactly K keys
// are >= t when the remaining keys of the selected digit are exactly the ones
// still wanted.
template <typename ForEach>
__device__ __forceinline__ u64 block_kth(ForEach for_each, int K, unsigned* hist, FMisc* M) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    u64 prefix = 0ull, pmask = 0ull;
    int kk = K;
    for (int shift = 56; shift >= 0; shift -= 8) {
        if (tid < 256) hist[tid] = 0u;
        fbar(1);
        for_each([&](u64 k) {
            if (k && (k & pmask) == prefix) atomicAdd(&hist[(unsigned)(k >> shift) & 255u], 1u);
        });
        fbar(1);
        if (warp == 0) {
            unsigned c[8], s = 0;
#pragma unroll
            for (int i = 0; i < 8; i++) { c[i] = hist[255 - 8 * lane - i]; s += c[i]; }
            unsigned incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            unsigned run = incl - s;
            int dsel = -1;
            unsigned above = 0, cd = 0;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                if (dsel < 0 && run + c[i] >= (unsigned)kk) { dsel = 255 - 8 * lane - i; above = run; cd = c[i]; }
                run += c[i];
            }
            const unsigned hit = __ballot_sync(0xffffffffu, dsel >= 0);
            const int src = hit ? __ffs(hit) - 1 : 0;
            dsel = __shfl_sync(0xffffffffu, dsel, src);
            above = __shfl_sync(0xffffffffu, above, src);
            cd = __shfl_sync(0xffffffffu, cd, src);
            if (lane == 0) { M->sel_d = dsel; M->sel_above = above; M->sel_cd = (int)cd; }
        }
        fbar(1);
        const int d = M->sel_d;
        const int above = (int)M->sel_above, cd = M->sel_cd;
        prefix |= (u64)(unsigned)d << shift;
        pmask |= 0xFFull << shift;
        kk -= above;
        if (cd == kk) return prefix;   // exactly K keys >= prefix (lower bits zero)
    }
    return prefix;
}

// Warp-wide valid bounds for two queues at once from R high words per lane each
// (0 = absent): t[x] has its low kFLowBit bits zero and #(v[x] >= t[x]) >= K
// over the real (nonzero) values, or 0 if fewer than K are present.  MSB-first
// descent started below the common prefix of the real values and stopped at
// bit kFLowBit (for fp32 bits: within 2^-(23-kFLowBit) relative), so the
// queue's K-th key is >= (t << 32).  The two descents are interleaved and the
// per-lane counts are summed as a tree, so a step is a few independent
// compares + two REDUX (the dependent chain of a sequential count made this
// ~250 cycles per step).
constexpr int kFLowBit = 15;
template <int R>
__device__ __forceinline__ int tree_count_ge(const u32 (&v)[R], u32 cand) {
    int c[R];
#pragma unroll
    for (int r = 0; r < R; r++) c[r] = v[r] >= cand ? 1 : 0;
#pragma unroll
    for (int w = 1; w < R; w <<= 1)
#pragma unroll
        for (int r = 0; r + w < R; r += 2 * w) c[r] += c[r + w];
    return c[0];
}
template <int R>
__device__ __forceinline__ void warp_kth_hi2(const u32 (&v0)[R], const u32 (&v1)[R], int K, u32* t_out) {
    u32 mx[2] = {0u, 0u}, mn[2] = {0xffffffffu, 0xffffffffu};
    int nz[2] = {0, 0};
#pragma unroll
    for (int r = 0; r < R; r++) {
        mx[0] = max(mx[0], v0[r]); mx[1] = max(mx[1], v1[r]);
        mn[0] = v0[r] ? min(mn[0], v0[r]) : mn[0]; mn[1] = v1[r] ? min(mn[1], v1[r]) : mn[1];
        nz[0] += v0[r] != 0u; nz[1] += v1[r] != 0u;
    }
    u32 t[2];
    int hb = -1;
    bool on[2];
#pragma unroll
    for (int x = 0; x < 2; x++) {
        mx[x] = __reduce_max_sync(0xffffffffu, mx[x]);
        mn[x] = __reduce_min_sync(0xffffffffu, mn[x]);
        nz[x] = __reduce_add_sync(0xffffffffu, nz[x]);
        on[x] = nz[x] >= K && K >= 1;
        const u32 diff = mx[x] ^ mn[x];
        const int h = diff ? 31 - __clz(diff) : -1;
        t[x] = h >= 0 ? (mx[x] & ~((2u << h) - 1u)) : mx[x];   // common prefix: every real value is >= t
        if (on[x]) hb = max(hb, h);
    }
    for (int bit = hb; bit >= kFLowBit; bit--) {
        const u32 c0 = t[0] | (1u << bit), c1 = t[1] | (1u << bit);
        const int n0 = __reduce_add_sync(0xffffffffu, tree_count_ge(v0, c0));
        const int n1 = __reduce_add_sync(0xffffffffu, tree_count_ge(v1, c1));
        if (n0 >= K) t[0] = c0;
        if (n1 >= K) t[1] = c1;
    }
    t_out[0] = on[0] ? t[0] : 0u;
    t_out[1] = on[1] ? t[1] : 0u;
}

// CTA-wide: copy the keys >= t given by for_each into out[] (any order), returns the count.
template <typename ForEach>
__device__ __forceinline__ int block_collect(ForEach for_each, u64 t, u64* out, int cap, FMisc* M) {
    if (threadIdx.x == 0) M->pn = 0;
    fbar(1);
    for_each([&](u64 k) {
        if (k && k >= t) {
            const int p = atomicAdd(&M->pn, 1);
            if (p < cap) out[p] = k;
        }
    });
    fbar(1);
    const int n = M->pn;
    fbar(1);
    return n < cap ? n : cap;
}

template <int MODE, bool HAS_COST>
__global__ void __launch_bounds__(kFT, 1)
    ftick_kernel(const __grid_constant__ FArgs A, const Policy* __restrict__ Pd,
                 const __grid_constant__ MergeArgs MA) {
    // the policy tables (6 KB) live in device memory, uploaded only when they change:
    // as a kernel parameter they added ~4.5 us to every launch (measured); only the
    // setup, the rare path and the merge read them
    const Policy& P = *Pd;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int nslots = A.nslots, K = A.K, RC = A.RC, HWM = A.HWM;
    const int lutsz = A.lut_size;
    const int R = A.stages;
    constexpr bool SCORE = MODE == EWSJF_SELECT_SCORE;
    constexpr int narr = HAS_COST ? 3 : 2;
    const FSmem L = fsmem_layout(HAS_COST, lutsz, nslots, R);
    unsigned char* lut = smem + kFLutOff;
    // per-code records, two arrays of 16-byte entries (one [code][2] array put the lanes of
    // a warp with mixed codes on 4 bank groups: 8 wavefronts per LDS.128 instead of 4)
    float4* recA = (float4*)(smem + kFRecOff);          // [code]: {wb, wu, wf', thrf}
    float4* recB = recA + 256;                          // [code]: {secf, qid, cntoff, -}
    u64* thr64 = (u64*)(smem + L.thr64);
    u64* sec64 = (u64*)(smem + L.sec64);
    u32* bmax = (u32*)(smem + L.bmax);     // [q][m] high words of the CTA's top keys (native u32 atomics)
    int* rcnt = (int*)(smem + L.rcnt);
    FMisc* M = (FMisc*)(smem + L.misc);
    unsigned* hist = (unsigned*)(smem + L.hist);
    u64* surv = (u64*)(smem + L.surv);
    unsigned char* cntb = smem + L.cnt;
    unsigned* ctot = (unsigned*)(smem + L.ctot);
    const bool dbg = A.dbg != nullptr;
    auto stamp = [&](int s) {
        if (dbg && tid == 0) A.dbg[cta * kDbgStride + s] = fgtime();
    };
    stamp(0);
    if (A.diag & 4) return;   // timing diagnostic (EWSJF_DIAG=4): launch + teardown of this configuration only

    // ---- chunk schedule.  The pool is cut into chunks of CH = kFW * kFTile requests;
    // CTA cta takes chunks cta, cta + G, cta + 2G, ... (iteration i: chunk cta + G*i), so at
    // any time the grid sweeps one contiguous window of the pool.  Warp w owns tile w of every
    // chunk (global tile (cta + G*i)*kFW + w).  Full chunks are staged into shared memory by
    // a CTA-level ring of R stages of 1-D TMA bulk copies (one CH*4-byte copy per array, one
    // mbarrier per stage); the last warp to release a stage refills it with iteration i + R.
    // (Measured, tools/mb_stream.cu: this pipeline streams the 16 B/request pattern at
    // 5.6 TB/s; the per-warp cp.async ring reached 4.3 TB/s and dynamic per-warp tile
    // claims from a grid-wide counter cost another ~9 us.)  A ragged last chunk is read
    // with direct loads.  Iteration 0 is each CTA's sample chunk.
    constexpr int CH = kFW * kFTile;
    const int64_t nchunks = (A.n + CH - 1) / CH;
    const int64_t nfullc = A.n / CH;
    const int64_t nfull = A.n / kFTile;
    // The last A.dyn_tail rounds of chunks are claimed from a grid-wide counter by whichever
    // CTA refills a stage first (one atomic per chunk, by the refilling thread): the CTAs
    // finish together instead of waiting for the slowest SM's last static chunks.  The
    // chunk id of every stage is published in shared memory with the stage (-1: no more).
    const int my_iters = cta < nchunks ? (int)((nchunks - 1 - cta) / G + 1) : 0;
    const int64_t srounds = A.dyn_tail > 0 ? max((int64_t)0, nchunks / G - A.dyn_tail) : (int64_t)my_iters;
    const int my_static = (int)min((int64_t)my_iters, srounds);
    const int64_t sbase = srounds * G;                                   // first dynamically claimed chunk
    unsigned char* ringc = smem + L.ring;
    uint64_t* fullb = (uint64_t*)(smem + L.bars);                       // [R] stage landed
    unsigned* relc = (unsigned*)(smem + L.bars + 8 * kFMaxStages);      // [R] warp releases (monotone)
    int64_t* schunk = (int64_t*)(smem + L.bars + 12 * kFMaxStages);     // [R] chunk of the stage, -1: done
    auto stage = [&](int st, int a) -> unsigned char* { return ringc + (st * narr + a) * (CH * 4) + warp * (kFTile * 4); };
    auto issue_chunk = [&](int i) {   // one thread: iteration i's chunk into stage i % R
        int64_t c = -1;
        if (i < my_static) c = (int64_t)cta + (int64_t)G * i;
        else if (A.dyn_tail > 0) c = sbase + (int64_t)atomicAdd(&A.ctr->ftiles, 1ull);
        if (c >= nchunks) c = -1;
        EWSJF_CHECK(c < nfullc ? (c + 1) * CH <= A.n : c == -1 || c == nchunks - 1);
        const int s = i % R;
        uint64_t* b = &fullb[s];
        *(volatile int64_t*)&schunk[s] = c;
        if (c >= 0 && c < nfullc) {
            mbar_arrive_expect_tx(b, (uint32_t)(narr * CH * 4));     // release: orders the chunk id before
            unsigned char* d = ringc + s * narr * (CH * 4);
            if (A.l2_hint) {
                uint64_t pol;
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                tma_load_1d_hint(d, A.len + c * CH, CH * 4, b, pol);
                tma_load_1d_hint(d + CH * 4, A.arrival + c * CH, CH * 4, b, pol);
                if (HAS_COST) tma_load_1d_hint(d + 2 * CH * 4, A.cost + c * CH, CH * 4, b, pol);
            } else {
                tma_load_1d(d, A.len + c * CH, CH * 4, b);
                tma_load_1d(d + CH * 4, A.arrival + c * CH, CH * 4, b);
                if (HAS_COST) tma_load_1d(d + 2 * CH * 4, A.cost + c * CH, CH * 4, b);
            }
        } else {
            // the ragged last chunk (direct loads) or the end: complete the phase without data
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
        }
    };
    {   // the LUT first (its own commit group, issued before the ring's bulk copies)
        const int l16 = (lutsz + 1 + 15) / 16;
        const int4* src = reinterpret_cast<const int4*>(A.lut_dev);
        for (int i = tid; i < l16; i += kFT) cp_async16(smem + kFLutOff + 16 * i, src + i);
        // and the per-queue weights / stable ids of the first 64 positions (the setup's
        // only policy reads) into the surv region, 16 chunks of 16 B per array
        if (tid < 64) {
            const int arr = tid >> 4, ch = tid & 15;
            const int32_t* srcp = arr == 0 ? (const int32_t*)Pd->wb : arr == 1 ? (const int32_t*)Pd->wu
                                : arr == 2 ? (const int32_t*)Pd->wf : Pd->sid;
            cp_async16(smem + L.surv + arr * 256 + ch * 16, srcp + ch * 4);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (tid == 0) {   // after the LUT: its 32 KB (L2 hits) must not queue behind the ring's HBM reads
        for (int s = 0; s < R; s++) { mbar_init(&fullb[s], 1); relc[s] = 0u; }
        fence_mbar_init();
        // the sample chunk first; with sample_first the rest of the ring follows the setup
        // (~2 us later) so that the sample's HBM reads are not queued behind them
        for (int i = 0; i < (A.sample_first ? 1 : R); i++) issue_chunk(i);
        // the chunks after the ring go to L2 while the CTAs agree on the sample bound
        // (the HBM would otherwise idle for ~6 us)
        for (int i = R; i < R + A.l2_prefetch && i < my_static; i++) {
            const int64_t c = (int64_t)cta + (int64_t)G * i;
            if (c >= nfullc) break;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.len + c * CH), "r"(CH * 4) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.arrival + c * CH), "r"(CH * 4) : "memory");
            if (HAS_COST)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.cost + c * CH), "r"(CH * 4) : "memory");
        }
    }
    stamp(10);

    // ---- setup while the first tiles are in flight
    {
        for (int q = tid; q < kFMaxSlots; q += kFT) {
            thr64[q] = 0ull; sec64[q] = 0ull; rcnt[q] = 0;
            for (int m = 0; m < kFBoardMax; m++) bmax[q * kFBoardMax + m] = 0u;
        }
        if (dbg && tid == 0) A.dbg[cta * kDbgStride + 11] = fgtime();
        uint4* c4 = (uint4*)cntb;
        const int n16 = (kFT * (nslots + 1)) / 16;
        for (int q = tid; q <= kFMaxSlots; q += kFT) ctot[q] = 0u;
        for (int i = tid; i < n16; i += kFT) c4[i] = make_uint4(0u, 0u, 0u, 0u);
        if (dbg && tid == 0) A.dbg[cta * kDbgStride + 12] = fgtime();
        if (tid == 0) {
            M->flag = 0; M->novf = 0; M->ndone = 0; M->last = 0; M->ncoll = 0; M->pn = 0;
            M->members = 0ull; M->sec = 0ull; M->tcoll = 0ull;
            M->agg[0] = M->agg[1] = M->agg[2] = 0ull;
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");   // this thread's LUT / policy chunks have landed
    }
    __syncthreads();
    {
        // per-code records from the staged policy
        const float inf = __int_as_float(0x7f800000), nan = __int_as_float(0x7fffffff);
        const float* pw = (const float*)(smem + L.surv);        // staged {wb, wu, wf, sid}[64]
        for (int c = tid; c < 256; c += kFT) {
            float4 a = make_float4(0.f, 0.f, 0.f, nan), b = make_float4(nan, 0.f, 0.f, 0.f);
            int cnto = nslots + 1, qid = -2;
            if (c == kFCodeGap || c == kFCodeFar) {
                // always into the rare path: the arrival compare (a NaN arrival is !ok anyway)
                if (SCORE) b.x = inf; else a.w = inf;
            }
            if (c < nslots) {
                // sample phase: no primary filter, no secondary filter (the sample block takes both)
                a = make_float4(pw[c], pw[64 + c], pw[128 + c], nan);
                cnto = c;
                qid = ((const int*)pw)[192 + c];
            } else if (c == kFCodeBad) {
                cnto = nslots;
                qid = -1;
            }
            b.y = __int_as_float(qid);
            b.z = __int_as_float(cnto * kFT);
            recA[c] = a;
            recB[c] = b;
        }
        if (tid == 0 && lutsz >= 0) lut[lutsz] = (unsigned char)kFCodeFar;   // lengths >= lut_size
    }
    __syncthreads();
    if (A.sample_first && tid == 0)
        for (int i = 1; i < R; i++) issue_chunk(i);
    stamp(1);

    const uint32_t gbase = A.gbase;
    const bool write_qid = A.qid_out != nullptr;
    // per-thread u8 member counters, bumped with no-return atomics on the containing word
    // (ATOMS.ADD of 1 << 8*(warp & 3)): thread (warp, lane) of row r is byte warp & 3 of
    // word r*kFCntRow + (warp >> 2)*32 + lane, so the 32 lanes of a warp hit 32 distinct
    // words (no same-word serialisation) and a row is kFT bytes (the u16 rows it replaces
    // took 25 KB more shared memory: a fourth ring stage).  A byte gains <= 4 per
    // iteration; every warp moves its bytes into ctot[] every A.cnt_flush iterations.
    uint32_t* cntw = (uint32_t*)cntb + (warp >> 2) * 32 + lane;
    const int cshift = 8 * (warp & 3);
    const uint32_t cinc = 1u << cshift;
    auto flush_counters = [&]() {       // all lanes of the warp
        for (int r = 0; r <= nslots; r++) {
            const uint32_t old = atomicAnd(cntw + r * kFCntRow, ~(0xFFu << cshift));
            const unsigned v = __reduce_add_sync(0xffffffffu, (old >> cshift) & 0xFFu);
            if (lane == 0 && v) atomicAdd(&ctot[r], v);
        }
    };
    unsigned n_exc = 0, n_ins = 0, n_gap = 0, n_bad = 0;
    u64* const rows_cta = A.rows.keys + (size_t)cta * RC;     // row of queue q: rows_cta + q*G*RC
    const size_t row_stride = (size_t)G * RC;

    auto raise_thr = [&](int q, u64 t) {   // one lane; thr64 + fast float (may lag looser, never tighter)
        if (t > *(volatile u64*)&thr64[q]) {
            atomicMax(&thr64[q], t);
            const u32 hi = (u32)(t >> 32);
            ((volatile float*)&recA[q])[3] = SCORE ? __uint_as_float(hi) : fifo_hi_to_f(hi);
        }
    };
    auto insert = [&](int q, u64 k) {
        const u32 kh = (u32)(k >> 32);       // CTA max high word (refresh board)
        if (kh > *(volatile u32*)&bmax[q * kFBoardMax]) atomicMax(&bmax[q * kFBoardMax], kh);
        EWSJF_CHECK(q >= 0 && q < nslots);
        const int pos = atomicAdd(&rcnt[q], 1);
        if (pos < RC) {
            rows_cta[q * row_stride + pos] = k;
        } else {
            const int o = atomicAdd(&M->novf, 1);
            if (o < kFOvf) { A.ovf_keys[(size_t)cta * kFOvf + o] = k; A.ovf_code[(size_t)cta * kFOvf + o] = (unsigned char)q; }
        }
        if (pos + 1 >= HWM) *(volatile int*)&M->flag = 1;
        n_ins++;
    };
    auto sec_update = [&](int q, u64 k2) {
        if (k2 > *(volatile u64*)&sec64[q]) {
            atomicMax(&sec64[q], k2);
            const u32 hi = (u32)(k2 >> 32);
            ((volatile float*)&recB[q])[0] = SCORE ? fifo_hi_to_f(hi) : __uint_as_float(hi);
        }
    };
    // queue position of a length beyond the LUT (binary search over the policy bounds), -1 = gap
    auto bsearch = [&](int b) -> int {
        int lo = 0, hi = nslots;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (P.min_len[mid] <= b) lo = mid + 1; else hi = mid;
        }
        const int i = lo - 1;
        return (i >= 0 && b < P.max_len[i]) ? i : -1;
    };

    // ---- the rare path of one request (lane-divergent)
    auto rare = [&](int c, int b, float a, float co, float sp, bool ok, int64_t idx) {
        const uint32_t gid = gbase + (uint32_t)idx;
        if (c == kFCodeFar) {
            if (b < 1) {                      // negative length (clamped to the FAR code): invalid,
                if (write_qid) A.qid_out[idx] = -1;   // already counted in the invalid row
                return;
            }
            atomicSub(cntw + nslots * kFCntRow, cinc);      // not invalid after all
            const int q = bsearch(b);
            if (q >= 0) {
                const float4 w = recA[q];
                ok = score_sp(b, a, co, HAS_COST, A.sp, w.x, w.y, w.z, &sp);
                atomicAdd(cntw + q * kFCntRow, cinc);
                if (write_qid) A.qid_out[idx] = P.sid[q];
                c = q;
            } else {
                c = kFCodeGap;
            }
        } else if (c == kFCodeGap) {
            atomicSub(cntw + nslots * kFCntRow, cinc);      // counted in the invalid row by the body
        }
        if (c == kFCodeGap) {
            const unsigned long long p = atomicAdd(&A.ctr->gap_count, 1ull);
            if (p < (unsigned long long)A.gap_cap) {
                GapEntry e;
                e.gid = gid; e.len = b; e.arrival = a;
                e.cost = HAS_COST ? co : __int_as_float(0x7fc00000);
                A.gap[p] = e;
            }
            n_gap++;
            return;
        }
        if (c >= nslots) return;   // bad length / padding
        if (!ok) { atomicSub(cntw + c * kFCntRow, cinc); n_exc++; return; }
        const u64 ks = score_key(sp, gid), kf = fifo_key(a, gid);
        const u64 k1 = SCORE ? ks : kf, k2 = SCORE ? kf : ks;
        if (k1 >= *(volatile u64*)&thr64[c]) insert(c, k1);
        sec_update(c, k2);
    };

    // ---- one tile of 128 requests (4 per lane); sample: keep the keys, fill the sample maxima
    u64 skey[4] = {0ull, 0ull, 0ull, 0ull};
    int scode[4] = {kFCodeNone, kFCodeNone, kFCodeNone, kFCodeNone};
    auto body = [&](auto full_tag, auto sample_tag, auto wait_tag, int64_t t, int st) {
        constexpr bool FULL = decltype(full_tag)::value;
        constexpr bool SAMPLE = decltype(sample_tag)::value;
        const int64_t i0 = t * kFTile + 4 * lane;
        int b[4];
        float a[4], co[4];
        int nv = 4;
        if (FULL) {            // the caller has waited for the stage
            const int4 bv = ((const int4*)stage(st, 0))[lane];
            const float4 av = ((const float4*)stage(st, 1))[lane];
            float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (HAS_COST) cv = ((const float4*)stage(st, 2))[lane];
            b[0] = bv.x; b[1] = bv.y; b[2] = bv.z; b[3] = bv.w;
            a[0] = av.x; a[1] = av.y; a[2] = av.z; a[3] = av.w;
            co[0] = cv.x; co[1] = cv.y; co[2] = cv.z; co[3] = cv.w;
        } else {                              // the ragged last tile: direct loads
            nv = (int)max((int64_t)0, min((int64_t)4, A.n - i0));
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const bool v = j < nv;
                b[j] = v ? __ldg(A.len + i0 + j) : 0;
                a[j] = v ? __ldg(A.arrival + i0 + j) : 0.f;
                co[j] = (HAS_COST && v) ? __ldg(A.cost + i0 + j) : 0.f;
            }
        }
        int code[4];
        float sp[4];
        int qo[4];
        bool okv[4];
        unsigned pm = 0u;             // request slots j of this lane that need the rare path
#pragma unroll
        for (int j = 0; j < 4; j++) {
            // lengths < 0 clamp to lut_size (FAR: the rare path sorts them out); lut[0] = bad
            const int c = (FULL || j < nv) ? (int)lut[min((unsigned)b[j], (unsigned)lutsz)] : kFCodeNone;
            code[j] = c;
            // member counter row straight from the code (no wait on the record load):
            // rows 0..nslots-1 members, nslots every other code (invalid length, and the
            // FAR / GAP codes, which the rare path takes back out); padding uncounted
            const int crow = min(c, nslots);
            if (FULL || j < nv) atomicAdd(cntw + crow * kFCntRow, cinc);
            const float4 w = recA[c];
            const float4 r2 = recB[c];
            const bool ok = score_sp(b[j], a[j], co[j], HAS_COST, A.sp, w.x, w.y, w.z, &sp[j]);
            okv[j] = ok;
            qo[j] = __float_as_int(r2.y);
            const float f1 = SCORE ? sp[j] : a[j];
            const float f2 = SCORE ? a[j] : sp[j];
            const bool p1 = SCORE ? (f1 >= w.w) : (f1 <= w.w);
            const bool p2 = SCORE ? (f2 <= r2.x) : (f2 >= r2.x);
            bool pj = p1 || p2 || !ok;
            if (SAMPLE) pj = pj && !(c < nslots && ok);    // members of the sample: the sample block
            pm |= pj ? (1u << j) : 0u;
        }
        if (write_qid) {
            if (FULL) {
                __stcs((int4*)(A.qid_out + i0), make_int4(qo[0], qo[1], qo[2], qo[3]));
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (j < nv) A.qid_out[i0 + j] = qo[j];
            }
        }
        if (SAMPLE) {
            // sample maxima (board) and exact secondary max of every valid member
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int c = code[j];
                const bool mem = c < nslots && okv[j];
                const uint32_t gid = gbase + (uint32_t)(i0 + j);
                const u64 ks = score_key(sp[j], gid), kf = fifo_key(a[j], gid);
                const u64 k1 = SCORE ? ks : kf, k2 = SCORE ? kf : ks;
                skey[j] = mem ? k1 : 0ull;
                scode[j] = mem ? c : kFCodeNone;
                if (mem) {
                    // board: native u32 atomicMax of the high word; exact secondary: a
                    // 64-bit CAS only when the high word ties or beats the current one
                    const u32 h1 = (u32)(k1 >> 32);
                    if (h1 > *(volatile u32*)&bmax[c * kFBoardMax]) atomicMax(&bmax[c * kFBoardMax], h1);
                    if (k2 > *(volatile u64*)&sec64[c]) atomicMax(&sec64[c], k2);
                }
            }
        }
        // the rare path: one inline copy, each lane walks its own flagged slots (the
        // operands of slot j picked by selects; 4 inlined copies made the loop body too
        // large for the instruction cache)
        while (__any_sync(0xffffffffu, pm != 0u)) {
            if (pm) {
                const int j = __ffs(pm) - 1;
                pm &= pm - 1u;
                const int bj = j == 0 ? b[0] : (j == 1 ? b[1] : (j == 2 ? b[2] : b[3]));
                const float aj = j == 0 ? a[0] : (j == 1 ? a[1] : (j == 2 ? a[2] : a[3]));
                const float cj = j == 0 ? co[0] : (j == 1 ? co[1] : (j == 2 ? co[2] : co[3]));
                const float sj = j == 0 ? sp[0] : (j == 1 ? sp[1] : (j == 2 ? sp[2] : sp[3]));
                const int dj = j == 0 ? code[0] : (j == 1 ? code[1] : (j == 2 ? code[2] : code[3]));
                const bool oj = j == 0 ? okv[0] : (j == 1 ? okv[1] : (j == 2 ? okv[2] : okv[3]));
                rare(dj, bj, aj, cj, sj, oj, i0 + j);
            }
        }
    };
    // release stage st of iteration i (lane 0, after the warp's last read of it): the
    // last of the kFW warps refills it with iteration i + R
    auto release = [&](int st, int i) {
        __syncwarp();
        if (lane == 0) {
            const unsigned o = atomicAdd(&relc[st], 1u);
            if (o % kFW == kFW - 1) issue_chunk(i + R);
        }
    };
    // ---- collective: cut every row at/over its high-water mark to its exact K-th key
    auto collective = [&]() {
        const unsigned long long tc = dbg ? fgtime() : 0ull;
        fbar(1);
        const int no = min(*(volatile int*)&M->novf, kFOvf);
        const u64* ok_ = A.ovf_keys + (size_t)cta * kFOvf;
        const unsigned char* oc_ = A.ovf_code + (size_t)cta * kFOvf;
        for (int q = 0; q < nslots; q++) {
            const int rc = rcnt[q];
            fbar(1);                          // everyone has read rcnt[q] before it changes
            if (rc < HWM) continue;
            const int nr = min(rc, RC);
            u64* row = rows_cta + q * row_stride;
            auto fe = [&](auto f) {
                for (int j = tid; j < nr; j += kFT) f(__ldcg(row + j));
                for (int j = tid; j < no; j += kFT)
                    if (oc_[j] == q) f(__ldcg(ok_ + j));
            };
            const u64 t = block_kth(fe, K, hist, M);
            const int nk = block_collect(fe, t, surv, EWSJF_MAX_K, M);
            for (int j = tid; j < nk; j += kFT) row[j] = surv[j];
            if (tid == 0) {
                rcnt[q] = nk;
                raise_thr(q, t);
                atomicMax(&A.gthr[q], t);
            }
            fbar(1);
        }
        if (tid == 0) {
            M->novf = 0;
            M->flag = 0;
            M->ncoll++;
            if (dbg) M->tcoll += fgtime() - tc;
        }
        fbar(1);
    };

    // ---- sample tile, board, bound
    if (dbg && tid == 0) A.dbg[cta * kDbgStride + 25] = fgtime();
    bool more = true;                     // iteration 0 is not the end of this CTA's chunks
    {
        mbar_wait(&fullb[0], 0u);
        if (dbg && tid == 0) A.dbg[cta * kDbgStride + 15] = fgtime();   // the sample chunk has landed
        const int64_t c = *(volatile int64_t*)&schunk[0];
        if (c < 0) more = false;
        else {
            if (c < nfullc) body(std::true_type(), std::true_type(), std::integral_constant<int, 0>(), c * kFW + warp, 0);
            else body(std::false_type(), std::true_type(), std::integral_constant<int, 0>(), c * kFW + warp, 0);
            release(0, 0);
        }
    }
    if (dbg && tid == 0) A.dbg[cta * kDbgStride + 26] = fgtime();
    __syncthreads();
    stamp(2);
    const int bm = A.board_m;
    if (bm > 0) {
        // further board rounds (m > 1): the largest key below the previous round's
        for (int m = 1; m < bm; m++) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int c = scode[j];
                if (c < nslots) {
                    const u32 prev = bmax[c * kFBoardMax + m - 1];
                    const u32 k = (u32)(skey[j] >> 32);
                    if (k < prev && k > *(volatile u32*)&bmax[c * kFBoardMax + m]) atomicMax(&bmax[c * kFBoardMax + m], k);
                }
            }
            __syncthreads();
        }
        for (int i = tid; i < nslots * bm; i += kFT) {
            const int q = i / bm, m = i % bm;
            A.board[((size_t)q * G + cta) * bm + m] = (u64)bmax[q * kFBoardMax + m] << 32;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            // publish, then wait until every CTA of this launch has published
            // (monotone ticket: generation = ticket / G)
            const unsigned tk = atomicAdd(&A.ctr->pub, 1u);
            const unsigned target = (tk / (unsigned)G + 1u) * (unsigned)G;
            if (dbg) A.dbg[cta * kDbgStride + 13] = fgtime();
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&A.ctr->pub) : "memory");
                if ((int)(v - target) < 0) __nanosleep(32);
            } while ((int)(v - target) < 0);
        }
        __syncthreads();
        // every CTA turns the complete board into the same bounds (one warp per
        // queue): the K-th largest high word t of the G*bm published keys, so
        // >= K distinct real requests have keys >= (t << 32) -- a valid bound
        const int nb = G * bm;
        auto bounds = [&](auto regs_tag) {
            constexpr int RR = decltype(regs_tag)::value;
            for (int q = warp; q < nslots; q += 2 * kFW) {
                const int q1 = q + kFW;
                u32 v0[RR], v1[RR];
#pragma unroll
                for (int r = 0; r < RR; r++) {
                    const int j = lane + 32 * r;
                    v0[r] = j < nb ? (u32)(__ldcg(A.board + (size_t)q * nb + j) >> 32) : 0u;
                    v1[r] = (j < nb && q1 < nslots) ? (u32)(__ldcg(A.board + (size_t)q1 * nb + j) >> 32) : 0u;
                }
                u32 t[2];
                warp_kth_hi2<RR>(v0, v1, K, t);
                if (lane == 0) {
                    thr64[q] = (u64)t[0] << 32;
                    if (cta == 0 && t[0]) atomicMax(&A.gthr[q], (u64)t[0] << 32);
                    if (q1 < nslots) {
                        thr64[q1] = (u64)t[1] << 32;
                        if (cta == 0 && t[1]) atomicMax(&A.gthr[q1], (u64)t[1] << 32);
                    }
                }
            }
        };
        if (nb <= 160) bounds(std::integral_constant<int, 5>());
        else bounds(std::integral_constant<int, kFBoardRegs>());
        stamp(14);
        __syncthreads();
    }
    // thresholds from the bound, fast secondary from the sample's exact max
    for (int q = tid; q < nslots; q += kFT) {
        const u64 g = thr64[q];
        const u32 hi = (u32)(g >> 32);
        const float inf = __int_as_float(0x7f800000);
        recA[q].w = SCORE ? __uint_as_float(hi) : (g ? fifo_hi_to_f(hi) : inf);
        const u64 s = sec64[q];
        const u32 sh = (u32)(s >> 32);
        recB[q].x = SCORE ? (s ? fifo_hi_to_f(sh) : inf) : __uint_as_float(sh);
        if (A.diag & 1) {   // timing diagnostic only (EWSJF_DIAG=1): no candidate ever passes (wrong outputs)
            recA[q].w = SCORE ? inf : -inf;
            recB[q].x = SCORE ? -inf : inf;
            thr64[q] = ~0ull;
            sec64[q] = ~0ull;
        }
    }
    __syncthreads();
    stamp(3);
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int c = scode[j];
        if (c < nslots && skey[j] >= thr64[c]) insert(c, skey[j]);
    }
    __syncwarp();

    // ---- stream the rest of the block; collectives on demand
    // Progressive bound: at its checkpoint tile (1/16 .. 3/4 of the block) warp
    // w < 6 publishes the CTA's running max key of every queue to the refresh
    // board and turns the board's current content into a bound for one queue
    // (K-th largest high word of the CTA maxima present: K distinct real keys
    // lie above it, so it is valid however incomplete the board is).  No CTA
    // waits; the bounds reach the others through gthr.
    int chk = -1;
    if (A.refresh && warp < 6) {
        const int num = warp == 0 ? 1 : warp == 1 ? 2 : warp == 2 ? 4 : warp == 3 ? 6 : warp == 4 ? 8 : 12;
        chk = ((int)((nchunks + G - 1) / G) * num) >> 4;
        if (chk < 1) chk = -1;
    }
    auto refresh = [&]() {
        u64* rb = A.rboard;
        for (int q = lane; q < nslots; q += 32) rb[(size_t)q * G + cta] = (u64)(*(volatile u32*)&bmax[q * kFBoardMax]) << 32;
        __syncwarp();
        const int qa = (cta * 12 + warp * 2) % nslots, qb = (qa + 1) % nslots;
        u32 va[5], vb[5];
#pragma unroll
        for (int r = 0; r < 5; r++) {
            const int j = lane + 32 * r;
            va[r] = j < G ? (u32)(__ldcg(rb + (size_t)qa * G + j) >> 32) : 0u;
            vb[r] = j < G ? (u32)(__ldcg(rb + (size_t)qb * G + j) >> 32) : 0u;
        }
        u32 t[2];
        warp_kth_hi2<5>(va, vb, K, t);
        if (lane == 0) {
            if (t[0]) { atomicMax(&A.gthr[qa], (u64)t[0] << 32); raise_thr(qa, (u64)t[0] << 32); }
            if (t[1]) { atomicMax(&A.gthr[qb], (u64)t[1] << 32); raise_thr(qb, (u64)t[1] << 32); }
        }
    };
    // pick up raised global bounds: one queue per warp every 4 tiles, the L2 load
    // issued one poll ahead (a global access waits behind the SM's ~100 KB of
    // streaming loads in flight, ~2 us)
    int rq = warp % max(nslots, 1);
    u64 gpoll = (lane == 0 && nslots > 0) ? __ldcg(&A.gthr[rq]) : 0ull;
    // the streaming loop with the ring depth fixed at compile time (stage / phase counters
    // without divisions)
    auto stream = [&](auto r_tag) {
        constexpr int RR = decltype(r_tag)::value;
        __syncwarp();
        int st = 1 % RR;
        uint32_t ph = (1 / RR) & 1;
        int since_flush = 1;            // the sample iteration
        for (int i = 1; more; i++) {
            if (*(volatile int*)&M->flag) collective();
            mbar_wait(&fullb[st], ph);
            const int64_t c = *(volatile int64_t*)&schunk[st];
            if (c < 0) break;
            const int64_t t = c * kFW + warp;
            if (c < nfullc) body(std::true_type(), std::false_type(), std::integral_constant<int, 0>(), t, st);
            else body(std::false_type(), std::false_type(), std::integral_constant<int, 0>(), t, st);
            release(st, i);
            if (++st == RR) { st = 0; ph ^= 1u; }
            if (++since_flush == A.cnt_flush) { flush_counters(); since_flush = 0; }
            if (i == chk) refresh();
            if (A.refresh && (i & 3) == 0 && nslots > 0) {   // the global bounds only move with the refresh
                                                              // (or a rare collective: its CTA's own bound rises)
                if (lane == 0) {
                    if (gpoll) raise_thr(rq, gpoll);
                    rq += kFW;
                    if (rq >= nslots) rq = (rq - nslots) % nslots;
                    gpoll = __ldcg(&A.gthr[rq]);
                }
            }
        }
    };
    if (R == 2) stream(std::integral_constant<int, 2>());
    else if (R == 3) stream(std::integral_constant<int, 3>());
    else stream(std::integral_constant<int, 4>());
    // done: keep serving collectives until every warp is done (a flag raised by
    // this warp is handled before its ndone increment; ndone is read before the flag)
    __syncwarp();
    if (lane == 0) { __threadfence_block(); atomicAdd(&M->ndone, 1); }
    for (;;) {
        int f = 0, dn = 0;
        if (lane == 0) {
            dn = *(volatile int*)&M->ndone;
            __threadfence_block();
            f = *(volatile int*)&M->flag;
        }
        f = __shfl_sync(0xffffffffu, f, 0);
        dn = __shfl_sync(0xffffffffu, dn, 0);
        if (f) { collective(); continue; }
        if (dn == kFW) break;
        __nanosleep(256);      // a done warp must not steal issue slots from the streaming ones
    }
    __syncthreads();
    if (tid == 0)      // the ring's shared memory is reused by the merge
        for (int st = 0; st < R; st++)
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&fullb[st])) : "memory");
    stamp(4);

    // ---- per-CTA rows: cut to the best bound known now (this CTA's threshold or the
    // global one, max of the two) -- the merge then reads a few keys per row instead of
    // every insert (the dominant queue's merge read ~400 per CTA, ~10 us); rows of <= 32
    // keys are left as they are (the merge loads those whole and filters them itself) --
    // then count (<= RC, no overflow pending), members, secondary, in one pass per queue
    for (int q = warp; q < nslots; q += kFW) {
        const int nr = min(rcnt[q], RC);
        int wpos = nr;
        if (nr > 32) {
            u64 g = __ldcg(&A.gthr[q]);
            const u64 tl = thr64[q];
            g = g > tl ? g : tl;
            u64* row = rows_cta + q * row_stride;
            wpos = 0;
            for (int base = 0; base < nr; base += 32 * 16) {
                u64 kv[16];
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    const int j = base + u * 32 + lane;
                    kv[u] = j < nr ? __ldcg(row + j) : 0ull;
                }
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    const bool keep = kv[u] != 0ull && kv[u] >= g;
                    const unsigned bal = __ballot_sync(0xffffffffu, keep);
                    if (keep) row[wpos + __popc(bal & ((1u << lane) - 1u))] = kv[u];
                    wpos += __popc(bal);
                }
            }
        }
        const uint32_t* c32 = (const uint32_t*)(cntb + (size_t)q * kFT);
        unsigned long long mm = lane == 0 ? ctot[q] : 0u;
#pragma unroll
        for (int k = 0; k < kFCntRow / 32; k++) mm += __dp4a(c32[lane + 32 * k], 0x01010101u, 0u);
        for (int o = 16; o; o >>= 1) mm += __shfl_xor_sync(0xffffffffu, mm, o);
        if (lane == 0) {
            const size_t r = (size_t)q * G + cta;
            A.rows.cnt[r] = wpos;
            A.rows.members[r] = (int64_t)mm;
            A.rows.sec[r] = sec64[q];
        }
    }
    if (dbg && tid == 0) A.dbg[cta * kDbgStride + 28] = fgtime();
    if (dbg && tid == 0) A.dbg[cta * kDbgStride + 29] = fgtime();
    {
        // invalid lengths (counter row nslots) + excluded + diagnostics
        unsigned long long bad = n_bad;
        if (warp == 0) {
            const uint32_t* c32 = (const uint32_t*)(cntb + (size_t)nslots * kFT);
            if (lane == 0) bad += ctot[nslots];
            for (int k = lane; k < kFCntRow; k += 32) bad += __dp4a(c32[k], 0x01010101u, 0u);
        }
        unsigned long long ex = n_exc, ins = n_ins;
        for (int o = 16; o; o >>= 1) {
            bad += __shfl_xor_sync(0xffffffffu, bad, o);
            ex += __shfl_xor_sync(0xffffffffu, ex, o);
            ins += __shfl_xor_sync(0xffffffffu, ins, o);
        }
        // CTA totals first (smem), then one global atomic per CTA and counter
        if (lane == 0) {
            if (bad) atomicAdd(&M->agg[0], bad);
            if (ex) atomicAdd(&M->agg[1], ex);
            if (ins) atomicAdd(&M->agg[2], ins);
        }
        __syncthreads();
        if (tid == 0) {
            if (M->agg[0]) atomicAdd(&A.ctr->n_invalid, M->agg[0]);
            if (M->agg[1]) atomicAdd(&A.ctr->n_excluded, M->agg[1]);
            if (M->agg[2]) atomicAdd(&A.ctr->dbg_inserted, M->agg[2]);
        }
        if (tid == 0 && M->ncoll) atomicAdd(&A.ctr->dbg_compactions, (unsigned long long)M->ncoll);
        if (dbg && tid == 0) { A.dbg[cta * kDbgStride + 8] = (unsigned long long)M->ncoll; A.dbg[cta * kDbgStride + 9] = M->tcoll; }
    }
    (void)n_gap;
    __syncthreads();
    if (dbg && tid == 0) A.dbg[cta * kDbgStride + 30] = fgtime();
    if (tid == 0) __threadfence();   // cumulative over the CTA's writes ordered by the bar.sync (as a grid sync)
    stamp(5);
    if (A.merge == 0) return;

    // ---- grid barrier (monotone ticket: generation = ticket / G)
    if (tid == 0) {
        const unsigned tk = atomicAdd(&A.ctr->done, 1u);
        const unsigned target = (tk / (unsigned)G + 1u) * (unsigned)G;
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&A.ctr->done) : "memory");
            if ((int)(v - target) < 0) __nanosleep(32);
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
    stamp(6);
    if (cta == 0 && tid == 0) A.ctr->ftiles = 0ull;   // every chunk claim of this launch is done
    if (dbg && tid == 0) A.dbg[cta * kDbgStride + 24] = fgtime();
    if (A.refresh)   // nobody reads the refresh board past the barrier: clear this CTA's column for the next tick
        for (int q = tid; q < nslots; q += kFT) A.rboard[(size_t)q * G + cta] = 0ull;

    // The fast merge's loads (this queue's rows, its bound) are issued together with
    // the gap-count check, so the common case pays one round trip, not two.
    const int q = cta;
    // 8 threads per row, 16 bytes each per load: a row's first 32 keys are two
    // coalesced 128-byte segments (rows kFT/8 apart in two passes, G <= 2 * kFT/8)
    constexpr int kRowT = 8, kRowsPass = kFT / kRowT;
    const int t8 = tid & (kRowT - 1), rg = tid / kRowT;
    int ncv[2] = {0, 0};
    u64 kv[8];
    unsigned long long mm = 0;
    u64 sk = 0ull;
#pragma unroll
    for (int ps = 0; ps < 2; ps++) {
        const int rrow = rg + ps * kRowsPass;
#pragma unroll
        for (int u = 0; u < 4; u++) kv[4 * ps + u] = 0ull;
        if (q < nslots && rrow < G) {
            // one round trip: count, members and secondary and, speculatively, the first 32
            // keys (masked by the count below; the rows were cut to the end-of-stream bound)
            const size_t rr = (size_t)q * G + rrow;
            ncv[ps] = __ldcg(&A.rows.cnt[rr]);
            if (t8 == 0) { mm += (unsigned long long)__ldcg(&A.rows.members[rr]); const u64 s2 = __ldcg(&A.rows.sec[rr]); sk = s2 > sk ? s2 : sk; }
            const ulonglong2* rk2 = (const ulonglong2*)(A.rows.keys + rr * RC);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const ulonglong2 v = __ldcg(rk2 + t8 + kRowT * h);
                kv[4 * ps + 2 * h] = v.x;
                kv[4 * ps + 2 * h + 1] = v.y;
            }
        }
    }
    u64 thr = q < nslots ? __ldcg(&A.gthr[q]) : 0ull;
    const unsigned long long graw = __ldcg(&A.ctr->gap_count);
    if (dbg && tid == 0) A.dbg[cta * kDbgStride + 23] = fgtime() ^ (unsigned long long)(graw == 0x123456789ull);
    if (graw > 0 || A.merge == 2) {
        // gap requests (App. D, Alg. 2) / exchange record: the general merge
        if (A.merge == 2) merge_phase<MERGE_IN_ROWS, MERGE_OUT_EXCHANGE, HAS_COST, kFT>(MA, P, smem);
        else merge_phase<MERGE_IN_ROWS, MERGE_OUT_FINAL, HAS_COST, kFT>(MA, P, smem);
        stamp(7);
        return;
    }

    // ---- fast merge: CTA q merges queue q (no gap requests in this tick)
    if (q < nslots) {
        // the whole shared memory is free now: [rowoff | pool]
        int* rowoff = (int*)(smem + L.cnt);                  // [G + 1]
        u64* pool = (u64*)(smem + L.ring);
        // the candidate pool takes the ring region only (the control block M, hist and
        // surv that follow it are still in use): >= 2 stages x 2 arrays x 16 warps x 512 B
        const int pcap = (int)((L.bars - L.ring) / 8);
        constexpr int kChunk = 3 * kFT;                       // candidates scanned per round
        if (tid == 0) { M->pn = 0; M->members = 0ull; M->sec = 0ull; M->ncoll = 0; M->maxnc = 0; }
        __syncthreads();
        if (dbg && tid == 0) A.dbg[cta * kDbgStride + 21] = fgtime();
        {
            for (int o = 16; o; o >>= 1) {
                mm += __shfl_xor_sync(0xffffffffu, mm, o);
                const u64 so = shfl_xor_u64(sk, o);
                sk = so > sk ? so : sk;
            }
            if (lane == 0) {
                if (mm) atomicAdd(&M->members, mm);
                if (sk) atomicMax(&M->sec, sk);
            }
            if (t8 == 0) {
#pragma unroll
                for (int ps = 0; ps < 2; ps++) {
                    const int rrow = rg + ps * kRowsPass, nc = ncv[ps];
                    if (rrow >= G) continue;
                    if (nc) {
                        atomicAdd(&M->ncoll, nc);      // total candidates (ncoll reused)
                        atomicMax(&M->maxnc, nc);
                    }
                    rowoff[rrow + 1] = nc;             // counts for the prefix of the chunked path
                }
            }
            if (dbg && tid == 0) A.dbg[cta * kDbgStride + 22] = fgtime();
        }
        __syncthreads();
        if (dbg && tid == 0) A.dbg[cta * kDbgStride + 20] = fgtime();
        // SCORE head (the FIFO key's max): its request's fields, loaded now and used at the end
        int h_len = 0;
        float h_arr = 0.f, h_cost = 0.f;
        if (SCORE && tid == 0 && M->sec) {
            const int64_t li = (int64_t)key_gid(M->sec) - (int64_t)gbase;
            h_len = __ldg(A.len + li);
            h_arr = __ldg(A.arrival + li);
            if (HAS_COST) h_cost = __ldg(A.cost + li);
        }
        const int total = M->ncoll;
        int pn = 0;
        if (M->maxnc <= 2 * 2 * kRowT) {       // every row fully loaded already
            // one shared atomic per warp (a single counter hit by every passing key
            // serialised ~100 atomics, ~1 us)
            unsigned pmask = 0u;
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int ps = u >> 2, j = 2 * t8 + 2 * kRowT * ((u >> 1) & 1) + (u & 1);
                pmask |= (j < ncv[ps] && kv[u] && kv[u] >= thr) ? (1u << u) : 0u;
            }
            const int c = __popc(pmask);
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int wbase = 0;
            if (lane == 31 && incl) wbase = atomicAdd(&M->pn, incl);
            wbase = __shfl_sync(0xffffffffu, wbase, 31);
            int o = wbase + incl - c;
            EWSJF_CHECK(o + c <= pcap);
#pragma unroll
            for (int u = 0; u < 8; u++)
                if (pmask & (1u << u)) pool[o++] = kv[u];
            __syncthreads();
            pn = M->pn;
            __syncthreads();
        } else {
            // long rows: prefix of the counts (already in rowoff[1..G]), then rounds of
            // kChunk candidates over all threads with cuts to the top K
            {
                const int c = tid < G ? rowoff[tid + 1] : 0;
                int incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += u;
                }
                if (lane == 31) hist[warp] = (unsigned)incl;
                __syncthreads();
                int woff = 0;
                for (int w = 0; w < warp; w++) woff += (int)hist[w];
                __syncthreads();
                if (tid < G) rowoff[tid + 1] = woff + incl;
                if (tid == 0) rowoff[0] = 0;
            }
            __syncthreads();
            for (int base = 0; base < total; base += kChunk) {
                u64 kx[kChunk / kFT];
#pragma unroll
                for (int u = 0; u < kChunk / kFT; u++) {
                    const int e = base + tid + kFT * u;
                    kx[u] = 0ull;
                    if (e < total) {
                        int lo = 0, hi = G;                      // row r: rowoff[r] <= e < rowoff[r + 1]
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (rowoff[mid] <= e) lo = mid; else hi = mid;
                        }
                        kx[u] = __ldcg(A.rows.keys + ((size_t)q * G + lo) * RC + (e - rowoff[lo]));
                    }
                }
#pragma unroll
                for (int u = 0; u < kChunk / kFT; u++)
                    if (kx[u] && kx[u] >= thr) {
                        const int o = atomicAdd(&M->pn, 1);
                        EWSJF_CHECK(o < pcap);
                        pool[o] = kx[u];
                    }
                __syncthreads();
                pn = M->pn;
                __syncthreads();
                if (pn > pcap - kChunk && base + kChunk < total) {
                    auto fe = [&](auto f) { for (int j = tid; j < pn; j += kFT) f(pool[j]); };
                    const u64 t = block_kth(fe, K, hist, M);
                    const int nk = block_collect(fe, t, surv, EWSJF_MAX_K, M);
                    for (int j = tid; j < nk; j += kFT) pool[j] = surv[j];
                    if (tid == 0) M->pn = nk;
                    thr = t;
                    __syncthreads();
                    pn = nk;
                }
            }
        }
        if (dbg && tid == 0) { A.dbg[cta * kDbgStride + 16] = fgtime(); A.dbg[cta * kDbgStride + 17] = (unsigned long long)pn; }
        const int ns = min(pn, K);
        if (pn <= kFT) {
            // small pool: one counting pass ranks every candidate (keys are unique),
            // rank < K are the top K already in order -- no radix select, no sort.
            // tpc = 4 / 2 / 1 threads per candidate (pools of <= 192 / 384 / 768), each
            // counting the keys above it in every tpc-th 16-byte pair; pool padded with
            // zeros.  (Up to 128 only, the merge fell back to the 8-pass radix select
            // for the ~180 candidates of the dominant queue: 3.1 vs ~1 us.)
            const int tpc = pn <= kFT / 4 ? 4 : (pn <= kFT / 2 ? 2 : 1);
            const int pn8 = (pn + 7) & ~7;
            if (tid >= pn && tid < pn8) pool[tid] = 0ull;
            __syncthreads();
            const int ci = tid / tpc, part = tid - ci * tpc;
            const u64 k0 = ci < pn ? pool[ci] : 0ull;
            int r0 = 0;
            if (ci < pn) {
                int r1 = 0;
                int j = 2 * part;
                for (; j + 2 * tpc < pn8; j += 4 * tpc) {          // two pairs in flight
                    const ulonglong2 x = *(const ulonglong2*)(pool + j);
                    const ulonglong2 y = *(const ulonglong2*)(pool + j + 2 * tpc);
                    r0 += (x.x > k0) + (x.y > k0);
                    r1 += (y.x > k0) + (y.y > k0);
                }
                if (j < pn8) {
                    const ulonglong2 x = *(const ulonglong2*)(pool + j);
                    r0 += (x.x > k0) + (x.y > k0);
                }
                r0 += r1;
            }
            if (tpc >= 2) r0 += __shfl_xor_sync(0xffffffffu, r0, 1);
            if (tpc == 4) r0 += __shfl_xor_sync(0xffffffffu, r0, 2);
            __syncthreads();
            if (ci < pn && part == 0 && r0 < K) surv[r0] = k0;
            __syncthreads();
        } else {
            auto fe = [&](auto f) { for (int j = tid; j < pn; j += kFT) f(pool[j]); };
            const u64 t = block_kth(fe, K, hist, M);
            block_collect(fe, t, surv, EWSJF_MAX_K, M);
            // surv holds the K best keys (any order): rank sort
            u64 myk = 0ull;
            int myr = -1;
            if (tid < ns) {
                myk = surv[tid];
                int r = 0;
                for (int j = 0; j < ns; j++) r += surv[j] > myk;
                myr = r;
            }
            __syncthreads();
            if (tid < ns) surv[myr] = myk;
            __syncthreads();
        }
        if (dbg && tid == 0) A.dbg[cta * kDbgStride + 18] = fgtime();
        const float qi = (float)(q + 1);
        const float4 wq = recA[q];        // the staged weights (rec is untouched by the merge)
        const float wb = wq.x, wu = wq.y, wf = wq.z;
        auto payload = [&](u64 k) -> float {   // s' of the request with key k
            if (SCORE) return key_sp(k);
            const int64_t li = (int64_t)key_gid(k) - (int64_t)gbase;
            float s = 0.f;
            score_sp(__ldg(A.len + li), __ldg(A.arrival + li), HAS_COST ? __ldg(A.cost + li) : 0.f, HAS_COST, A.sp,
                     wb, wu, wf, &s);
            return s;
        };
        for (int r = tid; r < K; r += kFT) {
            const size_t o = (size_t)q * K + r;
            if (r < ns) {
                A.topk_id[o] = (int64_t)key_gid(surv[r]);
                A.topk_score[o] = qi * payload(surv[r]);
            } else {
                A.topk_id[o] = -1;
                A.topk_score[o] = 0.f;
            }
        }
        if (tid == 0) {
            const unsigned long long members = M->members;
            const u64 sec = M->sec;
            A.count[q] = (int64_t)members;
            if (members == 0 || ns == 0) {
                A.head_id[q] = -1; A.head_score[q] = 0.f; A.max_score[q] = 0.f;
            } else if (SCORE) {
                float s = 0.f;
                score_sp(h_len, h_arr, h_cost, HAS_COST, A.sp, wb, wu, wf, &s);
                A.head_id[q] = (int64_t)key_gid(sec);
                A.head_score[q] = qi * s;
                A.max_score[q] = qi * key_sp(surv[0]);
            } else {
                A.head_id[q] = (int64_t)key_gid(surv[0]);
                A.head_score[q] = qi * payload(surv[0]);
                A.max_score[q] = qi * key_sp(sec);
            }
            A.gthr[q] = 0ull;
        }
        if (dbg && tid == 0) A.dbg[cta * kDbgStride + 19] = fgtime();
    }
    stamp(7);
    // ---- last CTA: Alg. 1 ArgMax (ties -> lowest position, R24), summary, counter reset
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const unsigned tk = atomicAdd(&A.ctr->ticket, 1u);
        M->last = tk == (unsigned)(G - 1);
    }
    __syncthreads();
    if (!M->last || warp != 0) return;
    __threadfence();
    u64 best = 0ull;
    for (int p = lane; p < nslots; p += 32)
        if (__ldcg(&A.count[p]) > 0) {
            const u64 k = ((u64)ord_f32(__ldcg(&A.head_score[p])) << 32) | (u64)(~(u32)p);
            best = k > best ? k : best;
        }
    best = warp_max_u64(best);
    if (lane != 0) return;
    const long long inv = (long long)__ldcg(&A.ctr->n_invalid), exc = (long long)__ldcg(&A.ctr->n_excluded);
    if (A.summary) {
        ewsjf_summary sm;
        sm.n_queues = nslots;
        sm.primary = best ? (int)(~(u32)best) : -1;
        sm.n_invalid = inv;
        sm.n_excluded = exc;
        sm.n_gap = 0;
        sm.n_bubbles = 0;
        sm.n_dropped = 0;
        sm.status = (inv || exc) ? EWSJF_ERR_DOMAIN : EWSJF_OK;
        sm.pad = 0;
        *A.summary = sm;
    }
    A.ctr->n_invalid = 0;
    A.ctr->n_excluded = 0;
    A.ctr->gap_count = 0;
    A.ctr->ticket = 0;
}

int64_t merge_smem_total(int in_mode);

template <int MO, bool C>
static cudaError_t launch_f(const FArgs& A, const Policy* P, const MergeArgs& MA, int grid, cudaStream_t st) {
    const int64_t ls = fsmem_layout(C, A.lut_size, A.nslots, A.stages).total;
    const int64_t lm = A.merge ? merge_smem_total(MERGE_IN_ROWS) : 0;
    const int64_t smem = ls > lm ? ls : lm;
    auto k = ftick_kernel<MO, C>;
    // the attribute only grows per device (a host call per launch otherwise)
    static int64_t attr[32] = {0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 32 || attr[dev] < smem) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 32) attr[dev] = smem;
    }
    void* args[] = {(void*)&A, (void*)&P, (void*)&MA};   // &P: address of the device pointer
    return cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kFT), args, (size_t)smem, st);
}

cudaError_t launch_ftick(const FArgs& A, const Policy* P, const MergeArgs& MA, bool has_cost, int grid,
                         cudaStream_t st) {
    if (A.sp.mode == EWSJF_SELECT_FIFO)
        return has_cost ? launch_f<EWSJF_SELECT_FIFO, true>(A, P, MA, grid, st)
                        : launch_f<EWSJF_SELECT_FIFO, false>(A, P, MA, grid, st);
    return has_cost ? launch_f<EWSJF_SELECT_SCORE, true>(A, P, MA, grid, st)
                    : launch_f<EWSJF_SELECT_SCORE, false>(A, P, MA, grid, st);
}

}  // namespace ewsjf
