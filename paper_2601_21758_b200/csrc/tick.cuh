// tick.cuh — argument blocks shared by tick.cu and api.cu.
#pragma once
#include "common.cuh"

namespace ewsjf {

// One gap-falling request, captured by the partial pass for Alg. 2 (App. D).
struct GapEntry {
    uint32_t gid;        // global id
    int32_t len;
    float arrival;
    float cost;          // NaN if the pool has no cost field
};

// Scratch produced by the partial pass ("CTA rows"), consumed by the merge.
struct Rows {
    u64* keys;           // [nslots][G][cap]
    int32_t* cnt;        // [nslots][G]  entries in row
    int64_t* members;    // [nslots][G]  scored members seen by the CTA
    u64* sec;            // [nslots][G]  secondary top-1 key
    int32_t G, cap;
};

constexpr int kDbgStride = 32;   // EWSJF_PHASES: per-CTA timestamp slots

// Device-global counters.  Every field that many CTAs hit (atomics, spin loads)
// sits on its own 128-byte line: same-line atomics serialise in L2 and a load of
// a neighbouring field waited behind them (measured ~4.5 us after the fused
// tick's grid barrier with the counters packed together).
#define EWSJF_LINE(t, name) alignas(128) t name
struct Counters {        // zeroed at ctx creation; per-call fields are reset by the merge
    EWSJF_LINE(unsigned long long, n_invalid);
    EWSJF_LINE(unsigned long long, n_excluded);
    EWSJF_LINE(unsigned long long, gap_count);
    EWSJF_LINE(unsigned int, ticket);
    EWSJF_LINE(unsigned int, barrier);      // grid barrier of the stream kernel
    EWSJF_LINE(unsigned long long, tiles);  // dynamic tile scheduler of the stream kernel
    // diagnostics, accumulated over calls (never reset by the kernels)
    EWSJF_LINE(unsigned long long, dbg_inserted);
    unsigned long long dbg_compactions, dbg_overflow;
    // ftick.cu: monotone tickets (never reset; launch generation = ticket / grid)
    EWSJF_LINE(unsigned int, pub);          // sample boards published
    EWSJF_LINE(unsigned int, ready);        // generations whose sample bounds are in gthr
    EWSJF_LINE(unsigned int, done);         // CTAs past the streaming phase (grid barrier)
    EWSJF_LINE(unsigned long long, ftiles); // ftick.cu: dynamic tile claims (reset after the grid barrier)
    EWSJF_LINE(unsigned int, gap_done);     // merge.cuh: launch sequence whose Alg. 2 table is published
};
#undef EWSJF_LINE

// Fused streaming tick (ftick.cu): route + score + filter + rows, sample bound,
// grid barrier, per-queue merge.
struct FArgs {
    const int32_t* len;
    const float* arrival;
    const float* cost;          // nullable
    int32_t* qid_out;           // nullable
    int64_t n;
    uint32_t gbase;
    int32_t nslots;             // <= 64
    int32_t K;
    int32_t RC, HWM;            // row capacity per (queue, CTA) / high-water mark
    int32_t lut_size;           // LUT covers lengths [0, lut_size); longer: binary search (rare path)
    int32_t stages;             // TMA ring depth (CTA-level chunk stages)
    int32_t l2_prefetch;        // chunks after the ring prefetched into L2 at launch
    int32_t cnt_flush;          // iterations between u8 member-counter flushes (<= 62)
    int32_t sample_first;       // ring prologue: the sample chunk alone, the rest after the setup
    int32_t dyn_tail;           // last rounds of chunks claimed dynamically (0: all static)
    int32_t l2_hint;            // evict-first L2 policy on the pool's bulk copies
    int32_t board_m;            // sample board keys per (queue, CTA); 0 = no sample bound
    int32_t merge;              // 0: rows only; 1: final outputs; 2: exchange record (merge_phase)
    int32_t diag;               // timing diagnostics (EWSJF_DIAG bits); 0 in normal use
    const unsigned char* lut_dev;
    ScoreParams sp;
    Rows rows;                  // keys [64][G][RC]
    u64* gthr;                  // [nslots]
    u64* board;                 // [64][G][board_m]
    u64* rboard;                // [64][G] refresh board: CTA max key per queue (zero between ticks)
    int32_t refresh;            // progressive bound refresh on (needs K <= G)
    u64* ovf_keys;              // [G][kFOvf]
    unsigned char* ovf_code;    // [G][kFOvf]
    GapEntry* gap;
    int32_t gap_cap;
    Counters* ctr;
    unsigned long long* dbg;    // nullable: per-CTA phase timestamps [G][16]
    int64_t* topk_id;
    float* topk_score;
    int64_t* count;
    int64_t* head_id;
    float* head_score;
    float* max_score;
    ewsjf_summary* summary;
};
constexpr int kFOvf = 6144;     // per-CTA overflow list: >= 24 warps x 2 tiles x 128 requests

struct PartialArgs {
    const int32_t* len;
    const float* arrival;
    const float* cost;          // nullable
    const int32_t* qid_in;      // score_select: routed stable ids
    int32_t* qid_out;           // tick/route: nullable
    int64_t n;
    uint32_t gbase;             // global id of element 0
    int32_t tma;                // 1: pipelined TMA path (aligned pointers)
    int32_t K, cap, tgt, hwm;   // selection depth, buffer capacity, compaction target / trigger
    int32_t ids_identity;       // stable id == position for every queue (qid = slot)
    int32_t cnt_thread;         // per-thread u16 member counters (<= 64 queues) vs warp match-any
    int32_t dyn;                // dynamic tile scheduling (fused single-pass kernel)
    int32_t board_m;            // cross-CTA threshold board: keys per (queue, CTA); 0 = off
    u64* board;                 // [nslots][G][board_m]
    int32_t g_lo, g_hi;         // slot group handled by this pass (candidates)
    int32_t pass0;              // counts, qid, gaps, counters
    int32_t select;             // 0 = route only
    int32_t lut_size;           // LUT covers lengths [0, lut_size); 0 = binary search
    const unsigned char* lut_dev;   // stream.cu: prebuilt byte LUT (ctx cache, 16-byte padded) or null
    int32_t stages;             // stream.cu: TMA ring depth per warp
    ScoreParams sp;
    Rows rows;
    u64* gthr;                  // [nslots] cross-CTA filter thresholds
    unsigned long long* dbg;    // nullable: per-CTA phase timestamps [G][16] (EWSJF_PHASES)
    GapEntry* gap;
    int32_t gap_cap;
    Counters* ctr;
    // score_select: stable id -> slot map (sorted ids)
    int32_t nids;
    int32_t sorted_ids[kMaxSlots];
    int32_t sorted_slot[kMaxSlots];
};

// Bubble creation log written by the merge (host replays it into *part).
struct BubbleLog {
    int32_t n;
    int32_t pad;
    int32_t pos[kMaxSlots];     // insertion position at creation time
    int32_t lo[kMaxSlots], hi[kMaxSlots], L[kMaxSlots];
};

// Exchange record (one per rank) for the sharded tick.  Byte offsets.
struct ExLayout {
    int64_t hdr, members, sec, sec_sp, cnt, keys, sp, gaps, total;
    int32_t nq, k, gap_cap;
};
constexpr int kExGapDefault = 1024;   // gap entries per record unless the ctx sets another capacity
__host__ __device__ inline ExLayout ex_layout(int nq, int k, int gap_cap) {
    auto al = [](int64_t x) { return (x + 255) & ~(int64_t)255; };
    ExLayout L;
    L.nq = nq; L.k = k; L.gap_cap = gap_cap;
    int64_t o = 0;
    L.hdr = o;      o = al(o + 64);
    L.members = o;  o = al(o + 8 * (int64_t)nq);
    L.sec = o;      o = al(o + 8 * (int64_t)nq);
    L.sec_sp = o;   o = al(o + 4 * (int64_t)nq);
    L.cnt = o;      o = al(o + 4 * (int64_t)nq);
    L.keys = o;     o = al(o + 8 * (int64_t)nq * k);
    L.sp = o;       o = al(o + 4 * (int64_t)nq * k);
    L.gaps = o;     o = al(o + (int64_t)sizeof(GapEntry) * gap_cap);
    L.total = o;
    return L;
}
struct ExHeader {                // at L.hdr
    int64_t gap_count, n_invalid, n_excluded, pad[5];
};

// Inputs of the merge.
enum { MERGE_IN_ROWS = 0, MERGE_IN_EXCHANGE = 1 };
enum { MERGE_OUT_FINAL = 0, MERGE_OUT_EXCHANGE = 1, MERGE_OUT_ROUTE = 2 };

struct MergeArgs {
    int32_t in_mode, out_mode;
    int32_t K;
    int32_t nq;                 // queues of the input partition
    int32_t next_id;            // for bubble ids
    int32_t bubble_width;
    ScoreParams sp;
    double theta[6];            // a_b, b_b, a_u, b_u, a_f, b_f (bubble weights, R21)
    // --- rows input (in_mode ROWS)
    Rows rows;
    const int32_t* len;         // local pool (payload recompute)
    const float* arrival;
    const float* cost;
    uint32_t gbase;
    int64_t n_local;
    const GapEntry* gap;        // single gap list
    Counters* ctr;
    int32_t gap_cap;
    // epoch-parallel Alg. 2 (merge.cuh): per gap entry its final internal slot, a
    // classification scratch and two ping-pong lists of unresolved entries
    // [gap capacity each]; the final queue table; launch sequence of this merge
    int32_t* g_slot;
    int32_t* g_res;
    int32_t* g_u0;
    int32_t* g_u1;
    int32_t* g_tab;             // [0] n, [1] nb, [2] nd, then lo/hi/slot/L/id [256] each
    uint32_t seq;
    // --- exchange input (in_mode EXCHANGE)
    const unsigned char* ex_in; // world records
    int32_t world;
    int64_t ex_bytes;
    int32_t ex_gap;             // gap entries per exchange record (ctx->ex_gap)
    // --- outputs
    unsigned char* ex_out;      // out_mode EXCHANGE: this rank's record
    int64_t* topk_id;
    float* topk_score;
    int64_t* count;
    int64_t* head_id;
    float* head_score;
    float* max_score;
    ewsjf_summary* summary;
    BubbleLog* blog;
    int32_t* qid;               // gap requests' qid write-back (local pool)
    u64* gthr;                  // zeroed for the next call
    unsigned long long* dbg;    // nullable: phase timestamps (EWSJF_PHASES)
};

}  // namespace ewsjf
