// ctx.h — the ewsjf_ctx definition shared by the host-side translation units.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "tick.cuh"

using namespace ewsjf;

namespace ewsjf {
struct RpScratch;
struct SweepScratch;
}

struct ewsjf_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t stream_ev = nullptr;   // ewsjf_ctx_set_stream: orders the new stream after the old
    // fused tick policy tables in device memory (ftick.cu), cached by content
    void* d_policy = nullptr;
    void* h_policy = nullptr;          // pinned staging
    void* h_policy_shadow = nullptr;   // last uploaded content
    cudaEvent_t policy_ev = nullptr;
    bool policy_valid = false;
    int64_t max_pool = 0, max_history = 0;
    int32_t max_k = 0;
    int num_sms = 0;
    int smem_optin = 0;
    int coop = 0;
    int32_t cap_max = 0;
    char err[512] = {0};
    // scratch
    Rows rows{};
    u64* gthr = nullptr;
    u64* board = nullptr;
    Counters* ctr = nullptr;
    GapEntry* gap = nullptr;
    unsigned long long* dbg = nullptr;   // [num_sms][16] phase timestamps
    // length -> queue-position byte LUT of the last partition routed (stream.cu),
    // rebuilt on the host and uploaded only when the queue bounds change
    unsigned char* d_lut = nullptr;     // device, kLutCap + 32 bytes
    unsigned char* h_lut = nullptr;     // pinned staging
    cudaEvent_t lut_ev = nullptr;       // last upload
    int32_t lut_n = -1, lut_size = 0;
    std::vector<int32_t> lut_bounds;    // min/max of the cached partition
    int32_t gap_cap = 8192;             // gap list entries (max(8192, max_pool))
    int32_t *g_slot = nullptr, *g_res = nullptr, *g_u0 = nullptr, *g_u1 = nullptr, *g_tab = nullptr;
    uint32_t merge_seq = 0;             // launches of merge_phase (Alg. 2 table publication)
    BubbleLog* d_blog = nullptr;
    BubbleLog* h_blog = nullptr;        // pinned
    ewsjf_summary* d_summary = nullptr;
    ewsjf_summary* h_summary = nullptr; // pinned
    // host-variant staging (tick_host)
    int32_t* d_len = nullptr;
    float* d_arr = nullptr;
    float* d_cost = nullptr;
    int32_t* d_qid = nullptr;
    int64_t* d_topk_id = nullptr;
    float* d_topk_score = nullptr;
    int64_t* d_count = nullptr;
    int64_t* d_head_id = nullptr;
    float* d_head_score = nullptr;
    float* d_max_score = nullptr;
    // partition (R&P) scratch lives in partition.cu
    ewsjf::RpScratch* rp = nullptr;
    // Θ-sweep scratch (sweep.cu), grown on demand and kept
    ewsjf::SweepScratch* sw = nullptr;
    // fused tick (ftick.cu): rows [64][G][f_rc], per-CTA overflow lists
    u64* f_rows = nullptr;
    int32_t f_rc = 0;
    u64* f_ovf_keys = nullptr;
    unsigned char* f_ovf_code = nullptr;
    // NCCL communicator of the index-sharded tick (nccl.cu); exchange buffers
    // sized for 256 queues x max_k, allocated when the comm is set
    void* nccl_comm = nullptr;
    bool nccl_owned = false;
    int32_t nccl_rank = 0, nccl_world = 0;
    unsigned char* ex_local = nullptr;
    unsigned char* ex_all = nullptr;
    int64_t ex_cap = 0;
    int32_t ex_gap = 1024;              // gap entries per exchange record (ewsjf_ctx_set_exchange_gap_cap)
    // ewsjf_tick_host pipeline: chunks copied on h2d_st, reduced by local ticks into
    // exchange records on the ctx stream, qid slices copied back on d2h_st
    static constexpr int kPipeMax = 8;
    cudaStream_t h2d_st = nullptr, d2h_st = nullptr;
    cudaEvent_t pipe_h2d[kPipeMax] = {}, pipe_cmp[kPipeMax] = {};
    cudaEvent_t pipe_start = nullptr, pipe_d2h = nullptr;
    unsigned char* ex_pipe = nullptr;
    int64_t ex_pipe_per = 0;
    // batch builder prefix scratch (batch.cu)
    uint32_t* d_bpre = nullptr;
    int64_t bpre_cap = 0;
    int64_t batch_smem_attr = 0;
    // instrumentation
    long long launches = 0;
    bool timing = false;
    std::vector<cudaEvent_t> ev_a, ev_b;
    std::vector<int> ev_kind;
    size_t ev_n = 0;
};

namespace ewsjf {
enum { KIND_TICK = 0, KIND_MERGE = 1, KIND_PARTITION = 2, KIND_SWEEP = 3, KIND_BATCH = 4 };
// Bracket one launch with events when timing is on; count it always.
struct LaunchScope {
    ewsjf_ctx* c;
    int kind;
    bool rec = false;
    LaunchScope(ewsjf_ctx* ctx, int k) : c(ctx), kind(k) {
        c->launches++;
        if (c->timing && c->ev_n < c->ev_a.size()) {
            cudaEventRecord(c->ev_a[c->ev_n], c->stream);
            rec = true;
        }
    }
    ~LaunchScope() {
        if (rec) {
            cudaEventRecord(c->ev_b[c->ev_n], c->stream);
            c->ev_kind[c->ev_n] = kind;
            c->ev_n++;
        }
    }
};
}  // namespace ewsjf

namespace ewsjf {
void rp_free(ewsjf_ctx* ctx);
ewsjf_status rp_alloc(ewsjf_ctx* ctx);
void sweep_free(ewsjf_ctx* ctx);
}

static inline ewsjf_status fail(ewsjf_ctx* ctx, ewsjf_status s, const char* fmt, ...) {
    if (ctx) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(ctx->err, sizeof ctx->err, fmt, ap);
        va_end(ap);
    }
    return s;
}
#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(ctx, EWSJF_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                       \
    } while (0)

