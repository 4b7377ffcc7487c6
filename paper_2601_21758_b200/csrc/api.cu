// api.cu — C ABI of libewsjf (include/ewsjf.h): context, policy upload,
// launch orchestration of the tick / score_select / route / sharded tick.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include "tick.cuh"

namespace ewsjf {
cudaError_t launch_partial(const PartialArgs& A, const Policy& P, const MergeArgs* MA, bool route, bool has_cost,
                           bool use_lut, int grid, cudaStream_t st);
int64_t partial_smem_bytes(bool route, bool has_cost, bool tma, int lut_size, int nslots, int nids, int pass0,
                           int cnt_thread, int ngs, int cap);
cudaError_t launch_merge(const MergeArgs& A, const Policy& P, bool has_cost, int grid, cudaStream_t st);
int64_t merge_smem_total(int in_mode);
cudaError_t launch_stream(const PartialArgs& A, const Policy& P, const MergeArgs* MA, bool has_cost, int grid,
                          cudaStream_t st);
int64_t stream_smem_bytes(bool has_cost, int lut_size, int nslots, int cap, int stages);
cudaError_t launch_ftick(const FArgs& A, const Policy* P, const MergeArgs& MA, bool has_cost, int grid,
                         cudaStream_t st);
int64_t ftick_smem_bytes(bool has_cost, int lut_size, int nslots, int stages);
bool sweep_diag(ewsjf_ctx* ctx, unsigned long long* cuts_inserts, long long* records);
ewsjf_status nccl_allgather(ewsjf_ctx* ctx, int64_t bytes);
void nccl_release(ewsjf_ctx* ctx);
}  // namespace ewsjf

using namespace ewsjf;

#include "ctx.h"

// ------------------------------------------------------------------ misc ---
extern "C" int ewsjf_abi_version(void) { return EWSJF_ABI_VERSION; }

extern "C" const char* ewsjf_status_str(ewsjf_status s) {
    switch (s) {
        case EWSJF_OK: return "ok";
        case EWSJF_ERR_INVALID_ARG: return "invalid argument";
        case EWSJF_ERR_DOMAIN: return "domain error (elements excluded)";
        case EWSJF_ERR_EMPTY: return "empty input";
        case EWSJF_ERR_CAPACITY: return "capacity exceeded";
        case EWSJF_ERR_CUDA: return "CUDA error";
        case EWSJF_ERR_UNSUPPORTED: return "unsupported input";
        case EWSJF_ERR_NCCL: return "NCCL error";
    }
    return "unknown status";
}

extern "C" const char* ewsjf_last_error(const ewsjf_ctx* ctx) { return ctx ? ctx->err : "null ctx"; }

extern "C" int32_t ewsjf_ctx_num_ctas(const ewsjf_ctx* ctx) { return ctx ? ctx->num_sms : 0; }

static int32_t cap_for(int32_t K) {
    int32_t c = std::max(2 * K, 64);
    return (c + 31) & ~31;
}

// ewsjf_tick_host pipelines pools of at least this size (chunks of >= 1M requests)
constexpr int64_t kPipeMinPool = 2000000;

// --------------------------------------------------------------- context ---
extern "C" ewsjf_status ewsjf_ctx_create(int device, void* cuda_stream, int64_t max_pool, int64_t max_history,
                                         int32_t max_k, ewsjf_ctx** out) {
    if (!out || max_pool < 0 || max_history < 0 || max_k < 1 || max_k > EWSJF_MAX_K || max_pool >= 0xffffffffll)
        return EWSJF_ERR_INVALID_ARG;
    *out = nullptr;
    ewsjf_ctx* ctx = new ewsjf_ctx();
    ctx->device = device;
    ctx->stream = (cudaStream_t)cuda_stream;
    ctx->max_pool = max_pool;
    ctx->max_history = max_history;
    ctx->max_k = max_k;
    ctx->cap_max = cap_for(max_k);
    auto bad = [&](ewsjf_status s) { ewsjf_ctx_destroy(ctx); return s; };
    if (cudaSetDevice(device) != cudaSuccess) return bad(EWSJF_ERR_CUDA);
    if (cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
        return bad(EWSJF_ERR_CUDA);
    cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&ctx->coop, cudaDevAttrCooperativeLaunch, device);
    if (getenv("EWSJF_NO_FUSE")) ctx->coop = 0;
    const int G = ctx->num_sms;
    const size_t nrow = (size_t)kMaxSlots * G;
    // gap list sized for the whole pool: App. D's Alg. 2 must stay exact however many
    // pending requests fall between the queues (a stale partition)
    ctx->gap_cap = (int32_t)std::max<int64_t>(8192, std::min<int64_t>(max_pool, 0x7fffffffLL));
    bool ok = cudaMalloc(&ctx->rows.keys, nrow * max_k * sizeof(u64)) == cudaSuccess &&
              cudaMalloc(&ctx->rows.cnt, nrow * sizeof(int32_t)) == cudaSuccess &&
              cudaMalloc(&ctx->rows.members, nrow * sizeof(int64_t)) == cudaSuccess &&
              cudaMalloc(&ctx->rows.sec, nrow * sizeof(u64)) == cudaSuccess &&
              cudaMalloc(&ctx->gthr, kMaxSlots * sizeof(u64)) == cudaSuccess &&
              cudaMalloc(&ctx->board, nrow * 8 * sizeof(u64)) == cudaSuccess &&
              cudaMalloc(&ctx->ctr, sizeof(Counters)) == cudaSuccess &&
              cudaMalloc(&ctx->dbg, (size_t)G * kDbgStride * 8) == cudaSuccess &&
              cudaMalloc(&ctx->d_lut, kLutCap + 32) == cudaSuccess &&
              cudaMallocHost(&ctx->h_lut, kLutCap + 32) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->lut_ev, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->stream_ev, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->policy_ev, cudaEventDisableTiming) == cudaSuccess &&
              cudaMalloc(&ctx->d_policy, sizeof(Policy)) == cudaSuccess &&
              cudaMallocHost(&ctx->h_policy, sizeof(Policy)) == cudaSuccess &&
              cudaMalloc(&ctx->gap, (size_t)ctx->gap_cap * sizeof(GapEntry)) == cudaSuccess &&
              cudaMalloc(&ctx->g_slot, (size_t)ctx->gap_cap * 4) == cudaSuccess &&
              cudaMalloc(&ctx->g_res, (size_t)ctx->gap_cap * 4) == cudaSuccess &&
              cudaMalloc(&ctx->g_u0, (size_t)ctx->gap_cap * 4) == cudaSuccess &&
              cudaMalloc(&ctx->g_u1, (size_t)ctx->gap_cap * 4) == cudaSuccess &&
              cudaMalloc(&ctx->g_tab, (3 + 5 * kMaxSlots) * 4) == cudaSuccess &&
              cudaMalloc(&ctx->d_blog, sizeof(BubbleLog)) == cudaSuccess &&
              cudaMallocHost(&ctx->h_blog, sizeof(BubbleLog)) == cudaSuccess &&
              cudaMalloc(&ctx->d_summary, sizeof(ewsjf_summary)) == cudaSuccess &&
              cudaMallocHost(&ctx->h_summary, sizeof(ewsjf_summary)) == cudaSuccess &&
              cudaMalloc(&ctx->d_topk_id, (size_t)kMaxSlots * max_k * 8) == cudaSuccess &&
              cudaMalloc(&ctx->d_topk_score, (size_t)kMaxSlots * max_k * 4) == cudaSuccess &&
              cudaMalloc(&ctx->d_count, kMaxSlots * 8) == cudaSuccess &&
              cudaMalloc(&ctx->d_head_id, kMaxSlots * 8) == cudaSuccess &&
              cudaMalloc(&ctx->d_head_score, kMaxSlots * 4) == cudaSuccess &&
              cudaMalloc(&ctx->d_max_score, kMaxSlots * 4) == cudaSuccess;
    // fused tick rows: 64 queues x G CTAs x f_rc keys; overflow lists G x kFOvf
    ctx->f_rc = std::max(512, 4 * max_k);
    ctx->h_policy_shadow = new unsigned char[sizeof(Policy)];
    ctx->bpre_cap = (int64_t)kMaxSlots * max_k;      // batch builder prefixes (global fallback)
    ok = ok && cudaMalloc(&ctx->d_bpre, (size_t)ctx->bpre_cap * sizeof(uint32_t)) == cudaSuccess;
    ok = ok && cudaMalloc(&ctx->f_rows, (size_t)64 * G * ctx->f_rc * sizeof(u64)) == cudaSuccess &&
         cudaMalloc(&ctx->f_ovf_keys, (size_t)G * kFOvf * sizeof(u64)) == cudaSuccess &&
         cudaMalloc(&ctx->f_ovf_code, (size_t)G * kFOvf) == cudaSuccess;
    if (ok && max_pool > 0) {
        ok = cudaMalloc(&ctx->d_len, (size_t)max_pool * 4) == cudaSuccess &&
             cudaMalloc(&ctx->d_arr, (size_t)max_pool * 4) == cudaSuccess &&
             cudaMalloc(&ctx->d_cost, (size_t)max_pool * 4) == cudaSuccess &&
             cudaMalloc(&ctx->d_qid, (size_t)max_pool * 4) == cudaSuccess;
    }
    if (ok && max_pool >= kPipeMinPool) {   // ewsjf_tick_host pipeline (streams, events, exchange records)
        ctx->ex_pipe_per = ex_layout(kMaxSlots, max_k, ctx->ex_gap).total;
        ok = cudaStreamCreateWithFlags(&ctx->h2d_st, cudaStreamNonBlocking) == cudaSuccess &&
             cudaStreamCreateWithFlags(&ctx->d2h_st, cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&ctx->pipe_start, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&ctx->pipe_d2h, cudaEventDisableTiming) == cudaSuccess &&
             cudaMalloc(&ctx->ex_pipe, (size_t)ctx->ex_pipe_per * ewsjf_ctx::kPipeMax) == cudaSuccess;
        for (int i = 0; ok && i < ewsjf_ctx::kPipeMax; i++)
            ok = cudaEventCreateWithFlags(&ctx->pipe_h2d[i], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&ctx->pipe_cmp[i], cudaEventDisableTiming) == cudaSuccess;
    }
    if (!ok) return bad(EWSJF_ERR_CUDA);
    ok = cudaMemset(ctx->gthr, 0, kMaxSlots * sizeof(u64)) == cudaSuccess &&
         cudaMemset(ctx->board, 0, nrow * 8 * sizeof(u64)) == cudaSuccess &&
         cudaMemset(ctx->ctr, 0, sizeof(Counters)) == cudaSuccess &&
         cudaMemset(ctx->rows.cnt, 0, nrow * sizeof(int32_t)) == cudaSuccess &&
         cudaMemset(ctx->rows.members, 0, nrow * sizeof(int64_t)) == cudaSuccess &&
         cudaMemset(ctx->rows.sec, 0, nrow * sizeof(u64)) == cudaSuccess &&
         cudaDeviceSynchronize() == cudaSuccess;
    if (!ok) return bad(EWSJF_ERR_CUDA);
    ctx->rows.G = G;
    if (max_history > 0 && rp_alloc(ctx) != EWSJF_OK) return bad(EWSJF_ERR_CUDA);
    *out = ctx;
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_ctx_set_stream(ewsjf_ctx* ctx, void* cuda_stream) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    cudaStream_t ns = (cudaStream_t)cuda_stream;
    if (ns != ctx->stream) {
        // all ctx scratch (rows, counters, LUT, gap list) is shared by the ctx's calls:
        // order the new stream after everything already queued on the old one
        CU(cudaSetDevice(ctx->device));
        // not while either stream is being captured into a CUDA graph: an event recorded
        // outside the capture would invalidate it (the capturing caller orders the streams)
        cudaStreamCaptureStatus cs_old = cudaStreamCaptureStatusNone, cs_new = cudaStreamCaptureStatusNone;
        CU(cudaStreamIsCapturing(ctx->stream, &cs_old));
        CU(cudaStreamIsCapturing(ns, &cs_new));
        if (cs_old == cudaStreamCaptureStatusNone && cs_new == cudaStreamCaptureStatusNone) {
            CU(cudaEventRecord(ctx->stream_ev, ctx->stream));
            CU(cudaStreamWaitEvent(ns, ctx->stream_ev, 0));
        }
        ctx->stream = ns;
    }
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_ctx_destroy(ewsjf_ctx* ctx) {
    if (!ctx) return EWSJF_OK;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->h_lut) cudaFreeHost(ctx->h_lut);
    if (ctx->lut_ev) cudaEventDestroy(ctx->lut_ev);
    if (ctx->stream_ev) cudaEventDestroy(ctx->stream_ev);
    if (ctx->policy_ev) cudaEventDestroy(ctx->policy_ev);
    if (ctx->h_policy) cudaFreeHost(ctx->h_policy);
    if (ctx->d_policy) cudaFree(ctx->d_policy);
    delete[] (unsigned char*)ctx->h_policy_shadow;
    nccl_release(ctx);
    for (int i = 0; i < ewsjf_ctx::kPipeMax; i++) {
        if (ctx->pipe_h2d[i]) cudaEventDestroy(ctx->pipe_h2d[i]);
        if (ctx->pipe_cmp[i]) cudaEventDestroy(ctx->pipe_cmp[i]);
    }
    if (ctx->pipe_start) cudaEventDestroy(ctx->pipe_start);
    if (ctx->pipe_d2h) cudaEventDestroy(ctx->pipe_d2h);
    if (ctx->h2d_st) cudaStreamDestroy(ctx->h2d_st);
    if (ctx->d2h_st) cudaStreamDestroy(ctx->d2h_st);
    if (ctx->ex_pipe) cudaFree(ctx->ex_pipe);
    void* d[] = {ctx->g_slot, ctx->g_res, ctx->g_u0, ctx->g_u1, ctx->g_tab, ctx->f_rows, ctx->f_ovf_keys, ctx->f_ovf_code, ctx->d_lut, ctx->dbg, ctx->rows.keys, ctx->rows.cnt, ctx->rows.members, ctx->rows.sec, ctx->gthr, ctx->board, ctx->ctr, ctx->gap,
                 ctx->d_blog, ctx->d_summary, ctx->d_len, ctx->d_arr, ctx->d_cost, ctx->d_qid, ctx->d_topk_id,
                 ctx->d_topk_score, ctx->d_count, ctx->d_head_id, ctx->d_head_score, ctx->d_max_score};
    for (void* p : d)
        if (p) cudaFree(p);
    for (auto e : ctx->ev_a) cudaEventDestroy(e);
    for (auto e : ctx->ev_b) cudaEventDestroy(e);
    if (ctx->h_blog) cudaFreeHost(ctx->h_blog);
    if (ctx->h_summary) cudaFreeHost(ctx->h_summary);
    rp_free(ctx);
    sweep_free(ctx);
    if (ctx->d_bpre) cudaFree(ctx->d_bpre);
    delete ctx;
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_ctx_set_timing(ewsjf_ctx* ctx, int32_t enable) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    CU(cudaSetDevice(ctx->device));
    if (enable && ctx->ev_a.empty()) {
        const size_t cap = 16384;
        ctx->ev_a.resize(cap); ctx->ev_b.resize(cap); ctx->ev_kind.resize(cap);
        for (size_t i = 0; i < cap; i++) {
            CU(cudaEventCreate(&ctx->ev_a[i]));
            CU(cudaEventCreate(&ctx->ev_b[i]));
        }
    }
    ctx->timing = enable != 0;
    ctx->ev_n = 0;
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_ctx_get_timing(ewsjf_ctx* ctx, ewsjf_timing* out) {
    if (!ctx || !out) return EWSJF_ERR_INVALID_ARG;
    CU(cudaSetDevice(ctx->device));
    CU(cudaStreamSynchronize(ctx->stream));
    memset(out, 0, sizeof *out);
    Counters c;
    CU(cudaMemcpy(&c, ctx->ctr, sizeof c, cudaMemcpyDeviceToHost));
    out->candidates_inserted = (int64_t)c.dbg_inserted;
    out->compactions = (int64_t)c.dbg_compactions;
    unsigned long long sw[2] = {0, 0};
    long long recs = 0;
    if (sweep_diag(ctx, sw, &recs)) {
        out->candidates_inserted += (int64_t)sw[1];
        out->compactions += (int64_t)sw[0];
        out->sweep_records = recs;
    }
    out->launches = ctx->launches;
    out->recorded = (int64_t)ctx->ev_n;
    for (size_t i = 0; i < ctx->ev_n; i++) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev_a[i], ctx->ev_b[i]));
        switch (ctx->ev_kind[i]) {
            case KIND_TICK: out->tick_ms += ms; out->tick_launches++; break;
            case KIND_MERGE: out->merge_ms += ms; out->merge_launches++; break;
            case KIND_PARTITION: out->partition_ms += ms; out->partition_launches++; break;
            case KIND_BATCH: out->batch_ms += ms; out->batch_launches++; break;
            default: out->sweep_ms += ms; out->sweep_launches++; break;
        }
    }
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_ctx_get_phases(ewsjf_ctx* ctx, uint64_t* out, int32_t n) {
    if (!ctx || !out || n < 0) return EWSJF_ERR_INVALID_ARG;
    CU(cudaSetDevice(ctx->device));
    CU(cudaStreamSynchronize(ctx->stream));
    const int64_t m = std::min<int64_t>(n, (int64_t)ctx->num_sms * kDbgStride);
    CU(cudaMemcpy(out, ctx->dbg, (size_t)m * 8, cudaMemcpyDeviceToHost));
    return EWSJF_OK;
}

// ---------------------------------------------------------------- policy ---
static ewsjf_status check_partition(ewsjf_ctx* ctx, const ewsjf_partition_t* part) {
    if (!part) return fail(ctx, EWSJF_ERR_INVALID_ARG, "null partition");
    if (part->n < 0 || part->n > EWSJF_MAX_QUEUES) return fail(ctx, EWSJF_ERR_INVALID_ARG, "partition n=%d", part->n);
    for (int i = 0; i < part->n; i++) {
        const ewsjf_queue& q = part->q[i];
        if (q.min_len >= q.max_len) return fail(ctx, EWSJF_ERR_INVALID_ARG, "queue %d: min_len >= max_len", i);
        if (i > 0 && part->q[i - 1].max_len > q.min_len)
            return fail(ctx, EWSJF_ERR_INVALID_ARG, "queues %d,%d overlap or are unsorted", i - 1, i);
        if (q.id < 0 || q.id >= part->next_id)
            return fail(ctx, EWSJF_ERR_INVALID_ARG, "queue %d: id %d outside [0, next_id)", i, q.id);
    }
    for (int i = 0; i < part->n; i++)
        for (int j = i + 1; j < part->n; j++)
            if (part->q[i].id == part->q[j].id) return fail(ctx, EWSJF_ERR_INVALID_ARG, "duplicate queue id");
    return EWSJF_OK;
}

// A7 on the host: w_x = fp32(max(0, a_x * b̄ + b_x)), fp64 with
// no contraction (this file is compiled with -fmad=false for host code too).
static inline float clamp_w(double a, double mean, double b) {
    volatile double t = a * mean;
    double v = t + b;
    return (float)(v > 0.0 ? v : 0.0);
}

extern "C" ewsjf_status ewsjf_weights_from_meta(const ewsjf_meta* th, const ewsjf_partition_t* part,
                                                ewsjf_weights* out) {
    if (!th || !part || !out || part->n < 0 || part->n > EWSJF_MAX_QUEUES) return EWSJF_ERR_INVALID_ARG;
    for (int i = 0; i < part->n; i++) {
        const double m = part->q[i].mean;
        out[i].w_base = clamp_w(th->a_b, m, th->b_b);
        out[i].w_urg = clamp_w(th->a_u, m, th->b_u);
        out[i].w_fair = clamp_w(th->a_f, m, th->b_f);
    }
    return EWSJF_OK;
}

static void fill_policy(const ewsjf_partition_t* part, const ewsjf_weights* w, Policy* P) {
    memset(P, 0, sizeof *P);
    P->nslots = part->n;
    for (int i = 0; i < part->n; i++) {
        P->min_len[i] = part->q[i].min_len;
        P->max_len[i] = part->q[i].max_len;
        P->sid[i] = part->q[i].id;
        P->wb[i] = w[i].w_base;
        P->wu[i] = w[i].w_urg;
        volatile double f = (double)w[i].w_fair * 0.69314718055994530942;
        P->wf[i] = (float)f;
    }
}

static ewsjf_status check_select(ewsjf_ctx* ctx, const ewsjf_select_params* sp) {
    if (!sp) return fail(ctx, EWSJF_ERR_INVALID_ARG, "null select params");
    if (sp->k < 1 || sp->k > ctx->max_k) return fail(ctx, EWSJF_ERR_INVALID_ARG, "k=%d outside 1..%d", sp->k, ctx->max_k);
    if (sp->mode != EWSJF_SELECT_SCORE && sp->mode != EWSJF_SELECT_FIFO)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad select mode");
    return EWSJF_OK;
}

static ScoreParams score_params(const ewsjf_select_params* sp) {
    ScoreParams s;
    s.now = sp->now;
    s.c0 = sp->cost.c0;
    s.c1 = sp->cost.c1;
    s.c2 = sp->cost.c2;
    s.mode = sp->mode;
    s.k = sp->k;
    return s;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// The streaming tick's length -> position byte LUT (lut[0] = bad, holes and
// lut[lutsz] = gap), built on the host and uploaded when the bounds change.
static ewsjf_status ensure_lut(ewsjf_ctx* ctx, const ewsjf_partition_t* part, int lutsz) {
    std::vector<int32_t> key;
    key.reserve(2 * part->n);
    for (int i = 0; i < part->n; i++) { key.push_back(part->q[i].min_len); key.push_back(part->q[i].max_len); }
    if (ctx->lut_n == part->n && ctx->lut_size == lutsz && key == ctx->lut_bounds) return EWSJF_OK;
    CU(cudaEventSynchronize(ctx->lut_ev));          // the staging buffer is free again
    unsigned char* h = ctx->h_lut;
    const int padded = (lutsz + 1 + 15) & ~15;
    memset(h, 0xFE, padded);
    for (int q = 0; q < part->n; q++) {
        const int lo = part->q[q].min_len, hi = std::min(part->q[q].max_len, lutsz);
        for (int b = std::max(lo, 0); b < hi; b++) h[b] = (unsigned char)q;
    }
    h[0] = 0xFF;
    h[lutsz] = 0xFE;
    CU(cudaMemcpyAsync(ctx->d_lut, h, padded, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaEventRecord(ctx->lut_ev, ctx->stream));
    ctx->lut_n = part->n;
    ctx->lut_size = lutsz;
    ctx->lut_bounds = key;
    return EWSJF_OK;
}

// The policy tables of the fused tick in device memory: uploaded (through a pinned
// staging copy) only when they differ from the last upload.
static ewsjf_status ensure_policy(ewsjf_ctx* ctx, const Policy& P) {
    if (ctx->policy_valid && memcmp(ctx->h_policy_shadow, &P, sizeof(Policy)) == 0) return EWSJF_OK;
    CU(cudaEventSynchronize(ctx->policy_ev));       // the staging buffer is free again
    memcpy(ctx->h_policy, &P, sizeof(Policy));
    memcpy(ctx->h_policy_shadow, &P, sizeof(Policy));
    CU(cudaMemcpyAsync(ctx->d_policy, ctx->h_policy, sizeof(Policy), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaEventRecord(ctx->policy_ev, ctx->stream));
    ctx->policy_valid = true;
    return EWSJF_OK;
}

// Run the partial pass(es) of a tick / score_select / route over [len, n).
static ewsjf_status run_partial(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arr, const float* d_cost,
                                const int32_t* d_qid_in, int32_t* d_qid_out, int64_t n, int64_t gbase,
                                const ewsjf_partition_t* part, const Policy& P, const ewsjf_select_params* sp,
                                bool route, bool select, const MergeArgs* fuse = nullptr, bool* fused = nullptr) {
    if (fused) *fused = false;
    const int nslots = part->n;
    const bool has_cost = d_cost != nullptr;
    const int K = select ? sp->k : 1;
    int cap = cap_for(K);
    PartialArgs A;
    memset(&A, 0, sizeof A);
    A.len = d_len;
    A.arrival = d_arr;
    A.cost = d_cost;
    A.qid_in = d_qid_in;
    A.qid_out = d_qid_out;
    A.n = n;
    A.gbase = (uint32_t)gbase;
    A.tma = aligned16(d_len) && aligned16(d_arr) && (!has_cost || aligned16(d_cost)) &&
            (route ? (!d_qid_out || aligned16(d_qid_out)) : aligned16(d_qid_in));
    A.K = K;
    A.cap = cap;
    A.ids_identity = 1;
    for (int i = 0; i < nslots; i++)
        if (part->q[i].id != i) A.ids_identity = 0;
    A.cnt_thread = nslots <= 64 ? 1 : 0;
    A.select = select ? 1 : 0;
    A.sp = select ? score_params(sp) : ScoreParams{0.f, 0.f, 0.f, 0.f, 0, 1};
    A.rows = ctx->rows;
    A.rows.cap = K;
    A.gthr = ctx->gthr;
    A.gap = ctx->gap;
    A.gap_cap = ctx->gap_cap;
    A.ctr = ctx->ctr;
    bool use_lut = false;
    if (route && nslots > 0 && nslots <= 250 && part->q[nslots - 1].max_len <= kLutCap) {
        use_lut = true;
        A.lut_size = part->q[nslots - 1].max_len;
    }
    if (!route) {
        std::vector<std::pair<int, int>> ids;
        for (int i = 0; i < nslots; i++) ids.push_back({part->q[i].id, i});
        std::sort(ids.begin(), ids.end());
        A.nids = nslots;
        for (int i = 0; i < nslots; i++) { A.sorted_ids[i] = ids[i].first; A.sorted_slot[i] = ids[i].second; }
    }
    const int budget = ctx->smem_optin > 0 ? ctx->smem_optin : 232448;
    // The barrier-free streaming pass (stream.cu): LUT-routable partitions of
    // <= 64 queues over a 16-byte aligned pool, all queues in one pass.
    if (route && select && use_lut && nslots <= 64 && A.tma && !getenv("EWSJF_OLD_TICK")) {
        // candidate buffer: K + 64 <= cap <= 256 (register selection holds 8 keys per lane)
        int scap = std::min(256, (std::max(K + 64, 3 * K) + 31) & ~31);
        int stages = 3;
        if (const char* e = getenv("EWSJF_STAGES")) stages = std::max(2, std::min(8, atoi(e)));
        while (scap > K + 64 && stream_smem_bytes(has_cost, A.lut_size, nslots, scap, stages) > budget) scap -= 32;
        while (stages > 2 && stream_smem_bytes(has_cost, A.lut_size, nslots, scap, stages) > budget) stages--;
        A.stages = stages;
        const int a_tma = A.tma;
        A.tma = getenv("EWSJF_TMA_RING") ? 1 : 0;      // per-warp TMA bulk ring vs per-lane cp.async ring
        if (scap >= K + 64 && stream_smem_bytes(has_cost, A.lut_size, nslots, scap, stages) <= budget) {
            A.cap = scap;
            A.hwm = scap - 32;
            if (ensure_lut(ctx, part, A.lut_size) != EWSJF_OK) return EWSJF_ERR_CUDA;
            A.lut_dev = ctx->d_lut;
            A.dbg = getenv("EWSJF_PHASES") ? ctx->dbg : nullptr;
            // cross-CTA board: bm keys per (queue, CTA), G*bm <= 320 and >= K
            A.board = ctx->board;
            A.board_m = std::min(2, 320 / std::max(ctx->num_sms, 1));
            if (const char* e = getenv("EWSJF_BOARD_M")) A.board_m = std::min(atoi(e), 320 / std::max(ctx->num_sms, 1));
            if (ctx->num_sms * A.board_m < K) A.board_m = 0;
            const bool fuse_s = fuse && ctx->coop && merge_smem_total(MERGE_IN_ROWS) <= budget;
            cudaError_t e;
            {
                LaunchScope ls(ctx, KIND_TICK);
                e = launch_stream(A, P, fuse_s ? fuse : nullptr, has_cost, ctx->num_sms, ctx->stream);
            }
            if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "stream tick kernel: %s", cudaGetErrorString(e));
            if (fused) *fused = fuse_s;
            return EWSJF_OK;
        }
        A.tma = a_tma;
    }
    // slot groups so that the candidate buffers fit in shared memory
    int ngs = std::max(nslots, 1);
    auto smem_for_cap = [&](int g, int c) {
        return partial_smem_bytes(route, has_cost, A.tma, use_lut ? A.lut_size : 0, nslots, A.nids, 1,
                                  A.cnt_thread, g, c);
    };
    auto smem_for = [&](int g) { return smem_for_cap(g, cap); };
    if (A.cnt_thread && smem_for(1) > budget) A.cnt_thread = 0;
    while (ngs > 1 && smem_for(ngs) > budget) ngs = (ngs + 1) / 2;
    if (smem_for(ngs) > budget)
        return fail(ctx, EWSJF_ERR_UNSUPPORTED, "tick does not fit shared memory (k=%d)", K);
    // grow the candidate buffers into the remaining shared memory (fewer compactions)
    if (select) {
        while (cap < 1024 && smem_for_cap(ngs, cap + 32) <= budget - 1024) cap += 32;
    }
    A.cap = cap;
    A.tgt = K + (cap - K) / 8;
    A.hwm = cap - 16;
    const int passes = select ? std::max(1, (nslots + ngs - 1) / ngs) : 1;
    const bool fuse_ok = fuse && passes == 1 && ctx->coop && smem_for(ngs) <= budget;
    A.dyn = (fuse_ok && !getenv("EWSJF_NO_DYN")) ? 1 : 0;
    // threshold board: one key per (queue, CTA) while G >= 2K
    A.board = ctx->board;
    A.board_m = 0;
    if (fuse_ok && select && 2 * K <= ctx->num_sms && ctx->num_sms <= 320 && getenv("EWSJF_BOARD")) A.board_m = 1;
    for (int p = 0; p < passes; p++) {
        A.pass0 = p == 0;
        A.g_lo = select ? std::min(nslots, p * ngs) : 0;
        A.g_hi = select ? std::min(nslots, (p + 1) * ngs) : 0;
        cudaError_t e;
        {
            LaunchScope ls(ctx, KIND_TICK);
            e = launch_partial(A, P, fuse_ok ? fuse : nullptr, route, has_cost, use_lut, ctx->num_sms, ctx->stream);
        }
        if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "tick kernel: %s", cudaGetErrorString(e));
    }
    if (fused) *fused = fuse_ok;
    return EWSJF_OK;
}

static MergeArgs merge_args(ewsjf_ctx* ctx, const ewsjf_partition_t* part, const ewsjf_select_params* sp,
                            const ewsjf_meta* theta, int32_t bubble_width) {
    MergeArgs M;
    memset(&M, 0, sizeof M);
    M.K = sp ? sp->k : 1;
    M.nq = part->n;
    M.next_id = part->next_id;
    M.bubble_width = bubble_width;
    M.ex_gap = ctx->ex_gap;
    M.sp = sp ? score_params(sp) : ScoreParams{0.f, 0.f, 0.f, 0.f, 0, 1};
    if (theta) {
        M.theta[0] = theta->a_b; M.theta[1] = theta->b_b; M.theta[2] = theta->a_u;
        M.theta[3] = theta->b_u; M.theta[4] = theta->a_f; M.theta[5] = theta->b_f;
    }
    M.rows = ctx->rows;
    M.rows.cap = M.K;
    M.ctr = ctx->ctr;
    M.gap = ctx->gap;
    M.gap_cap = ctx->gap_cap;
    M.g_slot = ctx->g_slot; M.g_res = ctx->g_res; M.g_u0 = ctx->g_u0; M.g_u1 = ctx->g_u1; M.g_tab = ctx->g_tab;
    M.seq = ++ctx->merge_seq;
    M.gthr = ctx->gthr;
    M.blog = ctx->d_blog;
    M.dbg = getenv("EWSJF_PHASES") ? ctx->dbg : nullptr;
    return M;
}

static int merge_grid(ewsjf_ctx* ctx, int nq, bool may_bubble) {
    int g = nq + (may_bubble ? 8 : 0);
    g = std::max(g, 1);
    return std::min(g, ctx->num_sms);
}

// Replay the device bubble log into the host partition.
static void apply_bubbles(const BubbleLog* log, ewsjf_partition_t* part) {
    if (!log || log->n <= 0) return;
    for (int b = 0; b < log->n; b++) {
        const int pos = log->pos[b];
        for (int i = part->n; i > pos; i--) part->q[i] = part->q[i - 1];
        ewsjf_queue& q = part->q[pos];
        memset(&q, 0, sizeof q);
        q.id = part->next_id++;
        q.min_len = log->lo[b];
        q.max_len = log->hi[b];
        q.mean = (double)log->L[b];
        q.is_bubble = 1;
        part->n++;
    }
    for (int i = 0; i < part->n; i++) part->q[i].index = i + 1;
    part->version++;
}

static ewsjf_status finish_sync(ewsjf_ctx* ctx, ewsjf_partition_t* part_update, ewsjf_summary* h_out,
                                const ewsjf_summary* d_sum) {
    CU(cudaMemcpyAsync(ctx->h_summary, d_sum, sizeof(ewsjf_summary), cudaMemcpyDeviceToHost, ctx->stream));
    if (part_update) CU(cudaMemcpyAsync(ctx->h_blog, ctx->d_blog, sizeof(BubbleLog), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (h_out) *h_out = *ctx->h_summary;
    if (part_update && ctx->h_summary->n_bubbles > 0) apply_bubbles(ctx->h_blog, part_update);
    return (ewsjf_status)ctx->h_summary->status;
}

static ewsjf_status check_out(ewsjf_ctx* ctx, const ewsjf_select_out* out) {
    if (!out || !out->d_topk_id || !out->d_topk_score || !out->d_count || !out->d_head_id || !out->d_head_score ||
        !out->d_max_score)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "select outputs must all be non-NULL device buffers");
    return EWSJF_OK;
}

// The fused streaming tick (ftick.cu) when the pool and partition allow it:
// <= 64 queues, 16-byte aligned pool, cooperative launch.  merge_mode 1 =
// final outputs (M: OUT_FINAL), 2 = exchange record (M: OUT_EXCHANGE).
// Returns false (nothing launched) when not eligible.
static bool run_ftick(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arr, const float* d_cost,
                      int32_t* d_qid_out, int64_t n, int64_t gbase, const ewsjf_partition_t* part, const Policy& P,
                      const ewsjf_select_params* sp, MergeArgs& M, int merge_mode, ewsjf_status* st) {
    const int nslots = part->n;
    const bool has_cost = d_cost != nullptr;
    if (getenv("EWSJF_OLD_TICK") || getenv("EWSJF_NO_FTICK") || !ctx->coop || nslots < 1 || nslots > 64 || ctx->num_sms > 160 ||
        ctx->num_sms < nslots || n >= (1ll << 37))   // tile indices are 32-bit in the fused kernel
        return false;
    if (!aligned16(d_len) || !aligned16(d_arr) || (has_cost && !aligned16(d_cost)) ||
        (d_qid_out && !aligned16(d_qid_out)))
        return false;
    const int K = sp->k;
    const int lutsz = std::min(part->q[nslots - 1].max_len, kLutCap);
    int stages = 3;       // measured: 3 stages 66.5 us, 4 stages 68.1 us at C3 (the 4th delays the sample chunk)
    if (const char* e = getenv("EWSJF_STAGES")) stages = std::max(2, std::min(4, atoi(e)));
    const int budget = ctx->smem_optin > 0 ? ctx->smem_optin : 232448;
    while (stages > 2 && ftick_smem_bytes(has_cost, lutsz, nslots, stages) > budget) stages--;
    if (ftick_smem_bytes(has_cost, lutsz, nslots, stages) > budget || merge_smem_total(MERGE_IN_ROWS) > budget)
        return false;
    if ((*st = ensure_lut(ctx, part, lutsz)) != EWSJF_OK) return true;
    if ((*st = ensure_policy(ctx, P)) != EWSJF_OK) return true;
    FArgs A;
    memset(&A, 0, sizeof A);
    A.len = d_len; A.arrival = d_arr; A.cost = d_cost; A.qid_out = d_qid_out;
    A.n = n;
    A.gbase = (uint32_t)gbase;
    A.nslots = nslots;
    A.K = K;
    A.RC = ctx->f_rc;
    A.HWM = ctx->f_rc * 3 / 4;
    A.lut_size = lutsz;
    A.stages = stages;
    A.l2_prefetch = 0;    // measured: no gain at C3 (EWSJF_L2PF)
    if (const char* e = getenv("EWSJF_L2PF")) A.l2_prefetch = std::max(0, atoi(e));
    A.diag = getenv("EWSJF_DIAG") ? atoi(getenv("EWSJF_DIAG")) : 0;
    A.sample_first = getenv("EWSJF_SAMPLE_FIRST") ? atoi(getenv("EWSJF_SAMPLE_FIRST")) : 1;   // measured: -0.7 us (C3 balanced)
    A.dyn_tail = getenv("EWSJF_DYN_TAIL") ? std::max(0, atoi(getenv("EWSJF_DYN_TAIL"))) : 2;
    A.l2_hint = getenv("EWSJF_L2_HINT") ? atoi(getenv("EWSJF_L2_HINT")) : 1;   // measured -0.45 us at C3
    A.cnt_flush = 62;     // a u8 counter gains <= 4 per iteration: (1 + 62) * 4 <= 255
    if (const char* e = getenv("EWSJF_CNT_FLUSH")) A.cnt_flush = std::max(1, std::min(62, atoi(e)));
    const int G = ctx->num_sms;
    // sample board: each CTA's top key per queue when G >= 2K (the bound's descent then runs
    // over G keys per queue instead of 2G), its top two otherwise
    A.board_m = 2 * K <= G ? 1 : 2;
    if (const char* e = getenv("EWSJF_BOARD_M")) A.board_m = std::max(0, std::min(2, atoi(e)));
    if (G * A.board_m < K || G * A.board_m > 320) A.board_m = 0;
    A.merge = merge_mode;
    A.lut_dev = ctx->d_lut;
    A.sp = score_params(sp);
    A.rows = ctx->rows;
    A.rows.keys = ctx->f_rows;
    A.rows.cap = ctx->f_rc;
    A.gthr = ctx->gthr;
    A.board = ctx->board;
    A.rboard = ctx->board + (size_t)64 * G * 2;      // [64][G] after the sample board [64][G][<=2]
    // progressive bound refresh (mid-stream board of CTA maxima): off by default -- the
    // refreshing warp held its ring stage for the board's L2 round trip and stalled the
    // CTA's pipeline (measured C3 68.4 -> 64.1 us without it, K=1 67.4 -> 60.6, balanced
    // 76.3 -> 73.9, FIFO 84.0 -> 76.5; never slower); EWSJF_REFRESH=1 turns it on
    A.refresh = (K <= G && G <= 160 && merge_mode != 0 && getenv("EWSJF_REFRESH") && atoi(getenv("EWSJF_REFRESH")))
                    ? 1 : 0;
    A.ovf_keys = ctx->f_ovf_keys;
    A.ovf_code = ctx->f_ovf_code;
    A.gap = ctx->gap;
    A.gap_cap = ctx->gap_cap;
    A.ctr = ctx->ctr;
    A.dbg = getenv("EWSJF_PHASES") ? ctx->dbg : nullptr;
    A.topk_id = M.topk_id; A.topk_score = M.topk_score; A.count = M.count;
    A.head_id = M.head_id; A.head_score = M.head_score; A.max_score = M.max_score;
    A.summary = M.summary;
    M.rows.keys = ctx->f_rows;
    M.rows.cap = ctx->f_rc;
    cudaError_t e;
    {
        LaunchScope ls(ctx, KIND_TICK);
        e = launch_ftick(A, (const Policy*)ctx->d_policy, M, has_cost, G, ctx->stream);
    }
    *st = e == cudaSuccess ? EWSJF_OK : fail(ctx, EWSJF_ERR_CUDA, "fused tick kernel: %s", cudaGetErrorString(e));
    return true;
}

static ewsjf_status tick_impl(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arr, const float* d_cost, int64_t n,
                              int64_t gbase, ewsjf_partition_t* part, int32_t bubble_width, const ewsjf_meta* theta,
                              const ewsjf_select_params* sp, int32_t* d_qid_out, const ewsjf_select_out* out) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    ewsjf_status s;
    if ((s = check_partition(ctx, part)) != EWSJF_OK) return s;
    if ((s = check_select(ctx, sp)) != EWSJF_OK) return s;
    if ((s = check_out(ctx, out)) != EWSJF_OK) return s;
    if (!theta) return fail(ctx, EWSJF_ERR_INVALID_ARG, "null theta");
    if (bubble_width < 1) return fail(ctx, EWSJF_ERR_INVALID_ARG, "bubble_width < 1");
    if (n < 0 || (n > 0 && (!d_len || !d_arr))) return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad pool");
    if (gbase < 0 || gbase + n >= 0xffffffffll) return fail(ctx, EWSJF_ERR_INVALID_ARG, "global ids must be < 2^32-1");
    CU(cudaSetDevice(ctx->device));
    ewsjf_weights w[EWSJF_MAX_QUEUES];
    ewsjf_weights_from_meta(theta, part, w);
    static thread_local Policy P;
    fill_policy(part, w, &P);
    MergeArgs M = merge_args(ctx, part, sp, theta, bubble_width);
    M.in_mode = MERGE_IN_ROWS;
    M.out_mode = MERGE_OUT_FINAL;
    M.len = d_len; M.arrival = d_arr; M.cost = d_cost;
    M.gbase = (uint32_t)gbase;
    M.n_local = n;
    M.topk_id = out->d_topk_id; M.topk_score = out->d_topk_score; M.count = out->d_count;
    M.head_id = out->d_head_id; M.head_score = out->d_head_score; M.max_score = out->d_max_score;
    M.summary = out->d_summary ? out->d_summary : ctx->d_summary;
    M.qid = d_qid_out;
    bool fused = false;
    if (run_ftick(ctx, d_len, d_arr, d_cost, d_qid_out, n, gbase, part, P, sp, M, 1, &s)) {
        if (s != EWSJF_OK) return s;
        fused = true;
    } else if ((s = run_partial(ctx, d_len, d_arr, d_cost, nullptr, d_qid_out, n, gbase, part, P, sp, true, true, &M,
                                &fused)) != EWSJF_OK) {
        return s;
    }
    if (!fused) {
        cudaError_t e;
        {
            LaunchScope ls(ctx, KIND_MERGE);
            e = launch_merge(M, P, d_cost != nullptr, merge_grid(ctx, part->n, true), ctx->stream);
        }
        if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "merge kernel: %s", cudaGetErrorString(e));
    }
    if (out->h_summary) return finish_sync(ctx, part, out->h_summary, M.summary);
    return EWSJF_OK;
}

static ewsjf_status sharded_impl(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arr, const float* d_cost,
                                 int64_t n, int64_t gbase, ewsjf_partition_t* part, int32_t bubble_width,
                                 const ewsjf_meta* theta, const ewsjf_select_params* sp, int32_t* d_qid_out,
                                 const ewsjf_select_out* out);

extern "C" ewsjf_status ewsjf_tick(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arrival, const float* d_cost,
                                   int64_t n, int64_t global_base, ewsjf_partition_t* part, int32_t bubble_width,
                                   const ewsjf_meta* theta, const ewsjf_select_params* params, int32_t* d_qid_out,
                                   ewsjf_select_out* out) {
    if (ctx && ctx->nccl_comm)
        return sharded_impl(ctx, d_len, d_arrival, d_cost, n, global_base, part, bubble_width, theta, params,
                            d_qid_out, out);
    return tick_impl(ctx, d_len, d_arrival, d_cost, n, global_base, part, bubble_width, theta, params, d_qid_out, out);
}

static ewsjf_status local_impl(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arrival, const float* d_cost,
                               int64_t n, int64_t global_base, const ewsjf_partition_t* part,
                               const ewsjf_meta* theta, const ewsjf_select_params* sp, int32_t* d_qid_out,
                               void* d_exchange);
static ewsjf_status merge_impl(ewsjf_ctx* ctx, const void* d_exchange_all, int32_t world, int64_t global_base,
                               int64_t n_local, int32_t* d_qid_local, ewsjf_partition_t* part, int32_t bubble_width,
                               const ewsjf_meta* theta, const ewsjf_select_params* sp, const ewsjf_select_out* out);

// Host-buffer tick, pipelined (pools >= kPipeMinPool): the pool goes up in P chunks on
// h2d_st; chunk i's local tick (route + score + per-queue reduction into exchange
// record i, the sharded tick's record) runs on the ctx stream as soon as its copy has
// landed, and its qid slice goes back on d2h_st while the next chunk is in flight; one
// merge of the P records gives the tick's result.  The PCIe copies of the two directions
// overlap each other and the kernels (serial: H2D, kernel, D2H back to back).  A result
// the exchange records cannot carry (more gap requests than their capacity) is redone
// by the single-pass tick over the pool now resident on the device.
static ewsjf_status tick_host_pipelined(ewsjf_ctx* ctx, const int32_t* h_len, const float* h_arrival,
                                        const float* h_cost, int64_t n, int64_t global_base, ewsjf_partition_t* part,
                                        int32_t bubble_width, const ewsjf_meta* theta,
                                        const ewsjf_select_params* params, int32_t* h_qid_out, bool* done,
                                        bool* on_device) {
    *done = false;
    *on_device = false;
    if (n < kPipeMinPool || !ctx->ex_pipe || part->n < 1 || part->n > 64 || getenv("EWSJF_NO_PIPE")) return EWSJF_OK;
    const int64_t per = ex_layout(part->n, params->k, ctx->ex_gap).total;
    if (per > ctx->ex_pipe_per) return EWSJF_OK;
    const int P = (int)std::min<int64_t>(ewsjf_ctx::kPipeMax, n / (kPipeMinPool / 2));
    const int64_t step = ((n + P - 1) / P + 4095) & ~(int64_t)4095;     // 16-byte aligned chunk starts
    cudaStream_t st = ctx->stream;
    CU(cudaEventRecord(ctx->pipe_start, st));                     // earlier work on the ctx buffers
    CU(cudaStreamWaitEvent(ctx->h2d_st, ctx->pipe_start, 0));
    CU(cudaStreamWaitEvent(ctx->d2h_st, ctx->pipe_start, 0));
    int nc = 0;
    for (int i = 0; i < P; i++) {
        const int64_t off = (int64_t)i * step, m = std::min<int64_t>(step, n - off);
        if (m <= 0) break;
        nc++;
        CU(cudaMemcpyAsync(ctx->d_len + off, h_len + off, (size_t)m * 4, cudaMemcpyHostToDevice, ctx->h2d_st));
        CU(cudaMemcpyAsync(ctx->d_arr + off, h_arrival + off, (size_t)m * 4, cudaMemcpyHostToDevice, ctx->h2d_st));
        if (h_cost) CU(cudaMemcpyAsync(ctx->d_cost + off, h_cost + off, (size_t)m * 4, cudaMemcpyHostToDevice, ctx->h2d_st));
        CU(cudaEventRecord(ctx->pipe_h2d[i], ctx->h2d_st));
        CU(cudaStreamWaitEvent(st, ctx->pipe_h2d[i], 0));
        ewsjf_status s = local_impl(ctx, ctx->d_len + off, ctx->d_arr + off, h_cost ? ctx->d_cost + off : nullptr, m,
                                    global_base + off, part, theta, params, ctx->d_qid + off,
                                    ctx->ex_pipe + (size_t)i * per);
        if (s != EWSJF_OK) return s;
        CU(cudaEventRecord(ctx->pipe_cmp[i], st));
        if (h_qid_out) {
            CU(cudaStreamWaitEvent(ctx->d2h_st, ctx->pipe_cmp[i], 0));
            CU(cudaMemcpyAsync(h_qid_out + off, ctx->d_qid + off, (size_t)m * 4, cudaMemcpyDeviceToHost, ctx->d2h_st));
        }
    }
    ewsjf_select_out out{ctx->d_topk_id, ctx->d_topk_score, ctx->d_count, ctx->d_head_id, ctx->d_head_score,
                         ctx->d_max_score, ctx->d_summary, nullptr};
    ewsjf_status s = merge_impl(ctx, ctx->ex_pipe, nc, global_base, n, ctx->d_qid, part, bubble_width, theta, params,
                                &out);
    if (s != EWSJF_OK) return s;
    CU(cudaEventRecord(ctx->pipe_d2h, ctx->d2h_st));
    CU(cudaStreamWaitEvent(st, ctx->pipe_d2h, 0));                // the qid slices are back before the ctx stream moves on
    *on_device = true;
    *done = true;            // the caller checks the summary (capacity -> single pass over the resident pool)
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_tick_host(ewsjf_ctx* ctx, const int32_t* h_len, const float* h_arrival,
                                        const float* h_cost, int64_t n, int64_t global_base, ewsjf_partition_t* part,
                                        int32_t bubble_width, const ewsjf_meta* theta,
                                        const ewsjf_select_params* params, int32_t* h_qid_out, int64_t* h_topk_id,
                                        float* h_topk_score, int64_t* h_count, int64_t* h_head_id,
                                        float* h_head_score, float* h_max_score, ewsjf_summary* h_summary) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (!h_summary) return fail(ctx, EWSJF_ERR_INVALID_ARG, "h_summary required");
    if (n < 0 || n > ctx->max_pool) return fail(ctx, EWSJF_ERR_INVALID_ARG, "n=%lld > max_pool", (long long)n);
    if (n > 0 && (!h_len || !h_arrival)) return fail(ctx, EWSJF_ERR_INVALID_ARG, "null host pool");
    CU(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    bool piped = false, on_device = false;
    {
        ewsjf_status ps = tick_host_pipelined(ctx, h_len, h_arrival, h_cost, n, global_base, part, bubble_width, theta,
                                              params, h_qid_out, &piped, &on_device);
        if (ps != EWSJF_OK) return ps;
    }
    const int K = params->k;
    auto copy_results = [&]() -> ewsjf_status {
        if (h_topk_id) CU(cudaMemcpyAsync(h_topk_id, ctx->d_topk_id, (size_t)kMaxSlots * K * 8, cudaMemcpyDeviceToHost, st));
        if (h_topk_score)
            CU(cudaMemcpyAsync(h_topk_score, ctx->d_topk_score, (size_t)kMaxSlots * K * 4, cudaMemcpyDeviceToHost, st));
        if (h_count) CU(cudaMemcpyAsync(h_count, ctx->d_count, kMaxSlots * 8, cudaMemcpyDeviceToHost, st));
        if (h_head_id) CU(cudaMemcpyAsync(h_head_id, ctx->d_head_id, kMaxSlots * 8, cudaMemcpyDeviceToHost, st));
        if (h_head_score) CU(cudaMemcpyAsync(h_head_score, ctx->d_head_score, kMaxSlots * 4, cudaMemcpyDeviceToHost, st));
        if (h_max_score) CU(cudaMemcpyAsync(h_max_score, ctx->d_max_score, kMaxSlots * 4, cudaMemcpyDeviceToHost, st));
        return EWSJF_OK;
    };
    if (piped) {
        // one synchronisation: results, summary and bubble log together; a capacity
        // overflow of the exchange records falls through to the single pass below
        ewsjf_status cs = copy_results();
        if (cs != EWSJF_OK) return cs;
        CU(cudaMemcpyAsync(ctx->h_summary, ctx->d_summary, sizeof(ewsjf_summary), cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(ctx->h_blog, ctx->d_blog, sizeof(BubbleLog), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (ctx->h_summary->status != EWSJF_ERR_CAPACITY) {
            if (ctx->h_summary->n_gap > 0 && h_qid_out) {   // Alg. 2 rewrote gap requests' qid after the copies
                CU(cudaMemcpyAsync(h_qid_out, ctx->d_qid, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
                CU(cudaStreamSynchronize(st));
            }
            *h_summary = *ctx->h_summary;
            if (ctx->h_summary->n_bubbles > 0) apply_bubbles(ctx->h_blog, part);
            return (ewsjf_status)ctx->h_summary->status;
        }
        piped = false;
    }
    if (!piped) {
        if (n > 0 && !on_device) {
            CU(cudaMemcpyAsync(ctx->d_len, h_len, (size_t)n * 4, cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(ctx->d_arr, h_arrival, (size_t)n * 4, cudaMemcpyHostToDevice, st));
            if (h_cost) CU(cudaMemcpyAsync(ctx->d_cost, h_cost, (size_t)n * 4, cudaMemcpyHostToDevice, st));
        }
        ewsjf_select_out out{ctx->d_topk_id, ctx->d_topk_score, ctx->d_count, ctx->d_head_id, ctx->d_head_score,
                             ctx->d_max_score, ctx->d_summary, nullptr};
        ewsjf_status s = tick_impl(ctx, ctx->d_len, ctx->d_arr, h_cost ? ctx->d_cost : nullptr, n, global_base, part,
                                   bubble_width, theta, params, ctx->d_qid, &out);
        if (s != EWSJF_OK) return s;
        if (h_qid_out && n > 0) CU(cudaMemcpyAsync(h_qid_out, ctx->d_qid, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    }
    {
        ewsjf_status cs = copy_results();
        if (cs != EWSJF_OK) return cs;
    }
    return finish_sync(ctx, part, h_summary, ctx->d_summary);
}

extern "C" ewsjf_status ewsjf_score_select(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arrival,
                                           const float* d_cost, const int32_t* d_qid, int64_t n,
                                           const ewsjf_partition_t* part, const ewsjf_weights* w,
                                           const ewsjf_select_params* sp, ewsjf_select_out* out) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    ewsjf_status s;
    if ((s = check_partition(ctx, part)) != EWSJF_OK) return s;
    if ((s = check_select(ctx, sp)) != EWSJF_OK) return s;
    if ((s = check_out(ctx, out)) != EWSJF_OK) return s;
    if (!w) return fail(ctx, EWSJF_ERR_INVALID_ARG, "null weights");
    if (n < 0 || (n > 0 && (!d_len || !d_arrival || !d_qid))) return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad pool");
    if (n >= 0xffffffffll) return fail(ctx, EWSJF_ERR_INVALID_ARG, "pool too large");
    for (int i = 0; i < part->n; i++)
        if (!(w[i].w_base >= 0.f && w[i].w_urg >= 0.f && w[i].w_fair >= 0.f))
            return fail(ctx, EWSJF_ERR_INVALID_ARG, "weights must be >= 0 (S:306)");
    CU(cudaSetDevice(ctx->device));
    static thread_local Policy P;
    fill_policy(part, w, &P);
    MergeArgs M = merge_args(ctx, part, sp, nullptr, 1);
    M.in_mode = MERGE_IN_ROWS;
    M.out_mode = MERGE_OUT_FINAL;
    M.len = d_len; M.arrival = d_arrival; M.cost = d_cost;
    M.n_local = n;
    M.topk_id = out->d_topk_id; M.topk_score = out->d_topk_score; M.count = out->d_count;
    M.head_id = out->d_head_id; M.head_score = out->d_head_score; M.max_score = out->d_max_score;
    M.summary = out->d_summary ? out->d_summary : ctx->d_summary;
    M.blog = nullptr;
    bool fused = false;
    if ((s = run_partial(ctx, d_len, d_arrival, d_cost, d_qid, nullptr, n, 0, part, P, sp, false, true, &M,
                         &fused)) != EWSJF_OK)
        return s;
    if (!fused) {
        cudaError_t e;
        {
            LaunchScope ls(ctx, KIND_MERGE);
            e = launch_merge(M, P, d_cost != nullptr, merge_grid(ctx, part->n, false), ctx->stream);
        }
        if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "merge kernel: %s", cudaGetErrorString(e));
    }
    if (out->h_summary) return finish_sync(ctx, nullptr, out->h_summary, M.summary);
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_route(ewsjf_ctx* ctx, const int32_t* d_len, int64_t n, ewsjf_partition_t* part,
                                    int32_t bubble_width, int32_t* d_qid, ewsjf_summary* h_summary) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    ewsjf_status s;
    if ((s = check_partition(ctx, part)) != EWSJF_OK) return s;
    if (bubble_width < 1) return fail(ctx, EWSJF_ERR_INVALID_ARG, "bubble_width < 1");
    if (n < 0 || (n > 0 && (!d_len || !d_qid))) return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad pool");
    if (n >= 0xffffffffll) return fail(ctx, EWSJF_ERR_INVALID_ARG, "pool too large");
    CU(cudaSetDevice(ctx->device));
    ewsjf_weights w[EWSJF_MAX_QUEUES];
    memset(w, 0, sizeof w);
    static thread_local Policy P;
    fill_policy(part, w, &P);
    // route-only pass: arrival is not read (the TMA path loads it; pass len as a dummy 16B-aligned source)
    if ((s = run_partial(ctx, d_len, (const float*)d_len, nullptr, nullptr, d_qid, n, 0, part, P, nullptr, true,
                         false)) != EWSJF_OK)
        return s;
    MergeArgs M = merge_args(ctx, part, nullptr, nullptr, bubble_width);
    M.in_mode = MERGE_IN_ROWS;
    M.out_mode = MERGE_OUT_ROUTE;
    M.n_local = n;
    M.qid = d_qid;
    M.summary = ctx->d_summary;
    cudaError_t e;
    {
        LaunchScope ls(ctx, KIND_MERGE);
        e = launch_merge(M, P, false, 1, ctx->stream);
    }
    if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "merge kernel: %s", cudaGetErrorString(e));
    ewsjf_summary tmp;
    return finish_sync(ctx, part, h_summary ? h_summary : &tmp, ctx->d_summary);
}

// ---------------------------------------------------------- sharded tick ---
extern "C" int64_t ewsjf_exchange_bytes(const ewsjf_ctx* ctx, int32_t n_queues, int32_t k) {
    if (n_queues < 0 || n_queues > EWSJF_MAX_QUEUES || k < 1 || k > EWSJF_MAX_K) return -1;
    return ex_layout(n_queues, k, ctx ? ctx->ex_gap : kExGapDefault).total;
}

static ewsjf_status local_impl(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arrival, const float* d_cost,
                               int64_t n, int64_t global_base, const ewsjf_partition_t* part,
                               const ewsjf_meta* theta, const ewsjf_select_params* sp, int32_t* d_qid_out,
                               void* d_exchange) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    ewsjf_status s;
    if ((s = check_partition(ctx, part)) != EWSJF_OK) return s;
    if ((s = check_select(ctx, sp)) != EWSJF_OK) return s;
    if (!theta || !d_exchange || ((uintptr_t)d_exchange & 255)) return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad theta/exchange");
    if (n < 0 || (n > 0 && (!d_len || !d_arrival))) return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad pool");
    if (global_base < 0 || global_base + n >= 0xffffffffll) return fail(ctx, EWSJF_ERR_INVALID_ARG, "ids >= 2^32-1");
    CU(cudaSetDevice(ctx->device));
    ewsjf_weights w[EWSJF_MAX_QUEUES];
    ewsjf_weights_from_meta(theta, part, w);
    static thread_local Policy P;
    fill_policy(part, w, &P);
    CU(cudaMemsetAsync(d_exchange, 0, ex_layout(part->n, sp->k, ctx->ex_gap).total, ctx->stream));
    MergeArgs M = merge_args(ctx, part, sp, theta, 1);
    M.in_mode = MERGE_IN_ROWS;
    M.out_mode = MERGE_OUT_EXCHANGE;
    M.len = d_len; M.arrival = d_arrival; M.cost = d_cost;
    M.gbase = (uint32_t)global_base;
    M.n_local = n;
    M.ex_out = (unsigned char*)d_exchange;
    M.blog = nullptr;
    // the fused kernel writes the exchange record itself (merge_phase after its grid barrier)
    if (run_ftick(ctx, d_len, d_arrival, d_cost, d_qid_out, n, global_base, part, P, sp, M, 2, &s)) return s;
    if ((s = run_partial(ctx, d_len, d_arrival, d_cost, nullptr, d_qid_out, n, global_base, part, P, sp, true,
                         true)) != EWSJF_OK)
        return s;
    cudaError_t e;
    {
        LaunchScope ls(ctx, KIND_MERGE);
        e = launch_merge(M, P, d_cost != nullptr, merge_grid(ctx, part->n, false), ctx->stream);
    }
    if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "local reduce: %s", cudaGetErrorString(e));
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_tick_local(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arrival,
                                         const float* d_cost, int64_t n, int64_t global_base,
                                         const ewsjf_partition_t* part, const ewsjf_meta* theta,
                                         const ewsjf_select_params* sp, int32_t* d_qid_out, void* d_exchange) {
    return local_impl(ctx, d_len, d_arrival, d_cost, n, global_base, part, theta, sp, d_qid_out, d_exchange);
}

static ewsjf_status merge_impl(ewsjf_ctx* ctx, const void* d_exchange_all, int32_t world, int64_t global_base,
                               int64_t n_local, int32_t* d_qid_local, ewsjf_partition_t* part, int32_t bubble_width,
                               const ewsjf_meta* theta, const ewsjf_select_params* sp, const ewsjf_select_out* out) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    ewsjf_status s;
    if ((s = check_partition(ctx, part)) != EWSJF_OK) return s;
    if ((s = check_select(ctx, sp)) != EWSJF_OK) return s;
    if ((s = check_out(ctx, out)) != EWSJF_OK) return s;
    if (!theta || !d_exchange_all || world < 1 || world > 1024 || bubble_width < 1)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad merge arguments");
    CU(cudaSetDevice(ctx->device));
    ewsjf_weights w[EWSJF_MAX_QUEUES];
    ewsjf_weights_from_meta(theta, part, w);
    static thread_local Policy P;
    fill_policy(part, w, &P);
    MergeArgs M = merge_args(ctx, part, sp, theta, bubble_width);
    M.in_mode = MERGE_IN_EXCHANGE;
    M.out_mode = MERGE_OUT_FINAL;
    M.ex_in = (const unsigned char*)d_exchange_all;
    M.world = world;
    M.ex_bytes = ex_layout(part->n, sp->k, ctx->ex_gap).total;
    M.gbase = (uint32_t)global_base;
    M.n_local = n_local;
    M.qid = d_qid_local;
    M.topk_id = out->d_topk_id; M.topk_score = out->d_topk_score; M.count = out->d_count;
    M.head_id = out->d_head_id; M.head_score = out->d_head_score; M.max_score = out->d_max_score;
    M.summary = out->d_summary ? out->d_summary : ctx->d_summary;
    cudaError_t e;
    {
        LaunchScope ls(ctx, KIND_MERGE);
        e = launch_merge(M, P, false, merge_grid(ctx, part->n, true), ctx->stream);
    }
    if (e != cudaSuccess) return fail(ctx, EWSJF_ERR_CUDA, "global merge: %s", cudaGetErrorString(e));
    if (out->h_summary) return finish_sync(ctx, part, out->h_summary, M.summary);
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_tick_merge(ewsjf_ctx* ctx, const void* d_exchange_all, int32_t world,
                                         int64_t global_base, int64_t n_local, int32_t* d_qid_local,
                                         ewsjf_partition_t* part, int32_t bubble_width, const ewsjf_meta* theta,
                                         const ewsjf_select_params* sp, ewsjf_select_out* out) {
    return merge_impl(ctx, d_exchange_all, world, global_base, n_local, d_qid_local, part, bubble_width, theta, sp,
                      out);
}

// The index-sharded tick through the ctx's NCCL communicator:
// local route + score + per-queue reduction into a fixed-size exchange record,
// ncclAllGather of the records on the ctx stream, the same deterministic merge
// on every rank.  No host synchronisation unless out->h_summary is set.
static ewsjf_status sharded_impl(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arr, const float* d_cost,
                                 int64_t n, int64_t gbase, ewsjf_partition_t* part, int32_t bubble_width,
                                 const ewsjf_meta* theta, const ewsjf_select_params* sp, int32_t* d_qid_out,
                                 const ewsjf_select_out* out) {
    ewsjf_status s;
    if ((s = check_partition(ctx, part)) != EWSJF_OK) return s;
    if ((s = check_select(ctx, sp)) != EWSJF_OK) return s;
    if ((s = check_out(ctx, out)) != EWSJF_OK) return s;
    if (sp->k > ctx->max_k) return fail(ctx, EWSJF_ERR_INVALID_ARG, "k > ctx max_k");
    const int64_t bytes = ex_layout(part->n, sp->k, ctx->ex_gap).total;
    if (bytes > ctx->ex_cap) return fail(ctx, EWSJF_ERR_CAPACITY, "exchange record %lld > %lld", (long long)bytes,
                                         (long long)ctx->ex_cap);
    if ((s = local_impl(ctx, d_len, d_arr, d_cost, n, gbase, part, theta, sp, d_qid_out, ctx->ex_local)) != EWSJF_OK)
        return s;
    if ((s = nccl_allgather(ctx, bytes)) != EWSJF_OK) return s;
    return merge_impl(ctx, ctx->ex_all, ctx->nccl_world, gbase, n, d_qid_out, part, bubble_width, theta, sp, out);
}
