// batch.cu — Alg. 1 Batch Builder
// and the empty-queue pruning of lines 8-12 (host bookkeeping).
//
// Input: one FIFO-mode selection (ewsjf_tick / ewsjf_score_select with
// mode = FIFO): per queue position p its k oldest members (arrival, id) best
// first, its member count, and the summary's ArgMax position (the primary).
// With k >= max_requests every queue's FIFO prefix the builder can pull is
// present in its row, so the batch equals Alg. 1 over the whole pool (R28-R29).
//
// One CTA (kBThreads threads), three phases:
//   1. every warp takes queues p = warp, warp + 32, …: the inclusive prefix of
//      the row's prompt lengths (warp scan, int64 carry) saturated to u32 into
//      scratch — the budget test "tokens + prefix <= max_tokens" is monotone
//      in the row position (lengths >= 1), so one ballot per 32 entries
//      answers "how many of this queue fit";
//   2. warp 0 walks the visiting order primary, p-1, p+1, p-2, p+2, … (R29):
//      j = #entries with prefix <= max_tokens - tokens (the first request of
//      an empty batch is always admitted), capped by max_requests;
//   3. all warps copy the admitted ids (queue row prefixes) into the batch.
// max_tokens < 2^32 - 1 keeps the saturated prefixes exact for every test
// (a saturated entry never fits).
#include <climits>
#include <algorithm>
#include "tick.cuh"
#include "ctx.h"

namespace ewsjf {

constexpr int kBThreads = 1024;
constexpr int kBPer = 8;                       // row entries per lane per gather pass
constexpr int kBSmemMax = 200 * 1024;          // prefix table in shared memory up to this size

// prefix entries are written by other warps of this CTA before __syncthreads:
// shared memory, or global scratch read past L1 (generic address either way)
__device__ __forceinline__ uint32_t ld_pre(const uint32_t* p) {
    return __isShared(p) ? *p : __ldcg(p);
}

struct BatchArgs {
    const int32_t* len;
    int64_t n, base;
    const int64_t* topk_id;
    const int64_t* count;
    const ewsjf_summary* summary;
    int32_t k, nq, max_req;
    int64_t max_tok;
    uint32_t* pre;          // [nq][kk] global scratch, or nullptr -> dynamic shared memory
    int32_t kk;             // min(k, max_req)
    int64_t* out_id;        // [max_req]
    int64_t* out_info;      // [4]: count, tokens, status, primary
};

__global__ void __launch_bounds__(kBThreads, 1) batch_build_kernel(BatchArgs A) {
    __shared__ int32_t s_m[EWSJF_MAX_QUEUES];
    __shared__ int32_t s_take[EWSJF_MAX_QUEUES];
    __shared__ int32_t s_off[EWSJF_MAX_QUEUES];
    __shared__ int32_t s_bad, s_nb;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // the primary is needed only in phase 2: issue its load now, ahead of the gathers
    const int prim0 = warp == 0 ? __ldg(&A.summary->primary) : 0;
    if (threadIdx.x == 0) { s_bad = 0; s_nb = 0; }
    __syncthreads();
    // ---- phase 1: per-queue prefix of lengths over the FIFO rows.  All of a
    // lane's row ids, then all of its lengths, are loaded before the scans so the
    // dependent gathers overlap (kBPer entries per lane per pass).
    extern __shared__ uint32_t s_dyn[];
    uint32_t* pre = A.pre ? A.pre : s_dyn;
    for (int p = warp; p < A.nq; p += nw) {
        const int64_t c = A.count[p];
        const int m = (int)(c < A.kk ? c : A.kk);
        const int64_t* row = A.topk_id + (int64_t)p * A.k;
        uint32_t* pr = pre + (int64_t)p * A.kk;
        int64_t carry = 0;
        for (int b0 = 0; b0 < m; b0 += 32 * kBPer) {
            int64_t id[kBPer];
            int32_t b[kBPer];
#pragma unroll
            for (int u = 0; u < kBPer; u++) {
                const int t = b0 + u * 32 + lane;
                id[u] = t < m ? __ldg(row + t) : 0;
            }
#pragma unroll
            for (int u = 0; u < kBPer; u++) {
                const int t = b0 + u * 32 + lane;
                const int64_t r = id[u] - A.base;
                b[u] = 0;
                if (t < m) {
                    if (id[u] < 0 || r < 0 || r >= A.n) atomicOr(&s_bad, 1);
                    else b[u] = __ldg(A.len + r);
                }
            }
#pragma unroll
            for (int u = 0; u < kBPer; u++) {
                const int t = b0 + u * 32 + lane;
                int64_t x = b[u];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                x += carry;
                if (t < m) pr[t] = x >= 0xffffffffll ? 0xffffffffu : (uint32_t)x;
                carry = __shfl_sync(0xffffffffu, x, 31);
            }
        }
        if (lane == 0) { s_m[p] = m; s_take[p] = 0; s_off[p] = 0; }
    }
    __syncthreads();
    // ---- phase 2: GreedyFill from the primary, Backfill nearest-first (lower first)
    if (warp == 0) {
        const int prim = prim0;
        int64_t nb = 0, tok = 0;
        if (!s_bad && prim >= 0 && prim < A.nq && A.max_req > 0) {
            for (int d = 0; d < A.nq && nb < A.max_req; d++) {
                for (int side = 0; side < (d == 0 ? 1 : 2) && nb < A.max_req; side++) {
                    const int p = d == 0 ? prim : (side == 0 ? prim - d : prim + d);
                    if (p < 0 || p >= A.nq) continue;
                    const int m = s_m[p];
                    if (m == 0) continue;
                    if (nb > 0 && tok >= A.max_tok) continue;     // nothing of length >= 1 fits
                    const int64_t R = A.max_tok - tok;            // >= 0 unless nb == 0
                    const uint32_t* pr = pre + (int64_t)p * A.kk;
                    int j = 0;
                    for (int t0 = 0; t0 < m; t0 += 32) {
                        const int t = t0 + lane;
                        const bool fit = t < m && (int64_t)ld_pre(pr + t) <= R;
                        const unsigned bal = __ballot_sync(0xffffffffu, fit);
                        j += __popc(bal);
                        if (bal != 0xffffffffu) break;
                    }
                    if (nb == 0 && j == 0) j = 1;                 // the first request is always admitted
                    if (j > A.max_req - nb) j = (int)(A.max_req - nb);
                    if (lane == 0) { s_take[p] = j; s_off[p] = (int)nb; }
                    if (j > 0) tok += (int64_t)ld_pre(pr + j - 1);
                    nb += j;
                }
            }
        }
        if (lane == 0) {
            s_nb = (int)nb;
            A.out_info[0] = nb;
            A.out_info[1] = tok;
            A.out_info[2] = s_bad ? (int64_t)EWSJF_ERR_INVALID_ARG : (int64_t)EWSJF_OK;
            A.out_info[3] = prim;
        }
    }
    __syncthreads();
    // ---- phase 3: copy the admitted FIFO prefixes, pad with -1
    for (int p = warp; p < A.nq; p += nw) {
        const int j = s_take[p];
        const int64_t* row = A.topk_id + (int64_t)p * A.k;
        for (int t = lane; t < j; t += 32) A.out_id[s_off[p] + t] = row[t];
    }
    for (int t = s_nb + threadIdx.x; t < A.max_req; t += blockDim.x) A.out_id[t] = -1;
}

}  // namespace ewsjf

extern "C" ewsjf_status ewsjf_batch_build(ewsjf_ctx* ctx, const int32_t* d_len, int64_t n, int64_t global_base,
                                          const ewsjf_select_out* sel, int32_t k, int32_t n_queues,
                                          const ewsjf_batch_budget* budget, int64_t* d_batch_id,
                                          int64_t* d_batch_info) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (!sel || !budget || !d_batch_id || !d_batch_info || !sel->d_topk_id || !sel->d_count)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "batch_build: null argument");
    if (n_queues < 0 || n_queues > EWSJF_MAX_QUEUES || k < 1 || n < 0 || (n > 0 && !d_len))
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "batch_build: bad n_queues / k / pool");
    if (budget->max_requests < 1 || budget->max_requests > k)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "batch_build: need 1 <= max_requests <= k (FIFO rows deep enough)");
    if (budget->max_tokens < 0 || budget->max_tokens >= 0xffffffffll)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "batch_build: max_tokens out of range [0, 2^32-1)");
    CU(cudaSetDevice(ctx->device));
    const int32_t kk = budget->max_requests;
    const int64_t need = (int64_t)std::max(n_queues, 1) * kk;
    const bool in_smem = need * 4 <= std::min<int64_t>(kBSmemMax, ctx->smem_optin - 4096);
    if (!in_smem && need > ctx->bpre_cap)      // preallocated by ewsjf_ctx_create for 256 queues x max_k
        return fail(ctx, EWSJF_ERR_CAPACITY, "batch_build: %lld prefix entries > ctx capacity %lld (max_k)",
                    (long long)need, (long long)ctx->bpre_cap);
    BatchArgs A;
    A.len = d_len; A.n = n; A.base = global_base;
    A.topk_id = sel->d_topk_id; A.count = sel->d_count;
    A.summary = sel->d_summary ? sel->d_summary : ctx->d_summary;
    A.k = k; A.nq = n_queues; A.max_req = budget->max_requests; A.max_tok = budget->max_tokens;
    A.pre = in_smem ? nullptr : ctx->d_bpre; A.kk = kk;
    const size_t smem = in_smem ? (size_t)need * 4 : 0;
    if (smem > 48 * 1024 && smem > ctx->batch_smem_attr) {
        CU(cudaFuncSetAttribute(batch_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBSmemMax));
        ctx->batch_smem_attr = kBSmemMax;
    }
    A.out_id = d_batch_id; A.out_info = d_batch_info;
    {
        LaunchScope ls(ctx, KIND_BATCH);
        batch_build_kernel<<<1, kBThreads, smem, ctx->stream>>>(A);
    }
    CU(cudaGetLastError());
    return EWSJF_OK;
}

// Alg. 1 lines 8-12: count empty ticks, drop queues whose counter
// exceeds the threshold (strict, R25), renumber the survivors.  The
// counter counts consecutive empty tactical steps: a queue with members
// resets it (R30).  Host bookkeeping over the host partition.
extern "C" ewsjf_status ewsjf_prune_empty(ewsjf_partition_t* part, const int64_t* h_count, int32_t threshold,
                                          int32_t* removed) {
    if (!part || !h_count || part->n < 0 || part->n > EWSJF_MAX_QUEUES || threshold < 0)
        return EWSJF_ERR_INVALID_ARG;
    int32_t k = 0, rm = 0;
    for (int32_t p = 0; p < part->n; p++) {
        ewsjf_queue q = part->q[p];
        q.empty_count = h_count[p] == 0 ? q.empty_count + 1 : 0;
        if (q.empty_count > threshold) { rm++; continue; }
        q.index = k + 1;
        part->q[k++] = q;
    }
    part->n = k;
    if (rm) part->version++;
    if (removed) *removed = rm;
    return EWSJF_OK;
}
