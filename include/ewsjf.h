/*
 * ewsjf.h — C ABI of libewsjf, the B200-native (sm_100a) data-parallel core of
 * one EWSJF scheduling tick (arXiv 2601.21758, "EWSJF").
 *
 * Citation format: P:n = PAPER.md line n, S:n = SPEC.md line n; readings of
 * silent/ambiguous passages R1..R27 are listed in DESIGN.md §3.
 *
 * Conventions (apply to every entry point):
 *  - All functions return ewsjf_status and never throw or abort across the ABI.
 *  - d_ prefix: device pointer (CUDA global memory of the ctx's device),
 *    caller-owned; h_ prefix: host pointer, caller-owned.  The library never
 *    frees caller memory.  Device inputs are read-only unless marked "out".
 *  - Work is enqueued on the ctx's CUDA stream and is asynchronous unless an
 *    h_ output is requested (then the call synchronises the stream).
 *  - EWSJF_ERR_INVALID_ARG: a parameter is out of range; nothing was launched.
 *    EWSJF_ERR_DOMAIN: some elements violated a precondition (len < 1, S:223;
 *    now < arrival; cost <= 0 or NaN; unknown qid); ALL outputs were
 *    written, the offending elements were excluded and counted.
 *    EWSJF_ERR_CAPACITY: more than EWSJF_MAX_QUEUES queues (incl. bubbles) or
 *    the gap list overflowed; outputs are written for what fitted.
 *    EWSJF_ERR_CUDA: a CUDA call failed (message: ewsjf_last_error()).
 *  - Layouts are structure-of-arrays, one element per request, contiguous.
 *    Request ids written by the library are GLOBAL pool indices
 *    (global_base + local index), < 2^32 - 1.
 *  - Per-queue outputs are indexed by queue POSITION (q_i - 1, ascending by
 *    prompt length) of the partition the call ends with, and must be sized for
 *    EWSJF_MAX_QUEUES queues (× k for top-k arrays).
 */
#ifndef EWSJF_H
#define EWSJF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EWSJF_ABI_VERSION 1
#define EWSJF_MAX_QUEUES 256      /* hard cap on queues incl. bubbles */
#define EWSJF_MAX_K 256           /* largest per-queue selection depth */

typedef enum {
    EWSJF_OK = 0,
    EWSJF_ERR_INVALID_ARG = 1,
    EWSJF_ERR_DOMAIN = 2,
    EWSJF_ERR_EMPTY = 3,          /* empty history (no length >= 1)          */
    EWSJF_ERR_CAPACITY = 4,
    EWSJF_ERR_CUDA = 5,
    EWSJF_ERR_UNSUPPORTED = 6,    /* e.g. a history length above the kernel's range */
    EWSJF_ERR_NCCL = 7            /* NCCL unavailable or a collective failed */
} ewsjf_status;

typedef struct ewsjf_ctx ewsjf_ctx;

/* --------------------------------------------------------------- context --- */
int          ewsjf_abi_version(void);
const char  *ewsjf_status_str(ewsjf_status s);
/* Last error message recorded on ctx (static storage owned by ctx). */
const char  *ewsjf_last_error(const ewsjf_ctx *ctx);

/* Create a context on `device`, enqueueing on `cuda_stream` (cudaStream_t, NULL
 * = legacy default stream).  The ctx owns ALL scratch, sized once here for
 * pools of up to max_pool requests, histories of up to max_history lengths
 * and selection depth up to max_k (1..EWSJF_MAX_K): no allocation happens on a
 * later call.  *out receives the ctx.  Not thread-safe; one ctx per stream.  */
ewsjf_status ewsjf_ctx_create(int device, void *cuda_stream, int64_t max_pool, int64_t max_history,
                              int32_t max_k, ewsjf_ctx **out);
/* Switch the ctx to another stream.  The ctx's scratch is shared by all its
 * calls, so the new stream is first made to wait (cudaStreamWaitEvent) for
 * everything already queued on the old one; no host synchronisation. */
ewsjf_status ewsjf_ctx_set_stream(ewsjf_ctx *ctx, void *cuda_stream);
ewsjf_status ewsjf_ctx_destroy(ewsjf_ctx *ctx);
/* ------------------------------------------------------ NCCL (multi-GPU) ---
 * The index-sharded tick (R22 "global index order" across ranks):
 * with a communicator set on the ctx, ewsjf_tick treats d_len/d_arrival/d_cost
 * as this rank's shard (ids global_base + i), runs the local route + score +
 * per-queue reduction into a fixed-size exchange record, ncclAllGather's the
 * records on the ctx stream and runs the same deterministic merge on every
 * rank, so every rank receives the identical global result (outputs, bubbles
 * in *part, primary).  All three steps are stream-ordered (CUDA-graph
 * capturable when no host output is requested).  NCCL is resolved at run time
 * (dlopen "libnccl.so.2": the process's loaded copy, else the system one);
 * EWSJF_ERR_NCCL when it is unavailable or a collective fails.
 *
 * ewsjf_nccl_get_unique_id: one rank creates the id (128 bytes) and the caller
 *   broadcasts it (e.g. over torch.distributed).
 * ewsjf_ctx_init_nccl: ncclCommInitRank on the ctx device; the ctx owns the
 *   communicator (destroyed by ewsjf_ctx_destroy / _detach_nccl).  Collective:
 *   every rank calls it.  Allocates the exchange buffers (256 queues x max_k
 *   per rank) once; no allocation on a later tick.
 * ewsjf_ctx_attach_nccl: use a caller-created ncclComm_t (caller keeps
 *   ownership and must outlive the ctx's use of it).
 * ewsjf_ctx_detach_nccl: synchronise the ctx stream, drop the communicator
 *   (destroy it if owned) and the exchange buffers; ewsjf_tick is single-GPU again. */
#define EWSJF_NCCL_ID_BYTES 128
ewsjf_status ewsjf_nccl_get_unique_id(uint8_t *id_out /* [128] */);
ewsjf_status ewsjf_ctx_init_nccl(ewsjf_ctx *ctx, const uint8_t *id /* [128] */, int32_t rank, int32_t world);
ewsjf_status ewsjf_ctx_attach_nccl(ewsjf_ctx *ctx, void *nccl_comm /* ncclComm_t */, int32_t rank, int32_t world);
ewsjf_status ewsjf_ctx_detach_nccl(ewsjf_ctx *ctx);

/* Number of SMs the ctx launches persistent kernels over (the "CTA rows"). */
int32_t      ewsjf_ctx_num_ctas(const ewsjf_ctx *ctx);

/* Instrumentation (tracing / bench): when enabled, every kernel the ctx launches
 * is bracketed by CUDA events on the ctx stream (up to 16384 launches are
 * recorded; enabling resets the record).  ewsjf_ctx_get_timing synchronises
 * and sums the device time per kernel kind since the last enable.  `launches`
 * counts every libewsjf kernel launched since ctx creation (timing or not).  */
typedef struct {
    int64_t launches;
    int64_t recorded;
    int64_t tick_launches;     /* partial (route/score/select) passes */
    int64_t merge_launches;
    int64_t partition_launches;
    int64_t sweep_launches;
    double  tick_ms, merge_ms, partition_ms, sweep_ms;
    int64_t candidates_inserted;   /* diagnostics since ctx creation: keys that passed the  */
    int64_t compactions;           /* per-queue filters, and per-queue buffer compactions   */
    int64_t batch_launches;        /* ewsjf_batch_build kernels                             */
    double  batch_ms;
    int64_t sweep_records;         /* records the last sweep's select passes read (after the
                                      Θ-independent prefilter when it ran), 0 if none ran  */
} ewsjf_timing;
ewsjf_status ewsjf_ctx_set_timing(ewsjf_ctx *ctx, int32_t enable);
ewsjf_status ewsjf_ctx_get_timing(ewsjf_ctx *ctx, ewsjf_timing *out);
/* Diagnostics: with EWSJF_PHASES set in the environment the streaming tick
 * records per-CTA phase timestamps (globaltimer ns): row c = out[16c .. 16c+15]
 * = {start, setup done, streaming done (max over warps), all warps done,
 * rows written, collectives, ns in collectives (CTA), first tile done, after
 * the grid barrier, merge done, 0...}.  Copies min(n, num_ctas*16) values.
 * Synchronises.                                                              */
ewsjf_status ewsjf_ctx_get_phases(ewsjf_ctx *ctx, uint64_t *out, int32_t n);

/* Measurement helper (bench.py): the GPU's fp32 FFMA rate, measured with a
 * throughput microbenchmark on the ctx stream (8 independent FMA chains per
 * thread, 8 x 256 threads per SM).  The Θ sweep's roofline peak is this rate
 * divided by its 4 fp32-pipe instructions per (request, Θ) pair.  Synchronises. */
ewsjf_status ewsjf_diag_ffma_rate(ewsjf_ctx *ctx, double *ffma_per_s);
/* Process-wide number of cudaMalloc / cudaMallocHost / cudaFree calls the
 * library has made (contract check: hot calls -- tick, score_select, route,
 * sweep, batch_build -- never change it once the ctx exists). */
int64_t      ewsjf_alloc_count(void);

/* ------------------------------------------------------------- partition --- */
/* Refine-and-Prune parameters (§4.2). alpha > 1 (Eq. 2 significance
 * ratio); min_width >= 1 (Stage-2 width stop, R13); max_queues in
 * 1..EWSJF_MAX_QUEUES (Stage-3 budget); epsilon > 0 (Eq. 3);
 * coarse_k in 1..3 (Stage 1); merge_rule 0 = MIN_U (literal
 * "lowest utility merged", default), 1 = MAX_U (R17).                      */
typedef struct {
    double  alpha;
    int32_t min_width;
    int32_t max_queues;
    double  epsilon;
    int32_t coarse_k;
    int32_t merge_rule;
    int32_t gap_rule;    /* 0: Eq. 2 gaps over the multiset D (R10, default);
                            1: over the set of distinct lengths (SURVEY ambiguity 10 variant) */
    int32_t kmeans_k;    /* 0: Refine-and-Prune (default).  1..EWSJF_MAX_QUEUES: the k-means-only
                            partition of Table 3 "EWSJF (K-Means)": exact 1-D
                            k-means of the history into kmeans_k clusters (DP, reading R32), then
                            the midpoint finalisation (R15); alpha/min_width/max_queues/epsilon/
                            coarse_k/merge_rule/gap_rule are not used.  k > distinct lengths ->
                            one queue per distinct length.  The DP table (4 B x k x distinct) is
                            allocated on first use and kept by the ctx. */
} ewsjf_partition_params;

/* One queue q_i = [min_len, max_len). */
typedef struct {
    int32_t id;          /* stable id (never renumbered; qid values refer to it) */
    int32_t index;       /* 1-based ordinal q_i ascending by length (R3)  */
    int32_t min_len;
    int32_t max_len;
    int64_t count;       /* history members n                                    */
    int64_t sum;         /* S1 = Σ b                                             */
    int64_t sumsq;       /* S2 = Σ b²                                            */
    double  mean;        /* b̄ = S1/n (a bubble: its creating length L, R21)     */
    double  density;     /* ρ = n / (max_len - min_len) (R16)                    */
    double  sse;         /* S2 - S1²/n (informational)                           */
    int32_t is_bubble;
    int32_t empty_count; /* Alg. 1 line 9 counter (maintained by the caller)     */
} ewsjf_queue;

/* Host POD, caller-owned, queues sorted by min_len.  (Named _t because the
 * function ewsjf_partition() takes the plain name.)                        */
typedef struct {
    int32_t     n;
    int32_t     next_id;
    uint64_t    version;
    ewsjf_queue q[EWSJF_MAX_QUEUES];
} ewsjf_partition_t;

typedef struct {
    int64_t n_valid, n_invalid;   /* history entries with len >= 1 / < 1       */
    int64_t distinct;             /* M distinct lengths                         */
    int32_t k_used, t1, t2;       /* Stage-1 k and distinct-index cuts          */
    int64_t segments;             /* m after Stage 2                            */
    int32_t depth;                /* Stage-2 recursion depth                    */
    int64_t merges;               /* Stage-3 merges                             */
    float   ms_hist, ms_kmeans, ms_refine, ms_prune, ms_total;   /* device times */
} ewsjf_partition_stats;

/* Strategic loop, offline mode: Refine-and-Prune over the device array
 * d_len[n] (int32 prompt lengths of the history window D) on the ctx
 * stream: counting sort + segmented prefix statistics (A1-A2), exact k-means
 * k<=3 (Stage 1, A3), Eq. 2 refinement (Stage 2, A4), midpoint finalisation
 * (A5), Eq. 3 pruning (Stage 3, A6).  Writes *out (ids 0..n-1, version
 * incremented from out->version) and optional *stats.  Synchronises.
 * Lengths < 1 are excluded and counted (DOMAIN).  Lengths >= 2^20 (long
 * prompts) are collected into an overflow list, sorted on the device and
 * appended as runs after the histogram's (A1 long tail): up to 32768 of them
 * per call and 2^20 distinct lengths in all, else UNSUPPORTED; every length
 * must stay below 2^31 - 1 (queue bounds are int32).  sumsq wraps modulo
 * 2^64 once sum(c b^2) exceeds 2^63 (no decision reads it).  n > max_history
 * -> INVALID_ARG; no valid length -> EMPTY.                                 */
ewsjf_status ewsjf_partition(ewsjf_ctx *ctx, const int32_t *d_len, int64_t n,
                             const ewsjf_partition_params *params, ewsjf_partition_t *out,
                             ewsjf_partition_stats *stats);

/* Multi-GPU Refine-and-Prune: A1 is a histogram, so a
 * history sharded across ranks partitions exactly by summing the ranks'
 * histograms (integer all-reduce over NCCL) and running A2..A6 from the sum.
 *
 * ewsjf_history_hist: A1 counting sort of d_len[n] into d_hist
 *   (device, caller-owned, EWSJF_HIST_BINS + 1 uint32 entries; bin b = number
 *   of lengths equal to b; bin 0 unused).  h_info[3] (host): lengths < 1,
 *   lengths >= EWSJF_HIST_BINS (UNSUPPORTED when > 0), largest valid length.
 *   Synchronises.
 * ewsjf_partition_from_hist: A2..A6 of ewsjf_partition from a summed
 *   histogram; max_len = largest length with a non-zero bin (all-reduce MAX of
 *   h_info[2]), n_invalid = summed h_info[0] (reported as stats->n_invalid and
 *   DOMAIN, as ewsjf_partition does).  The result is bit-identical to
 *   ewsjf_partition over the concatenated history.  Bins are uint32: at most
 *   2^32 - 1 history lengths per value.  Synchronises.                      */
#define EWSJF_HIST_BINS (1 << 20)
ewsjf_status ewsjf_history_hist(ewsjf_ctx *ctx, const int32_t *d_len, int64_t n, uint32_t *d_hist, int64_t *h_info);
ewsjf_status ewsjf_partition_from_hist(ewsjf_ctx *ctx, const uint32_t *d_hist, int32_t max_len, int64_t n_invalid,
                                       const ewsjf_partition_params *params, ewsjf_partition_t *out,
                                       ewsjf_partition_stats *stats);

/* Online adjust mode ("lightweight adjustments ... statistical
 * heuristics on recent data"; reading R31 in DESIGN.md): each
 * interior boundary B shared by queues [L, B) and [B, U) moves toward the
 * local empirical quantile of the window d_window[n] (device, prompt lengths;
 * < 1 ignored) restricted to [L, U) that keeps the history split
 * q[a].count : q[b].count, by at most floor(max_shift * (B - L)) left /
 * floor(max_shift * (U - B)) right; all boundaries from the original bounds.
 * Updates *part in place (bounds only; version bumped if any moved), *moved
 * (nullable) = boundaries moved.  max_shift in [0, 0.5) (S:191 default 0.25),
 * else INVALID_ARG; window lengths >= 2^20 -> UNSUPPORTED.  Synchronises.   */
ewsjf_status ewsjf_online_adjust(ewsjf_ctx *ctx, const int32_t *d_window, int64_t n, double max_shift,
                                 ewsjf_partition_t *part, int32_t *moved);

/* --------------------------------------------------------------- tactical -- */
/* Scoring part of Θ (§4.4.2): w_x(b̄) = a_x b̄ + b_x. */
typedef struct { double a_b, b_b, a_u, b_u, a_f, b_f; } ewsjf_meta;
/* Per-queue weights, clamped >= 0 (R8). */
typedef struct { float w_base, w_urg, w_fair; } ewsjf_weights;

/* A7 (host, O(n)): out[p] = fp32(max(0, a_x * q[p].mean + b_x)), p = position. */
ewsjf_status ewsjf_weights_from_meta(const ewsjf_meta *theta, const ewsjf_partition_t *part,
                                     ewsjf_weights *out);

/* C_prefill(b) = c0 + c1 b + c2 b² seconds (R4) — used when d_cost is NULL. */
typedef struct { float c0, c1, c2; } ewsjf_cost_params;

typedef enum { EWSJF_SELECT_SCORE = 0, EWSJF_SELECT_FIFO = 1 } ewsjf_select_mode;

/* k: per-queue selection depth (1..ctx max_k).  mode: top-k key, SCORE =
 * (Φ desc, id asc) or FIFO = (arrival asc, id asc) (R1).  now: the clock,
 * seconds in the same epoch as arrival (W_t = now - arrival, R5).           */
typedef struct {
    int32_t           k;
    int32_t           mode;
    float             now;
    ewsjf_cost_params cost;
} ewsjf_select_params;

/* Device summary of one tick / selection. */
typedef struct {
    int32_t n_queues;      /* queues after the call (incl. bubbles created)        */
    int32_t primary;       /* Alg. 1 ArgMax position, -1 if all empty (R24) */
    int64_t n_invalid;     /* len < 1, unknown qid, or refused at the queue cap     */
    int64_t n_excluded;    /* W < 0, C <= 0 or NaN                                  */
    int64_t n_gap;         /* gap-falling requests handled by Alg. 2                */
    int64_t n_bubbles;     /* bubble queues created (App. D)                        */
    int64_t n_dropped;     /* gap requests refused at EWSJF_MAX_QUEUES              */
    int32_t status;        /* ewsjf_status of the device-side work                  */
    int32_t pad;
} ewsjf_summary;

/* Outputs of a selection (all caller-owned device buffers unless h_).
 * d_topk_id / d_topk_score: [EWSJF_MAX_QUEUES * k], row p = queue position p,
 *   best first, id -1 / score 0 padding.  Φ per Eq. 4 in fp32.
 * d_count [MAXQ]: scored members per queue.  d_head_id / d_head_score [MAXQ]:
 *   the queue head (oldest by (arrival, id), R26) and its Φ — Alg. 1's
 *   per-queue score.  d_max_score [MAXQ]: max Φ in the queue.
 * d_summary [1] (nullable -> ctx scratch): see ewsjf_summary.
 * h_summary (optional): if non-NULL the call synchronises, copies the summary
 *   and (ewsjf_tick / ewsjf_tick_merge) writes bubbles created into *part.   */
typedef struct {
    int64_t           *d_topk_id;
    float             *d_topk_score;
    int64_t           *d_count;
    int64_t           *d_head_id;
    float             *d_head_score;
    float             *d_max_score;
    ewsjf_summary     *d_summary;
    ewsjf_summary     *h_summary;
} ewsjf_select_out;

/* A8+A9 Dispatcher (App. D Alg. 2): d_qid[r] = stable id of
 * the queue whose [min_len, max_len) contains d_len[r]; gap-falling lengths
 * go through Alg. 2 in pool-index order (R22) creating bubble queues of width
 * bubble_width (>= 1) inserted into *part (in/out; ids from part->next_id,
 * indices renumbered).  d_qid[r] = -1 for len < 1 or a request refused
 * at the cap.  Synchronises (the host partition is updated).                */
ewsjf_status ewsjf_route(ewsjf_ctx *ctx, const int32_t *d_len, int64_t n, ewsjf_partition_t *part,
                         int32_t bubble_width, int32_t *d_qid, ewsjf_summary *h_summary);

/* A10+A11 over an already-routed pool: Eq. 4 score of every request
 * Φ = q_i/(b+1) (w_base + w_urg W/C + w_fair ln(b+1)) (R2-R5) with
 * per-queue weights w[position] (d_cost NULL -> C from params->cost), then per
 * queue count, FIFO head, top-k, max score and the ArgMax queue (Alg. 1).
 * d_qid holds stable ids of *part (unknown / -1 -> excluded, counted). Async
 * unless out->h_summary.                                                     */
ewsjf_status ewsjf_score_select(ewsjf_ctx *ctx, const int32_t *d_len, const float *d_arrival,
                                const float *d_cost, const int32_t *d_qid, int64_t n,
                                const ewsjf_partition_t *part, const ewsjf_weights *w,
                                const ewsjf_select_params *params, ewsjf_select_out *out);

/* The fused tick: route (A8) + bubbles (A9) + weights from Θ (A7) + score (A10)
 * + select (A11) over the whole pending pool d_len/d_arrival/d_cost[n] (d_cost
 * may be NULL).  Request ids are global_base + r.  d_qid_out (nullable) gets
 * the stable queue ids.  Bubbles created by this tick (App. D) are written
 * back into *part when out->h_summary is non-NULL (synchronous call); an
 * asynchronous call leaves *part unchanged.                                  */
ewsjf_status ewsjf_tick(ewsjf_ctx *ctx, const int32_t *d_len, const float *d_arrival, const float *d_cost,
                        int64_t n, int64_t global_base, ewsjf_partition_t *part, int32_t bubble_width,
                        const ewsjf_meta *theta, const ewsjf_select_params *params,
                        int32_t *d_qid_out, ewsjf_select_out *out);

/* Host-buffer variant of ewsjf_tick for end-to-end use: copies h_len /
 * h_arrival / h_cost[n] (pinned host memory recommended) into ctx scratch,
 * runs the tick, copies qid into h_qid_out[n] (nullable) and the per-queue
 * results into the h_ arrays (same layouts as ewsjf_select_out, host side;
 * each nullable) and the summary into *h_summary (required).  Synchronises. */
ewsjf_status ewsjf_tick_host(ewsjf_ctx *ctx, const int32_t *h_len, const float *h_arrival, const float *h_cost,
                             int64_t n, int64_t global_base, ewsjf_partition_t *part, int32_t bubble_width,
                             const ewsjf_meta *theta, const ewsjf_select_params *params,
                             int32_t *h_qid_out, int64_t *h_topk_id, float *h_topk_score, int64_t *h_count,
                             int64_t *h_head_id, float *h_head_score, float *h_max_score,
                             ewsjf_summary *h_summary);

/* ------------------------------------------------- multi-GPU --- */
/* Rank-local half of a sharded tick.  The pool is sharded by index: this rank
 * owns global ids [global_base, global_base + n).  Routes, scores and reduces
 * its shard to a fixed-size exchange record written to d_exchange
 * (ewsjf_exchange_bytes(ctx, part->n, k) bytes, 256-byte aligned): per-queue
 * top-k keys with their scores, member counts, head candidates and the
 * shard's gap requests (capacity-bounded).  The caller all-gathers the
 * records of all ranks (NCCL over NVLink) and calls ewsjf_tick_merge.       */
int64_t      ewsjf_exchange_bytes(const ewsjf_ctx *ctx, int32_t n_queues, int32_t k);
/* Capacity of the gap-request section of this ctx's exchange records (App. D:
 * the requests of a shard whose length falls between queues, P:322-325 and
 * P:788-808).  Each record carries the shard's gap count plus up to gap_cap
 * entries (default 1024); ewsjf_exchange_bytes grows by 16 bytes per entry.
 * Size it for the expected novel lengths per shard (a shard of n requests
 * needs at most n).  A merge whose shards held more gap requests than the
 * capacity returns CAPACITY (the overflowing requests keep qid -2).
 * Strategic call: synchronises the ctx stream and, with a communicator
 * attached, reallocates the exchange buffers.  INVALID_ARG outside [1, 2^26]. */
ewsjf_status ewsjf_ctx_set_exchange_gap_cap(ewsjf_ctx *ctx, int32_t gap_cap);
ewsjf_status ewsjf_tick_local(ewsjf_ctx *ctx, const int32_t *d_len, const float *d_arrival, const float *d_cost,
                              int64_t n, int64_t global_base, const ewsjf_partition_t *part,
                              const ewsjf_meta *theta, const ewsjf_select_params *params,
                              int32_t *d_qid_out, void *d_exchange);
/* Global half: merges `world` exchange records (contiguous, rank order) into
 * the replicated global result (identical on every rank), running Alg. 2 over
 * the union of gap requests in global index order (R22) and writing this
 * rank's gap requests' qids into d_qid_local[0..n_local) (global ids
 * [global_base, global_base + n_local)).                                     */
ewsjf_status ewsjf_tick_merge(ewsjf_ctx *ctx, const void *d_exchange_all, int32_t world,
                              int64_t global_base, int64_t n_local, int32_t *d_qid_local,
                              ewsjf_partition_t *part, int32_t bubble_width, const ewsjf_meta *theta,
                              const ewsjf_select_params *params, ewsjf_select_out *out);

/* ----------------------------------------------- Θ sweep (A12, config C5) --- */
/* For each of n_theta meta-parameter vectors (§4.4.2):
 * A7 -> A10 -> A11 over one routed snapshot (d_qid: stable ids of *part).
 * outs[t] receives the selection for thetas[t] (device buffers as in
 * ewsjf_select_out; h_summary ignored; each outs[t].d_summary, when non-NULL,
 * gets that Θ's summary).  Every outs[t] equals what ewsjf_score_select returns
 * with ewsjf_weights_from_meta(&thetas[t], part).  SCORE mode only (the sweep
 * ranks scoring policies; FIFO keys do not depend on Θ): params->mode must be
 * EWSJF_SELECT_SCORE.  Async; returns DOMAIN if any Θ excluded elements,
 * INVALID_ARG on bad arguments (nothing launched).                          */
/* Reserve the sweep's scratch (records + candidate rows) for snapshots of up
 * to max_n requests; a strategic (setup) call that allocates and synchronises.
 * ewsjf_score_select_sweep itself never allocates: it returns CAPACITY for a
 * snapshot larger than the reservation (none made -> CAPACITY). */
ewsjf_status ewsjf_ctx_reserve_sweep(ewsjf_ctx *ctx, int64_t max_n);
ewsjf_status ewsjf_score_select_sweep(ewsjf_ctx *ctx, const int32_t *d_len, const float *d_arrival,
                                      const float *d_cost, const int32_t *d_qid, int64_t n,
                                      const ewsjf_partition_t *part, const ewsjf_meta *thetas,
                                      int32_t n_theta, const ewsjf_select_params *params,
                                      ewsjf_select_out *outs);

/* ------------------------------------ Alg. 1 batch builder --- */
/* Budget of one forward pass (BatchBudget). */
typedef struct {
    int32_t max_requests;  /* >= 1                                         */
    int32_t pad;
    int64_t max_tokens;    /* Σ prompt lengths, 0 <= max_tokens < 2^32 - 1  */
} ewsjf_batch_budget;

/* Alg. 1 lines 13-21: GreedyFill from the primary queue
 * (sel->d_summary->primary, the ArgMax of the per-queue head scores) in FIFO
 * order, stopping at the first request that does not fit (R28; the batch's
 * first request is always admitted), then Backfill from the queues at
 * index distance 1, 2, …, lower neighbour first, each FIFO under the same rule
 * (R29), until max_requests or the queues run out.
 * sel: the device outputs of a FIFO-mode selection (ewsjf_tick / ewsjf_score_select
 *   with params.mode = EWSJF_SELECT_FIFO) with depth k >= max_requests (so every
 *   queue's pullable FIFO prefix is in its row) over n_queues queue positions;
 *   d_summary NULL -> the ctx summary the last selection wrote.
 * d_len[n]: prompt lengths; the row ids are global_base + index into d_len.
 * d_batch_id [max_requests] (device, caller-owned): batch request ids in
 *   admission order, -1 padding.  d_batch_info [4] (device int64): batch size,
 *   tokens, status (EWSJF_OK, or INVALID_ARG if a row id fell outside d_len),
 *   primary position.  Async, one kernel on the ctx stream.  INVALID_ARG
 *   (nothing launched) on null pointers, k < max_requests, max_tokens range. */
ewsjf_status ewsjf_batch_build(ewsjf_ctx *ctx, const int32_t *d_len, int64_t n, int64_t global_base,
                               const ewsjf_select_out *sel, int32_t k, int32_t n_queues,
                               const ewsjf_batch_budget *budget, int64_t *d_batch_id, int64_t *d_batch_info);

/* Alg. 1 lines 8-12: for every queue position p with h_count[p] == 0
 * increment part->q[p].empty_count, else reset it to 0 (consecutive empty
 * tactical steps; R30); remove the queues whose
 * counter exceeds `threshold` (strict, R25), renumber the survivors' index
 * 1..n and bump part->version if any was removed.  Host-only (the
 * partition is host state); *removed (nullable) = queues removed.  h_count is
 * the d_count of the tick, copied to the host.                               */
ewsjf_status ewsjf_prune_empty(ewsjf_partition_t *part, const int64_t *h_count, int32_t threshold,
                               int32_t *removed);

#ifdef __cplusplus
}
#endif
#endif /* EWSJF_H */
