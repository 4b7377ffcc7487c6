/*
 * ewsjf_oracle.h — the CPU ORACLE for libewsjf.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct C99 in fp64 of what the EWSJF scheduling tick
 * and Refine-and-Prune compute (arXiv 2601.21758, PAPER.md; SPEC.md for the
 * interface shape).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA product under
 * paper_2601_21758_b200/ and include/ (and neither includes the other).
 *
 * Citation format: P:n = PAPER.md line n, S:n = SPEC.md line n.  Readings of
 * silent / ambiguous passages are numbered R1..R27 as in DESIGN.md §3.
 *
 * Steps:
 *   O1 sort + run-length encode the history          (§4.2 Formalism)
 *   O2 int64 prefix sums N, S1, S2                    (P:285 mean(G), P:295 b̄)
 *   O3 exact 1-D k-means, k = coarse_k <= 3          (§4.2 Stage 1; R9)
 *   O4 recursive gap refinement, Eq. 2               (§4.2 Stage 2; R10-R14)
 *   O5 midpoint finalization                         (R15)
 *   O6 utility pruning, Eq. 3                        (§4.2 Stage 3; R16-R18)
 *   O7 context-aware weights w = max(0, a*b̄ + b)    (§4.4.1; R8)
 *   O8 routing + on-demand bubble queues, Alg. 2     (App. D; R19-R23)
 *   O9 Eq. 1 / Eq. 4 score                            (R2-R5)
 *   O10 per-queue count, FIFO head, top-K, argmax     (Alg. 1; R1, R24, R26)
 *   O11 Θ sweep: O7 -> O9 -> O10 per Θ                (§4.4.2)
 *   O12 Alg. 1 Batch Builder + empty-queue pruning    (R28-R30)
 *
 * Parity unpinned (no paper-printed value exists):
 *   the C_prefill quadratic and its defaults (SPEC invention), the
 *   post-merge profile, the bubble b̄ = L (R21), SCORE-mode top-K
 *   (north_star generalisation of Alg. 1's head-only score).
 */
#ifndef EWSJF_ORACLE_H
#define EWSJF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAXQ 256              /* hard cap on queues incl. bubbles */

enum { OR_OK = 0, OR_INVALID = 1, OR_DOMAIN = 2, OR_EMPTY = 3, OR_CAPACITY = 4 };
enum { OR_MIN_U = 0, OR_MAX_U = 1 };          /* R17 merge rule */
enum { OR_SCORE = 0, OR_FIFO = 1 };           /* R1 selection key */

typedef struct {
    int32_t id;            /* stable id                                  */
    int32_t index;         /* 1-based ordinal q_i, ascending by length   */
    int32_t min_len;       /* [min_len, max_len)                         */
    int32_t max_len;
    int64_t count;         /* history members (0 for a bubble)           */
    int64_t sum;           /* S1 = Σ b over members                      */
    int64_t sumsq;         /* S2 = Σ b² over members                     */
    double  mean;          /* b̄ (bubble: its creating L, R21)           */
    double  density;       /* ρ = count / (max_len - min_len)  (R16)     */
    double  sse;           /* S2 - S1²/n, informational                  */
    int32_t is_bubble;
    int32_t pad;
} or_queue;

typedef struct {
    int32_t n;             /* queues, sorted by min_len */
    int32_t next_id;
    or_queue q[OR_MAXQ];
} or_partition;

typedef struct {
    double  alpha;         /* Eq. 2 significance ratio, > 1      */
    int32_t min_width;     /* Stage-2 width stop, >= 1           */
    int32_t max_queues;    /* Stage-3 budget, 1..256             */
    double  epsilon;       /* Eq. 3 ε > 0                        */
    int32_t coarse_k;      /* Stage-1 k, 1..3                    */
    int32_t merge_rule;    /* OR_MIN_U (literal) or OR_MAX_U     */
    int32_t gap_rule;      /* 0: gaps over the multiset D (R10); 1: over the set of distinct lengths */
} or_params;

typedef struct {
    int64_t n_valid;       /* history entries with len >= 1 */
    int64_t n_invalid;     /* len < 1, excluded              */
    int64_t distinct;      /* M                              */
    int32_t k_used;        /* min(coarse_k, M)               */
    int32_t t1, t2;        /* Stage-1 distinct-index cuts    */
    int64_t segments;      /* m after Stage 2                */
    int32_t depth;         /* Stage-2 recursion depth        */
    int64_t merges;        /* Stage-3 merges performed       */
} or_partition_stats;

typedef struct { double a_b, b_b, a_u, b_u, a_f, b_f; } or_meta;

typedef struct {
    int32_t k;             /* per-queue selection depth        */
    int32_t mode;          /* OR_SCORE / OR_FIFO               */
    float   now;           /* seconds, same epoch as arrival   */
    float   c0, c1, c2;    /* C_prefill(b) = c0 + c1 b + c2 b² */
} or_select_params;

/* Per-queue outputs are indexed by queue POSITION (index - 1) of the partition
 * the call ends with.  topk_* are [n_queues * k], best first, id -1 padding. */
typedef struct {
    int64_t *topk_id;
    double  *topk_score;
    int64_t *count;
    int64_t *head_id;
    double  *head_score;
    double  *max_score;
    int32_t  primary;      /* position of argmax head_score, -1 if all empty */
    int64_t  n_excluded;   /* W < 0 or C <= 0 (or NaN)       */
    int64_t  n_invalid;    /* len < 1                        */
    int64_t  n_bubbles;    /* bubble queues created          */
    int64_t  n_dropped;    /* gap requests refused at the 256-queue cap */
} or_select_out;

/* O1+O2: sort + RLE (v ascending, c counts) and prefix sums.  Returns M.
 * v, c must hold n entries; N, S1, S2 must hold n+1. */
int64_t or_rle(const int32_t *len, int64_t n, int32_t *v, int64_t *c, int64_t *n_invalid);
void    or_prefix(const int32_t *v, const int64_t *c, int64_t M, int64_t *N, int64_t *S1, int64_t *S2);

/* O3: exact 1-D k-means over the RLE, k <= 3. Writes cuts (k-1 of them). */
int     or_kmeans(const int64_t *N, const int64_t *S1, int64_t M, int32_t k, int32_t *cuts);

/* O4 on one distinct-index range [x, y): appends final ranges' starts to
 * seg_lo (ascending), returns number appended; *depth = max depth seen. */
/* O14: exact 1-D k-means for any k by DP (R32; Table 3 "EWSJF (K-Means)"). */
int     or_kmeans_dp(const int64_t *N, const int64_t *S1, int64_t M, int32_t k, int32_t *cuts);
int     or_partition_kmeans(const int32_t *len, int64_t n, int32_t k, or_partition *out, or_partition_stats *st);
int64_t or_refine(const int32_t *v, const int64_t *N, int64_t x, int64_t y, double alpha,
                  int32_t min_width, int64_t *seg_start, int32_t *depth);

/* Eq. 3 for one adjacent pair (exposed for the SPEC worked examples). */
double  or_utility(double rho_l, double rho_r, double mean_l, double mean_r, double eps);

/* O1..O6 end to end. */
int     or_partition_run(const int32_t *len, int64_t n, const or_params *p,
                         or_partition *out, or_partition_stats *st);

/* O6 alone on caller-given candidate queues (used by the SPEC pins). lo/hi are
 * interval bounds, cnt/s1/s2 member statistics; merges in place; returns m'. */
int64_t or_prune(int64_t m, int32_t *lo, int32_t *hi, int64_t *cnt, int64_t *s1, int64_t *s2,
                 int32_t max_queues, double eps, int32_t rule, int64_t *merges);

/* O7 */
void    or_weights(const or_meta *th, double mean, float w[3]);

/* O8: route in index order, creating bubbles (mutates part). qid = stable id,
 * -1 for len < 1 or a gap request refused at the cap. */
int     or_route(const int32_t *len, int64_t n, or_partition *part, int32_t bubble_width,
                 int32_t *qid, int64_t *n_invalid, int64_t *n_bubbles, int64_t *n_dropped);

/* O9 for one request (fp64 from the fp32 inputs). Returns 0 and sets *phi if
 * included; returns 1 if excluded (W < 0, C <= 0, or NaN). */
int     or_score_one(int32_t b, float arrival, const float *cost_or_null, int32_t index,
                     const float w[3], const or_select_params *sp, double *phi);

/* O9+O10 over a routed pool. w = [3 * part->n] by position. */
int     or_score_select(const int32_t *len, const float *arrival, const float *cost,
                        const int32_t *qid, int64_t n, int64_t global_base,
                        const or_partition *part, const float *w,
                        const or_select_params *sp, or_select_out *out);

/* O9 over a routed pool: phi[r] (fp64) and valid[r] (1 = scored). */
void    or_score_all(const int32_t *len, const float *arrival, const float *cost, const int32_t *qid, int64_t n,
                     const or_partition *part, const float *w, const or_select_params *sp,
                     double *phi, int8_t *valid);

/* O8 + O7 + O9 + O10: one tick (part is in/out: bubbles). */
int     or_tick(const int32_t *len, const float *arrival, const float *cost, int64_t n,
                int64_t global_base, or_partition *part, int32_t bubble_width,
                const or_meta *theta, const or_select_params *sp,
                int32_t *qid_out, or_select_out *out);

/* O11 (A12): the Θ-batched evaluation of the meta-optimizer's scoring inner
 * loop (§4.4.2): O7 -> O9 -> O10 for each thetas[t] over
 * one routed snapshot; outs[t] receives Θ t.  Returns the first non-OK
 * status of the per-Θ calls (DOMAIN if any request was excluded/invalid). */
int     or_sweep(const int32_t *len, const float *arrival, const float *cost, const int32_t *qid,
                 int64_t n, int64_t global_base, const or_partition *part,
                 const or_meta *thetas, int32_t n_theta, const or_select_params *sp,
                 or_select_out *outs);

/* O12: Alg. 1 lines 14-21, the Batch Builder (P:163,
 * P:178-193) over a routed pool.  Members of a queue are
 * the requests O9 scores (valid qid, len >= 1, W >= 0, C > 0), FIFO by
 * (arrival, id).  GreedyFill: from queue `primary` (position, the O10 ArgMax)
 * pull members in FIFO order while the budget admits them (count <
 * max_requests and tokens + len <= max_tokens; the batch's first request is
 * always admitted), stopping at the first one that does not fit
 * (R28).  Backfill (if the batch is not full): queues at position distance
 * 1, 2, ... from the primary, lower neighbour first (R29), each pulled
 * FIFO while the budget admits.  Writes batch ids (global) in pull order.
 * Returns the batch size. */
typedef struct { int32_t max_requests; int64_t max_tokens; } or_budget;
int64_t or_batch(const int32_t *len, const float *arrival, const float *cost, const int32_t *qid,
                 int64_t n, int64_t global_base, const or_partition *part, const or_select_params *sp,
                 int32_t primary, const or_budget *budget, int64_t *batch_ids, int64_t *batch_tokens);

/* Alg. 1 lines 8-12: every queue with count[p] == 0 increments its empty
 * counter (reset to 0 when the queue has members: consecutive empty steps, R30); a queue whose counter exceeds `threshold` (strict,
 * R25) is removed and the remaining indices renumbered.  empty_cnt[p] is
 * in/out by position (compacted like the queues).  Returns queues removed. */
int32_t or_prune_empty(or_partition *part, int32_t *empty_cnt, const int64_t *count, int32_t threshold);

/* O13 — online adjust mode ("lightweight adjustments ... statistical
 * heuristics on recent data", reading R31).  For every interior
 * boundary B shared by adjacent queues a = [L, B) and b = [B, U) (only where
 * a.max_len == b.min_len): with c_a, c_b the queues' history counts and the
 * window's m members in [L, U) sorted v_0 <= ... <= v_{m-1}, the local
 * empirical quantile is the smallest x with #(v < x) * (c_a + c_b) >= m * c_a,
 * i.e. T = L if k = ceil(m c_a / (c_a + c_b)) is 0, else v_{k-1} + 1.  B moves
 * toward T by at most floor(max_shift * (B - L)) leftwards and
 * floor(max_shift * (U - B)) rightwards (fp64 products), all boundaries from
 * the original bounds at once; m = 0 or c_a + c_b = 0 -> no move.  Lengths
 * < 1 in the window are ignored.  max_shift in [0, 0.5) keeps every queue's
 * width >= 1.  Profiles (counts, sums) are not re-binned.  Returns the number
 * of boundaries moved. */
int32_t or_online_adjust(const int32_t *window, int64_t n, double max_shift, or_partition *part);

#ifdef __cplusplus
}
#endif
#endif
