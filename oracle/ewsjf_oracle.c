/*
 * ewsjf_oracle.c — CPU ORACLE (test infrastructure only; see ewsjf_oracle.h).
 *
 * Plain scalar C99, fp64, built with -O2 -ffp-contract=off so that every
 * expression below is evaluated exactly as written (no FMA contraction).
 * Each function cites the PAPER.md / SPEC.md passage it follows.  Nothing here
 * is blocked, fused or reordered beyond the definition it transcribes.
 */
#include "ewsjf_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* O1  sort + run-length encode.  §4.2 Formalism: "D = {b_1..b_N}, b_1 <= ... <=
 * b_N, the sorted set of prompt lengths".  Entries < 1 violate the
 * Request invariant prompt_len >= 1 and are excluded and counted.    */
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

int64_t or_rle(const int32_t *len, int64_t n, int32_t *v, int64_t *c, int64_t *n_invalid) {
    int32_t *d = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int64_t nv = 0, bad = 0;
    for (int64_t i = 0; i < n; i++) {
        if (len[i] >= 1) d[nv++] = len[i];
        else bad++;
    }
    qsort(d, (size_t)nv, sizeof(int32_t), cmp_i32);
    int64_t M = 0;
    for (int64_t i = 0; i < nv; i++) {
        if (M > 0 && v[M - 1] == d[i]) c[M - 1]++;
        else { v[M] = d[i]; c[M] = 1; M++; }
    }
    free(d);
    if (n_invalid) *n_invalid = bad;
    return M;
}

/* O2  prefix sums over the RLE, exact in int64: N[i] = Σ_{j<i} c_j,
 * S1[i] = Σ c_j v_j, S2[i] = Σ c_j v_j².  (mean(G) P:285, b̄ P:295, SSE S:128) */
void or_prefix(const int32_t *v, const int64_t *c, int64_t M, int64_t *N, int64_t *S1, int64_t *S2) {
    N[0] = 0; S1[0] = 0; S2[0] = 0;
    for (int64_t j = 0; j < M; j++) {
        N[j + 1]  = N[j]  + c[j];
        S1[j + 1] = S1[j] + c[j] * (int64_t)v[j];
        S2[j + 1] = S2[j] + c[j] * (int64_t)v[j] * (int64_t)v[j];
    }
}

/* ------------------------------------------------------------------------- */
/* O3  Stage 1 "applying k-means with k=3".  Reading R9: the exact
 * 1-D optimum.  Minimising the within-cluster SSE of contiguous
 * clusters equals maximising Σ_c S1_c²/n_c; the optimum only cuts between
 * distinct values.  The canonical fp64 objective for cuts 0 < i < j < M is
 *   F(i,j) = ((S1[i]²/N[i]) + ((S1[j]-S1[i])²/(N[j]-N[i]))) + ((S1[M]-S1[j])²/(N[M]-N[j]))
 * each difference exact in int64 then converted, each x*x and /n rounded once;
 * argmax, ties -> lexicographically smallest (i, j).                        */
static double sq_over(int64_t s, int64_t n) {
    double d = (double)s;
    double sq = d * d;
    return sq / (double)n;
}

int or_kmeans(const int64_t *N, const int64_t *S1, int64_t M, int32_t k, int32_t *cuts) {
    if (k < 1 || k > 3 || k > M) return OR_INVALID;
    if (k == 1) return OR_OK;
    if (k == 2) {
        double best = -1.0; int64_t bi = -1;
        for (int64_t i = 1; i <= M - 1; i++) {
            double F = sq_over(S1[i], N[i]) + sq_over(S1[M] - S1[i], N[M] - N[i]);
            if (bi < 0 || F > best) { best = F; bi = i; }
        }
        cuts[0] = (int32_t)bi;
        return OR_OK;
    }
    double best = -1.0; int64_t bi = -1, bj = -1;
    for (int64_t i = 1; i <= M - 2; i++) {
        for (int64_t j = i + 1; j <= M - 1; j++) {
            double F = (sq_over(S1[i], N[i]) + sq_over(S1[j] - S1[i], N[j] - N[i]))
                       + sq_over(S1[M] - S1[j], N[M] - N[j]);
            if (bi < 0 || F > best) { best = F; bi = i; bj = j; }
        }
    }
    cuts[0] = (int32_t)bi; cuts[1] = (int32_t)bj;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O14 (next) exact 1-D k-means for any k: Table 3's
 * "EWSJF (K-Means)" variant partitions the history by k-means alone with
 * k = 5/10/30.  Same objective as O3 (R9: maximise
 * Σ_c S1_c²/n_c over contiguous clusters of distinct values), evaluated by
 * dynamic programming in O3's left-to-right summation order:
 *   D_1[j] = S1[j]²/N[j],   D_l[j] = max_{l-1 <= i < j} D_{l-1}[i] + (S1[j]-S1[i])²/(N[j]-N[i]),
 * then backtracking from j = M, at every level the SMALLEST i attaining the
 * maximum (reading R32).  k > M -> k = M (as S:165).  cuts[0..k-2] ascending.
 * O(k M²), plain.  For k <= 3 the value equals O3's optimum; only exact ties
 * may pick other cuts (O3 breaks them lexicographically, R9).              */
int or_kmeans_dp(const int64_t *N, const int64_t *S1, int64_t M, int32_t k, int32_t *cuts) {
    if (k < 1 || M < 1) return OR_INVALID;
    if (k > M) k = (int32_t)M;
    if (k == 1) return OR_OK;
    double *D = (double *)malloc(sizeof(double) * (size_t)k * (size_t)(M + 1));
    int64_t *A = (int64_t *)malloc(sizeof(int64_t) * (size_t)k * (size_t)(M + 1));
    for (int64_t j = 1; j <= M; j++) { D[j] = sq_over(S1[j], N[j]); A[j] = 0; }
    for (int32_t l = 2; l <= k; l++) {
        double *Dp = D + (size_t)(l - 2) * (M + 1), *Dl = D + (size_t)(l - 1) * (M + 1);
        int64_t *Al = A + (size_t)(l - 1) * (M + 1);
        for (int64_t j = l; j <= M; j++) {
            double best = 0.0; int64_t bi = -1;
            for (int64_t i = l - 1; i < j; i++) {
                double F = Dp[i] + sq_over(S1[j] - S1[i], N[j] - N[i]);
                if (bi < 0 || F > best) { best = F; bi = i; }
            }
            Dl[j] = best; Al[j] = bi;
        }
    }
    int64_t j = M;
    for (int32_t l = k; l >= 2; l--) {
        j = A[(size_t)(l - 1) * (M + 1) + j];
        cuts[l - 2] = (int32_t)j;
    }
    free(D); free(A);
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O4  Stage 2 recursive refinement, Eq. 2 "Gap_j > α · mean(G)".
 * G = consecutive gaps of the sorted MULTISET inside the cluster (R10), so
 * mean(G) = span/(n-1) (telescoping).  Split at EVERY qualifying gap (R11),
 * mean recomputed per sub-cluster (R12).  Stop when no gap qualifies or
 * the width span < min_width (R13).  Strict '>' evaluated as
 * (double)g*(double)(n-1) > alpha*(double)span (R14).                        */
static int64_t refine_rec(const int32_t *v, const int64_t *N, int64_t x, int64_t y, double alpha,
                          int32_t min_width, int64_t *out, int32_t level, int32_t *depth) {
    if (level > *depth) *depth = level;
    int64_t n = N[y] - N[x];
    int64_t span = (int64_t)v[y - 1] - (int64_t)v[x];
    if (n < 2 || span == 0 || span < (int64_t)min_width) { out[0] = x; return 1; }
    int64_t produced = 0, start = x;
    int any = 0;
    for (int64_t j = x; j < y - 1; j++) {
        int64_t g = (int64_t)v[j + 1] - (int64_t)v[j];
        if ((double)g * (double)(n - 1) > alpha * (double)span) {
            any = 1;
            produced += refine_rec(v, N, start, j + 1, alpha, min_width, out + produced, level + 1, depth);
            start = j + 1;
        }
    }
    if (!any) { out[0] = x; return 1; }
    produced += refine_rec(v, N, start, y, alpha, min_width, out + produced, level + 1, depth);
    return produced;
}

int64_t or_refine(const int32_t *v, const int64_t *N, int64_t x, int64_t y, double alpha,
                  int32_t min_width, int64_t *seg_start, int32_t *depth) {
    int32_t d = 0;
    int64_t r = refine_rec(v, N, x, y, alpha, min_width, seg_start, 1, &d);
    if (depth && d > *depth) *depth = d;
    return r;
}

/* ------------------------------------------------------------------------- */
/* O6  Stage 3, Eq. 3: U(q_i,q_{i+1}) = (ρ(q_i)+ρ(q_{i+1})) / (|b̄_{i+1} - b̄_i| + ε)
 * (P:291-296).  "Queues with the lowest utility are merged until the system
 * satisfies the configured max_queues budget".  R16: ρ = n/width; the
 * merged profile is recomputed from summed (n, S1, S2) over [lo_p, hi_q).
 * R17: MIN_U literal (default), MAX_U as a switch.  Ties -> lowest pair.
 * All U are recomputed from scratch every iteration (plain, O(m²)).        */
double or_utility(double rho_l, double rho_r, double mean_l, double mean_r, double eps) {
    return (rho_l + rho_r) / (fabs(mean_r - mean_l) + eps);
}

static double rho_of(int64_t cnt, int32_t lo, int32_t hi) {
    return (double)cnt / (double)((int64_t)hi - (int64_t)lo);
}
static double mean_of(int64_t s1, int64_t cnt) {
    return cnt > 0 ? (double)s1 / (double)cnt : 0.0;
}

int64_t or_prune(int64_t m, int32_t *lo, int32_t *hi, int64_t *cnt, int64_t *s1, int64_t *s2,
                 int32_t max_queues, double eps, int32_t rule, int64_t *merges) {
    int64_t nm = 0;
    double *rho = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *mu  = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    while (m > (int64_t)max_queues && m > 1) {
        for (int64_t p = 0; p < m; p++) {
            rho[p] = rho_of(cnt[p], lo[p], hi[p]);
            mu[p]  = mean_of(s1[p], cnt[p]);
        }
        int64_t bp = -1; double bu = 0.0;
        for (int64_t p = 0; p + 1 < m; p++) {
            double U = or_utility(rho[p], rho[p + 1], mu[p], mu[p + 1], eps);
            int better = (rule == OR_MAX_U) ? (U > bu) : (U < bu);
            if (bp < 0 || better) { bu = U; bp = p; }
        }
        /* merge bp and bp+1 */
        hi[bp] = hi[bp + 1];
        cnt[bp] += cnt[bp + 1]; s1[bp] += s1[bp + 1]; s2[bp] += s2[bp + 1];
        for (int64_t p = bp + 1; p + 1 < m; p++) {
            lo[p] = lo[p + 1]; hi[p] = hi[p + 1];
            cnt[p] = cnt[p + 1]; s1[p] = s1[p + 1]; s2[p] = s2[p + 1];
        }
        m--; nm++;
    }
    free(rho); free(mu);
    if (merges) *merges = nm;
    return m;
}

/* ------------------------------------------------------------------------- */
/* O1..O6  Refine-and-Prune pipeline.          */
int or_partition_run(const int32_t *len, int64_t n, const or_params *p,
                     or_partition *out, or_partition_stats *st) {
    or_partition_stats S;
    memset(&S, 0, sizeof S);
    memset(out, 0, sizeof *out);
    if (!(p->alpha > 1.0) || p->min_width < 1 || p->max_queues < 1 || p->max_queues > OR_MAXQ ||
        !(p->epsilon > 0.0) || p->coarse_k < 1 || p->coarse_k > 3 ||
        (p->merge_rule != OR_MIN_U && p->merge_rule != OR_MAX_U) || (p->gap_rule != 0 && p->gap_rule != 1) || n < 0)
        return OR_INVALID;
    size_t nn = (size_t)(n > 0 ? n : 1);
    int32_t *v = (int32_t *)malloc(sizeof(int32_t) * nn);
    int64_t *c = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t M = or_rle(len, n, v, c, &S.n_invalid);
    S.n_valid = n - S.n_invalid;
    S.distinct = M;
    if (M == 0) { free(v); free(c); if (st) *st = S; return OR_EMPTY; }
    int64_t *N  = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M + 1));
    int64_t *S1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M + 1));
    int64_t *S2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M + 1));
    or_prefix(v, c, M, N, S1, S2);

    /* Stage 1 (fewer distinct values than coarse_k -> k = distinct count) */
    int32_t k = p->coarse_k < M ? p->coarse_k : (int32_t)M;
    int32_t cuts[2] = {0, 0};
    or_kmeans(N, S1, M, k, cuts);
    S.k_used = k;
    S.t1 = k >= 2 ? cuts[0] : 0;
    S.t2 = k >= 3 ? cuts[1] : 0;
    int64_t bounds[4]; int nb = 0;
    bounds[nb++] = 0;
    for (int i = 0; i < k - 1; i++) bounds[nb++] = cuts[i];
    bounds[nb++] = M;

    /* Stage 2 */
    int64_t *seg = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M + 1));
    int64_t m = 0;
    int32_t depth = 0;
    /* gap_rule 1 (set reading of G): Eq. 2 counts distinct lengths, i.e. the
     * prefix of a multiplicity-1 multiset: Nset[i] = i */
    int64_t *Nset = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M + 1));
    for (int64_t i = 0; i <= M; i++) Nset[i] = i;
    for (int i = 0; i + 1 < nb; i++)
        m += or_refine(v, p->gap_rule ? Nset : N, bounds[i], bounds[i + 1], p->alpha, p->min_width, seg + m, &depth);
    free(Nset);
    seg[m] = M;
    S.segments = m;
    S.depth = depth;

    /* O5  finalization: B_0 = lo_1, B_i = floor((hi_i + lo_{i+1})/2) + 1 (R15),
     * B_m = hi_m + 1; queue i = [B_{i-1}, B_i).    */
    int32_t *qlo = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    int32_t *qhi = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    int64_t *qc  = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
    int64_t *qs1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
    int64_t *qs2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
    for (int64_t i = 0; i < m; i++) {
        int64_t x = seg[i], y = seg[i + 1];
        int64_t seg_hi = v[y - 1];
        qlo[i] = (i == 0) ? v[x] : qhi[i - 1];
        if (i + 1 < m) {
            int64_t next_lo = v[y];
            qhi[i] = (int32_t)((seg_hi + next_lo) / 2 + 1);   /* both >= 1: '/' floors */
        } else {
            qhi[i] = (int32_t)(seg_hi + 1);
        }
        qc[i] = N[y] - N[x]; qs1[i] = S1[y] - S1[x]; qs2[i] = S2[y] - S2[x];
    }

    /* Stage 3 */
    int64_t merges = 0;
    m = or_prune(m, qlo, qhi, qc, qs1, qs2, p->max_queues, p->epsilon, p->merge_rule, &merges);
    S.merges = merges;

    out->n = (int32_t)m;
    out->next_id = (int32_t)m;
    for (int64_t i = 0; i < m; i++) {
        or_queue *q = &out->q[i];
        q->id = (int32_t)i; q->index = (int32_t)(i + 1);
        q->min_len = qlo[i]; q->max_len = qhi[i];
        q->count = qc[i]; q->sum = qs1[i]; q->sumsq = qs2[i];
        q->mean = mean_of(qs1[i], qc[i]);
        q->density = rho_of(qc[i], qlo[i], qhi[i]);
        q->sse = (double)qs2[i] - ((double)qs1[i] * (double)qs1[i]) / (double)qc[i];
        q->is_bubble = 0;
    }
    free(v); free(c); free(N); free(S1); free(S2); free(seg);
    free(qlo); free(qhi); free(qc); free(qs1); free(qs2);
    if (st) *st = S;
    return S.n_invalid ? OR_DOMAIN : OR_OK;     /* b < 1 is a domain error */
}

/* O14 partition: k clusters from or_kmeans_dp, then O5's finalisation (R15) and
 * the queue profiles; no Stage 2 or 3 (Table 3 "EWSJF (K-Means)"). */
int or_partition_kmeans(const int32_t *len, int64_t n, int32_t k, or_partition *out, or_partition_stats *st) {
    or_partition_stats S;
    memset(&S, 0, sizeof S);
    memset(out, 0, sizeof *out);
    if (k < 1 || k > OR_MAXQ || n < 0) return OR_INVALID;
    size_t nn = (size_t)(n > 0 ? n : 1);
    int32_t *v = (int32_t *)malloc(sizeof(int32_t) * nn);
    int64_t *c = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t M = or_rle(len, n, v, c, &S.n_invalid);
    S.n_valid = n - S.n_invalid;
    S.distinct = M;
    if (M == 0) { free(v); free(c); if (st) *st = S; return OR_EMPTY; }
    int64_t *N  = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M + 1));
    int64_t *S1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M + 1));
    int64_t *S2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M + 1));
    or_prefix(v, c, M, N, S1, S2);
    int32_t ku = k < M ? k : (int32_t)M;
    int32_t *cuts = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ku > 1 ? ku : 1));
    or_kmeans_dp(N, S1, M, ku, cuts);
    S.k_used = ku;
    S.t1 = ku >= 2 ? cuts[0] : 0;
    S.t2 = ku >= 3 ? cuts[1] : 0;
    S.segments = ku;
    int64_t b[OR_MAXQ + 1];
    b[0] = 0;
    for (int32_t i = 0; i + 1 < ku; i++) b[i + 1] = cuts[i];
    b[ku] = M;
    out->n = ku;
    out->next_id = ku;
    for (int32_t i = 0; i < ku; i++) {
        int64_t x = b[i], y = b[i + 1];
        or_queue *q = &out->q[i];
        q->id = i; q->index = i + 1;
        q->min_len = (i == 0) ? v[x] : out->q[i - 1].max_len;
        q->max_len = (i + 1 < ku) ? (int32_t)(((int64_t)v[y - 1] + (int64_t)v[y]) / 2 + 1) : v[y - 1] + 1;
        q->count = N[y] - N[x]; q->sum = S1[y] - S1[x]; q->sumsq = S2[y] - S2[x];
        q->mean = mean_of(q->sum, q->count);
        q->density = rho_of(q->count, q->min_len, q->max_len);
        q->sse = (double)q->sumsq - ((double)q->sum * (double)q->sum) / (double)q->count;
        q->is_bubble = 0;
    }
    free(v); free(c); free(N); free(S1); free(S2); free(cuts);
    if (st) *st = S;
    return S.n_invalid ? OR_DOMAIN : OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O7  meta-policy w_x(b̄_q) = a_x·b̄_q + b_x (Θ "…" resolved
 * as base/urg/fair linear maps, R8), clamped >= 0, then cast
 * to fp32 (the value the device receives).                                 */
void or_weights(const or_meta *th, double mean, float w[3]) {
    double wb = th->a_b * mean; wb = wb + th->b_b;
    double wu = th->a_u * mean; wu = wu + th->b_u;
    double wf = th->a_f * mean; wf = wf + th->b_f;
    w[0] = (float)(wb > 0.0 ? wb : 0.0);
    w[1] = (float)(wu > 0.0 ? wu : 0.0);
    w[2] = (float)(wf > 0.0 ? wf : 0.0);
}

/* ------------------------------------------------------------------------- */
/* O8  Dispatcher: "Routes incoming requests to the appropriate queue based on
 * current prompt-length boundaries".  A gap-falling request triggers
 * Alg. 2 (App. D):
 *   L <= Q_i.max_len × 1.10      -> Q_i        (exact integer test 10L <= 11 max, R19)
 *   L >= Q_{i+1}.min_len × 0.90  -> Q_{i+1}    (10L >= 9 min, R19)
 *   else available = Q_{i+1}.min - Q_i.max, range = min(width, available),
 *        new = [max(L - range/2, Q_i.max), min(L + range/2, Q_{i+1}.min))
 *        with range/2 -> floor below, ceil above (R20).
 * Below the first queue there is no left neighbour: left bound 1; above the
 * last there is no right neighbour: right bound +inf (R20).  Requests are
 * processed in pool-index order (R22); bounds are never widened (R23).      */
static void insert_queue(or_partition *part, int32_t pos, int32_t lo, int32_t hi, int32_t L) {
    for (int32_t i = part->n; i > pos; i--) part->q[i] = part->q[i - 1];
    or_queue *q = &part->q[pos];
    memset(q, 0, sizeof *q);
    q->id = part->next_id++;
    q->min_len = lo; q->max_len = hi;
    q->mean = (double)L;                   /* R21 */
    q->is_bubble = 1;
    part->n++;
    for (int32_t i = 0; i < part->n; i++) part->q[i].index = i + 1;
}

int or_route(const int32_t *len, int64_t n, or_partition *part, int32_t bubble_width,
             int32_t *qid, int64_t *n_invalid, int64_t *n_bubbles, int64_t *n_dropped) {
    int64_t bad = 0, made = 0, dropped = 0;
    if (bubble_width < 1) return OR_INVALID;
    for (int64_t r = 0; r < n; r++) {
        int32_t L = len[r];
        if (L < 1) { qid[r] = -1; bad++; continue; }
        /* i = last queue with min_len <= L (binary search over the current partition) */
        int32_t a = 0, b = part->n;               /* count of queues with min_len <= L */
        while (a < b) {
            int32_t mid = (a + b) / 2;
            if (part->q[mid].min_len <= L) a = mid + 1; else b = mid;
        }
        int32_t i = a - 1;
        if (i >= 0 && L < part->q[i].max_len) { qid[r] = part->q[i].id; continue; }
        int has_l = (i >= 0), has_r = (i + 1 < part->n);
        int64_t L64 = L;
        if (has_l && 10 * L64 <= 11 * (int64_t)part->q[i].max_len) { qid[r] = part->q[i].id; continue; }
        if (has_r && 10 * L64 >= 9 * (int64_t)part->q[i + 1].min_len) { qid[r] = part->q[i + 1].id; continue; }
        if (part->n >= OR_MAXQ) { qid[r] = -1; dropped++; continue; }
        int64_t lb = has_l ? part->q[i].max_len : 1;
        int64_t rb = has_r ? part->q[i + 1].min_len : ((int64_t)1 << 40);
        int64_t avail = rb - lb;
        int64_t range = (int64_t)bubble_width < avail ? (int64_t)bubble_width : avail;
        int64_t nlo = L64 - range / 2;          if (nlo < lb) nlo = lb;
        int64_t nhi = L64 + (range + 1) / 2;    if (nhi > rb) nhi = rb;
        if (nhi > (int64_t)INT32_MAX) nhi = INT32_MAX;
        insert_queue(part, i + 1, (int32_t)nlo, (int32_t)nhi, L);
        qid[r] = part->q[i + 1].id;
        made++;
    }
    if (n_invalid) *n_invalid = bad;
    if (n_bubbles) *n_bubbles = made;
    if (n_dropped) *n_dropped = dropped;
    return dropped ? OR_CAPACITY : OR_OK;
}

/* ------------------------------------------------------------------------- */
/* O9  Eq. 4, = Eq. 1:
 *   Φ(r,q) = qf · (w_base + w_urg·cs + w_fair·log(b+1)),
 *   cs = W_t / C_prefill(b), qf = q_i/(b+1).
 * R2 natural log; R3 q_i 1-based ascending; R4 C = cost[r] or c0+c1 b+c2 b²
 * (S:222); R5 W_t = now - arrival, W < 0 is a contract violation ->
 * excluded; C <= 0 is a domain error -> excluded.  fp64 from the fp32
 * inputs exactly as stored.                                                */
int or_score_one(int32_t b, float arrival, const float *cost_or_null, int32_t index,
                 const float w[3], const or_select_params *sp, double *phi) {
    double W = (double)sp->now - (double)arrival;
    if (!(W >= 0.0)) return 1;
    double bd = (double)b;
    double C;
    if (cost_or_null) C = (double)(*cost_or_null);
    else C = (double)sp->c0 + (double)sp->c1 * bd + (double)sp->c2 * bd * bd;
    if (!(C > 0.0)) return 1;
    double qf = (double)index / (bd + 1.0);
    double cs = W / C;
    double inner = ((double)w[0] + (double)w[1] * cs) + (double)w[2] * log(bd + 1.0);
    *phi = qf * inner;
    return 0;
}

/* O10  Alg. 1: per non-empty queue the head request ("the oldest
 * request r in queue q"; R26: min (arrival, index)) is scored and the
 * argmax queue is primary (ties -> lowest index, R24).  Per the
 * north_star every request is scored and each queue's top-K is returned
 * (R1): SCORE key (Φ desc, index asc) or FIFO key (arrival asc, index asc),
 * by a full sort of the queue's members.                                    */
typedef struct { double k; int64_t r; } skey;
static int cmp_skey(const void *a, const void *b) {
    const skey *x = (const skey *)a, *y = (const skey *)b;
    if (x->k < y->k) return -1;
    if (x->k > y->k) return 1;
    return (x->r > y->r) - (x->r < y->r);
}
typedef struct { int32_t id, pos; } idpos;
static int cmp_idpos(const void *a, const void *b) {
    const idpos *x = (const idpos *)a, *y = (const idpos *)b;
    return (x->id > y->id) - (x->id < y->id);
}

int or_score_select(const int32_t *len, const float *arrival, const float *cost,
                    const int32_t *qid, int64_t n, int64_t global_base,
                    const or_partition *part, const float *w,
                    const or_select_params *sp, or_select_out *out) {
    int32_t nq = part->n, K = sp->k;
    if (K < 1 || (sp->mode != OR_SCORE && sp->mode != OR_FIFO)) return OR_INVALID;
    idpos map[OR_MAXQ];
    for (int32_t i = 0; i < nq; i++) { map[i].id = part->q[i].id; map[i].pos = i; }
    qsort(map, (size_t)nq, sizeof(idpos), cmp_idpos);

    size_t nn = (size_t)(n > 0 ? n : 1);
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * nn);
    double *phi = (double *)malloc(sizeof(double) * nn);
    int64_t *cnt = (int64_t *)calloc((size_t)nq + 1, sizeof(int64_t));
    int64_t excl = 0, bad = 0;
    for (int64_t r = 0; r < n; r++) {
        pos[r] = -1;
        if (qid[r] < 0) { bad++; continue; }
        int32_t a = 0, b = nq;
        while (a < b) { int32_t mid = (a + b) / 2; if (map[mid].id < qid[r]) a = mid + 1; else b = mid; }
        if (a >= nq || map[a].id != qid[r] || len[r] < 1) { bad++; continue; }
        int32_t p = map[a].pos;
        double f;
        if (or_score_one(len[r], arrival[r], cost ? &cost[r] : NULL, part->q[p].index, &w[3 * p], sp, &f)) {
            excl++; continue;
        }
        pos[r] = p; phi[r] = f; cnt[p]++;
    }
    /* bucket members per queue (index order within a bucket) */
    int64_t *start = (int64_t *)calloc((size_t)nq + 1, sizeof(int64_t));
    for (int32_t p = 0; p < nq; p++) start[p + 1] = start[p] + cnt[p];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)nq + 1));
    memcpy(fill, start, sizeof(int64_t) * ((size_t)nq + 1));
    int64_t *mem = (int64_t *)malloc(sizeof(int64_t) * (size_t)(start[nq] > 0 ? start[nq] : 1));
    for (int64_t r = 0; r < n; r++) if (pos[r] >= 0) mem[fill[pos[r]]++] = r;

    out->primary = -1;
    double best_head = 0.0;
    for (int32_t p = 0; p < nq; p++) {
        int64_t m = cnt[p];
        int64_t *M_ = mem + start[p];
        out->count[p] = m;
        for (int32_t t = 0; t < K; t++) { out->topk_id[(size_t)p * K + t] = -1; out->topk_score[(size_t)p * K + t] = 0.0; }
        out->head_id[p] = -1; out->head_score[p] = 0.0; out->max_score[p] = 0.0;
        if (m == 0) continue;
        skey *ks = (skey *)malloc(sizeof(skey) * (size_t)m);
        /* head: min (arrival, r) */
        int64_t h = M_[0];
        for (int64_t t = 1; t < m; t++) {
            int64_t r = M_[t];
            if ((double)arrival[r] < (double)arrival[h] || ((double)arrival[r] == (double)arrival[h] && r < h)) h = r;
        }
        out->head_id[p] = h + global_base;
        out->head_score[p] = phi[h];
        /* max score: best in SCORE order */
        int64_t bs = M_[0];
        for (int64_t t = 1; t < m; t++) {
            int64_t r = M_[t];
            if (phi[r] > phi[bs] || (phi[r] == phi[bs] && r < bs)) bs = r;
        }
        out->max_score[p] = phi[bs];
        for (int64_t t = 0; t < m; t++) {
            int64_t r = M_[t];
            ks[t].r = r;
            ks[t].k = (sp->mode == OR_SCORE) ? -phi[r] : (double)arrival[r];
        }
        qsort(ks, (size_t)m, sizeof(skey), cmp_skey);
        for (int64_t t = 0; t < m && t < K; t++) {
            out->topk_id[(size_t)p * K + t] = ks[t].r + global_base;
            out->topk_score[(size_t)p * K + t] = phi[ks[t].r];
        }
        free(ks);
        if (out->primary < 0 || out->head_score[p] > best_head) { out->primary = p; best_head = out->head_score[p]; }
    }
    out->n_excluded = excl;
    out->n_invalid = bad;
    free(pos); free(phi); free(cnt); free(start); free(fill); free(mem);
    return (excl || bad) ? OR_DOMAIN : OR_OK;
}

/* O8 + O7 + O9 + O10: one tactical tick over the whole pending pool. */
int or_tick(const int32_t *len, const float *arrival, const float *cost, int64_t n,
            int64_t global_base, or_partition *part, int32_t bubble_width,
            const or_meta *theta, const or_select_params *sp,
            int32_t *qid_out, or_select_out *out) {
    int64_t inv = 0, made = 0, dropped = 0;
    if (sp->k < 1 || (sp->mode != OR_SCORE && sp->mode != OR_FIFO) || bubble_width < 1) return OR_INVALID;
    int rs = or_route(len, n, part, bubble_width, qid_out, &inv, &made, &dropped);
    float w[3 * OR_MAXQ];
    for (int32_t p = 0; p < part->n; p++) or_weights(theta, part->q[p].mean, &w[3 * p]);
    int ss = or_score_select(len, arrival, cost, qid_out, n, global_base, part, w, sp, out);
    out->n_invalid = inv + dropped;
    out->n_bubbles = made;
    out->n_dropped = dropped;
    if (rs == OR_CAPACITY) return OR_CAPACITY;
    if (ss == OR_DOMAIN || inv) return OR_DOMAIN;
    return ss;
}

/* O9 over a routed pool (for comparators): phi[r] and valid[r] per request. */
void or_score_all(const int32_t *len, const float *arrival, const float *cost, const int32_t *qid, int64_t n,
                  const or_partition *part, const float *w, const or_select_params *sp,
                  double *phi, int8_t *valid) {
    for (int64_t r = 0; r < n; r++) {
        valid[r] = 0; phi[r] = 0.0;
        if (qid[r] < 0 || len[r] < 1) continue;
        int32_t p = -1;
        for (int32_t i = 0; i < part->n; i++) if (part->q[i].id == qid[r]) { p = i; break; }
        if (p < 0) continue;
        double f;
        if (!or_score_one(len[r], arrival[r], cost ? &cost[r] : NULL, part->q[p].index, &w[3 * p], sp, &f)) {
            phi[r] = f; valid[r] = 1;
        }
    }
}

/* O11 (A12): Θ sweep.  The meta-optimizer proposes Θ, evaluates the policy and
 * keeps the best; its inner loop over one snapshot is,
 * for every Θ, exactly one tactical scoring pass: O7 weights from Θ and the
 * queue means, O9 scores (Eq. 4), O10 selection (Alg. 1 + top-K). */
int or_sweep(const int32_t *len, const float *arrival, const float *cost, const int32_t *qid,
             int64_t n, int64_t global_base, const or_partition *part,
             const or_meta *thetas, int32_t n_theta, const or_select_params *sp,
             or_select_out *outs) {
    if (n_theta < 0 || sp->mode != OR_SCORE) return OR_INVALID;
    int status = OR_OK;
    float w[3 * OR_MAXQ];
    for (int32_t t = 0; t < n_theta; t++) {
        for (int32_t p = 0; p < part->n; p++) or_weights(&thetas[t], part->q[p].mean, &w[3 * p]);
        int s = or_score_select(len, arrival, cost, qid, n, global_base, part, w, sp, &outs[t]);
        if (status == OR_OK) status = s;
    }
    return status;
}

/* ---------------------------------------------------------------- O12 --- */
typedef struct { float arrival; int64_t r; } fkey;
static int cmp_fkey(const void *a, const void *b) {
    const fkey *x = (const fkey *)a, *y = (const fkey *)b;
    if ((double)x->arrival < (double)y->arrival) return -1;
    if ((double)x->arrival > (double)y->arrival) return 1;
    return x->r < y->r ? -1 : (x->r > y->r);
}

/* Pull queue p's members in FIFO order while the budget admits them (Alg. 1
 * GreedyFill / Backfill body; S:324 (3)-(4); first request of the batch always
 * admitted). */
static void pull_fifo(const fkey *mem, int64_t m, const int32_t *len, int64_t global_base, const or_budget *bd,
                      int64_t *batch_ids, int64_t *nb, int64_t *tok) {
    for (int64_t t = 0; t < m; t++) {
        if (*nb >= bd->max_requests) return;
        const int64_t b = len[mem[t].r];
        if (*nb > 0 && *tok + b > bd->max_tokens) return;     /* stop at the first that does not fit (R28) */
        batch_ids[(*nb)++] = global_base + mem[t].r;
        *tok += b;
    }
}

int64_t or_batch(const int32_t *len, const float *arrival, const float *cost, const int32_t *qid,
                 int64_t n, int64_t global_base, const or_partition *part, const or_select_params *sp,
                 int32_t primary, const or_budget *budget, int64_t *batch_ids, int64_t *batch_tokens) {
    int32_t nq = part->n;
    *batch_tokens = 0;
    if (primary < 0 || primary >= nq || budget->max_requests < 1) return 0;
    idpos map[OR_MAXQ];
    for (int32_t i = 0; i < nq; i++) { map[i].id = part->q[i].id; map[i].pos = i; }
    qsort(map, (size_t)nq, sizeof(idpos), cmp_idpos);
    /* members per position: what O9 scores (the weights do not matter for validity) */
    const float w0[3] = {1.0f, 0.0f, 0.0f};
    int64_t *cnt = (int64_t *)calloc((size_t)nq + 1, sizeof(int64_t));
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t r = 0; r < n; r++) {
        pos[r] = -1;
        if (qid[r] < 0 || len[r] < 1) continue;
        int32_t a = 0, b = nq;
        while (a < b) { int32_t mid = (a + b) / 2; if (map[mid].id < qid[r]) a = mid + 1; else b = mid; }
        if (a >= nq || map[a].id != qid[r]) continue;
        double f;
        if (or_score_one(len[r], arrival[r], cost ? &cost[r] : NULL, 1, w0, sp, &f)) continue;
        pos[r] = map[a].pos;
        cnt[pos[r]]++;
    }
    int64_t *start = (int64_t *)calloc((size_t)nq + 1, sizeof(int64_t));
    for (int32_t p = 0; p < nq; p++) start[p + 1] = start[p] + cnt[p];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)nq + 1));
    memcpy(fill, start, sizeof(int64_t) * ((size_t)nq + 1));
    fkey *mem = (fkey *)malloc(sizeof(fkey) * (size_t)(start[nq] > 0 ? start[nq] : 1));
    for (int64_t r = 0; r < n; r++)
        if (pos[r] >= 0) { fkey k; k.arrival = arrival[r]; k.r = r; mem[fill[pos[r]]++] = k; }
    for (int32_t p = 0; p < nq; p++) qsort(mem + start[p], (size_t)cnt[p], sizeof(fkey), cmp_fkey);

    int64_t nb = 0, tok = 0;
    /* GreedyFill from the primary queue (Alg. 1 line 16) */
    pull_fifo(mem + start[primary], cnt[primary], len, global_base, budget, batch_ids, &nb, &tok);
    /* Backfill from adjacent queues, nearest index first, lower neighbour first (lines 17-19) */
    for (int32_t d = 1; d < nq && nb < budget->max_requests; d++) {
        const int32_t cand[2] = {primary - d, primary + d};
        for (int c = 0; c < 2 && nb < budget->max_requests; c++) {
            const int32_t p = cand[c];
            if (p < 0 || p >= nq) continue;
            pull_fifo(mem + start[p], cnt[p], len, global_base, budget, batch_ids, &nb, &tok);
        }
    }
    *batch_tokens = tok;
    free(cnt); free(pos); free(start); free(fill); free(mem);
    return nb;
}

int32_t or_prune_empty(or_partition *part, int32_t *empty_cnt, const int64_t *count, int32_t threshold) {
    int32_t k = 0, removed = 0;
    for (int32_t p = 0; p < part->n; p++) {
        int32_t e = empty_cnt[p];
        /* Alg. 1 line 9; empty_count counts CONSECUTIVE empty tactical steps
           (S:107), so a queue with members resets it (R30) */
        e = count[p] == 0 ? e + 1 : 0;
        if (e > threshold) { removed++; continue; }       /* lines 10-11, strict (R25) */
        part->q[k] = part->q[p];
        part->q[k].index = k + 1;                         /* renumber */
        empty_cnt[k] = e;
        k++;
    }
    part->n = k;
    return removed;
}

/* ---------------------------------------------------------------- O13 ---- */
int32_t or_online_adjust(const int32_t *window, int64_t n, double max_shift, or_partition *part) {
    const int32_t nq = part->n;
    if (nq < 2 || n <= 0) return 0;
    int32_t newb[OR_MAXQ];
    int32_t *loc = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t moved = 0;
    for (int32_t i = 1; i < nq; i++) {
        const or_queue *qa = &part->q[i - 1], *qb = &part->q[i];
        const int32_t B = qb->min_len;
        newb[i] = B;
        if (qa->max_len != B) continue;                 /* not a shared boundary */
        const int32_t L = qa->min_len, U = qb->max_len;
        const int64_t ca = qa->count, cb = qb->count;
        if (ca + cb == 0) continue;
        int64_t m = 0;                                  /* the window's members in [L, U) */
        for (int64_t r = 0; r < n; r++)
            if (window[r] >= 1 && window[r] >= L && window[r] < U) loc[m++] = window[r];
        if (m == 0) continue;
        qsort(loc, (size_t)m, sizeof(int32_t), cmp_i32);
        const int64_t k = (m * ca + (ca + cb) - 1) / (ca + cb);     /* ceil(m ca / (ca + cb)) */
        const int32_t T = k == 0 ? L : loc[k - 1] + 1;
        int64_t d = (int64_t)T - B;
        const int64_t left = (int64_t)floor(max_shift * (double)(B - L));
        const int64_t right = (int64_t)floor(max_shift * (double)(U - B));
        if (d < -left) d = -left;
        if (d > right) d = right;
        newb[i] = (int32_t)(B + d);
    }
    for (int32_t i = 1; i < nq; i++) {
        if (newb[i] == part->q[i].min_len) continue;
        part->q[i - 1].max_len = newb[i];
        part->q[i].min_len = newb[i];
        moved++;
    }
    free(loc);
    return moved;
}
