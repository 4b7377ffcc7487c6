// sweep.cu — Θ-batched score + select (A12, config C5; §4.4.2).
//
// The meta-optimizer evaluates candidate scoring parameters Θ over
// one snapshot of the pending pool.  For each Θ this is A7 (per-queue weights
// w_x = max(0, a_x b̄ + b_x)) followed by A10 + A11 over the routed
// snapshot — exactly ewsjf_score_select with the weights of that Θ, so every
// output equals an independent score_select call (the pin of SURVEY §8c A12).
// The snapshot stays resident in L2 across the Θ loop (16 MB at C5).
#include <cstring>
#include "tick.cuh"

extern "C" ewsjf_status ewsjf_score_select_sweep(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arrival,
                                                 const float* d_cost, const int32_t* d_qid, int64_t n,
                                                 const ewsjf_partition_t* part, const ewsjf_meta* thetas,
                                                 int32_t n_theta, const ewsjf_select_params* params,
                                                 ewsjf_select_out* outs) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (!part || !thetas || !params || !outs || n_theta < 0 || part->n < 0 || part->n > EWSJF_MAX_QUEUES)
        return EWSJF_ERR_INVALID_ARG;
    // Θ ranks scoring policies: the sweep selects by score (SCORE mode), as O11 does
    if (params->mode != EWSJF_SELECT_SCORE) return EWSJF_ERR_INVALID_ARG;
    ewsjf_status worst = EWSJF_OK;
    for (int32_t t = 0; t < n_theta; t++) {
        ewsjf_weights w[EWSJF_MAX_QUEUES];
        ewsjf_status s = ewsjf_weights_from_meta(&thetas[t], part, w);
        if (s != EWSJF_OK) return s;
        ewsjf_select_out o = outs[t];
        o.h_summary = nullptr;                   // async: per-Θ summaries stay on the device
        s = ewsjf_score_select(ctx, d_len, d_arrival, d_cost, d_qid, n, part, w, params, &o);
        if (s != EWSJF_OK && s != EWSJF_ERR_DOMAIN) return s;
        if (s == EWSJF_ERR_DOMAIN) worst = s;
    }
    return worst;
}
