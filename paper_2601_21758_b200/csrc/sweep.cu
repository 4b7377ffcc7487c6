// sweep.cu — Θ-batched score + select (A12, config C5).  (Implemented later.)
#include "tick.cuh"

extern "C" ewsjf_status ewsjf_score_select_sweep(ewsjf_ctx* ctx, const int32_t* d_len, const float* d_arrival,
                                                 const float* d_cost, const int32_t* d_qid, int64_t n,
                                                 const ewsjf_partition_t* part, const ewsjf_meta* thetas,
                                                 int32_t n_theta, const ewsjf_select_params* params,
                                                 ewsjf_select_out* outs) {
    (void)ctx; (void)d_len; (void)d_arrival; (void)d_cost; (void)d_qid; (void)n; (void)part; (void)thetas;
    (void)n_theta; (void)params; (void)outs;
    return EWSJF_ERR_UNSUPPORTED;
}
