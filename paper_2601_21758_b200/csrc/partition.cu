// partition.cu — Refine-and-Prune (A1-A6) on sm_100a.  (Implemented in the next step.)
#include "tick.cuh"

struct ewsjf_ctx;
namespace ewsjf {
void rp_free(ewsjf_ctx*) {}
}

extern "C" ewsjf_status ewsjf_partition(ewsjf_ctx* ctx, const int32_t* d_len, int64_t n,
                                        const ewsjf_partition_params* params, ewsjf_partition_t* out,
                                        ewsjf_partition_stats* stats) {
    (void)ctx; (void)d_len; (void)n; (void)params; (void)out; (void)stats;
    return EWSJF_ERR_UNSUPPORTED;
}
