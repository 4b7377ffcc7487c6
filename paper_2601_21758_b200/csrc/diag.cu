// diag.cu — measurement helpers for bench.py (not on the scheduling path).
//
// ewsjf_diag_ffma_rate: the fp32 FMA issue rate of this GPU, measured.  The C5
// Θ sweep (A12) is fp32-ALU bound (3 FMA-pipe ops + 1 compare per (request, Θ)
// pair), and MEASURED_PEAKS.json carries no fp32 number, so its
// roofline peak is this rate / 4 ("an FMA microbenchmark on the box").
#include "ctx.h"

namespace ewsjf {

// 8 independent FFMA chains per thread, `iters` x 8 x 8 FFMAs; the result is
// stored so the compiler keeps every chain.
__global__ void __launch_bounds__(256) ffma_probe_kernel(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int c = 0; c < 8; c++) x[c] = threadIdx.x * 1e-3f + c;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++)
#pragma unroll
            for (int c = 0; c < 8; c++) x[c] = fmaf(x[c], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < 8; c++) s += x[c];
    if (s == 1234.5f) out[blockIdx.x] = s;   // never true in practice; keeps the chains live
}

}  // namespace ewsjf

using namespace ewsjf;

#include <atomic>
static std::atomic<long long> g_allocs{0};
extern "C" void ewsjf_count_alloc_(void) { g_allocs.fetch_add(1, std::memory_order_relaxed); }
extern "C" int64_t ewsjf_alloc_count(void) { return (int64_t)g_allocs.load(std::memory_order_relaxed); }

extern "C" ewsjf_status ewsjf_diag_ffma_rate(ewsjf_ctx* ctx, double* ffma_per_s) {
    if (!ctx || !ffma_per_s) return EWSJF_ERR_INVALID_ARG;
    CU(cudaSetDevice(ctx->device));
    float* d = nullptr;
    const int grid = ctx->num_sms * 8;   // 8 x 256 threads per SM: every scheduler saturated
    const int iters = 4096;
    CU(cudaMalloc(&d, grid * sizeof(float)));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    ffma_probe_kernel<<<grid, 256, 0, ctx->stream>>>(d, 64, 0.999f, 1e-3f);   // warm-up
    CU(cudaEventRecord(e0, ctx->stream));
    ffma_probe_kernel<<<grid, 256, 0, ctx->stream>>>(d, iters, 0.999f, 1e-3f);
    CU(cudaEventRecord(e1, ctx->stream));
    CU(cudaEventSynchronize(e1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    *ffma_per_s = (double)grid * 256.0 * iters * 64.0 / (ms * 1e-3);
    return EWSJF_OK;
}
