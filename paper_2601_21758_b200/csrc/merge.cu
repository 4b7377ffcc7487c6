// merge.cu — standalone merge kernel (exchange / route / multi-pass paths).
#include "merge.cuh"

namespace ewsjf {

template <int IN, int OUT, bool HAS_COST>
__global__ void __launch_bounds__(kMThreads, 1)
    merge_kernel(const __grid_constant__ MergeArgs A, const __grid_constant__ Policy P) {
    extern __shared__ __align__(128) unsigned char smem[];
    merge_phase<IN, OUT, HAS_COST>(A, P, smem);
}

// ---------------------------------------------------------------- launch ---
int64_t merge_smem_total(int in_mode) { return merge_layout(in_mode).total; }

template <int I, int O, bool C>
static cudaError_t launch_merge_t(const MergeArgs& A, const Policy& P, int grid, cudaStream_t st) {
    const MergeSmem L = merge_layout(I);
    auto k = merge_kernel<I, O, C>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    k<<<grid, kMThreads, L.total, st>>>(A, P);
    return cudaGetLastError();
}

cudaError_t launch_merge(const MergeArgs& A, const Policy& P, bool has_cost, int grid, cudaStream_t st) {
    if (A.in_mode == MERGE_IN_ROWS) {
        if (A.out_mode == MERGE_OUT_FINAL)
            return has_cost ? launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_FINAL, true>(A, P, grid, st)
                            : launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_FINAL, false>(A, P, grid, st);
        if (A.out_mode == MERGE_OUT_EXCHANGE)
            return has_cost ? launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_EXCHANGE, true>(A, P, grid, st)
                            : launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_EXCHANGE, false>(A, P, grid, st);
        return launch_merge_t<MERGE_IN_ROWS, MERGE_OUT_ROUTE, false>(A, P, grid, st);
    }
    return launch_merge_t<MERGE_IN_EXCHANGE, MERGE_OUT_FINAL, false>(A, P, grid, st);
}

}  // namespace ewsjf
