// mb_launch.cu — launch + teardown cost of an (almost) empty kernel by configuration:
// 148 CTAs x 768 threads, dynamic shared memory, parameter block size, cooperative launch.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb_launch tools/mb_launch.cu
#include <cstdio>
#include <cuda_runtime.h>
struct Big { char b[760]; };
__global__ void __launch_bounds__(768, 1) k_small(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 1; }
__global__ void __launch_bounds__(768, 1) k_big(const __grid_constant__ Big a, int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = a.b[blockIdx.x % 760]; }
template <typename F>
static void timeit(const char* name, F launch) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 20; i++) launch();
    cudaDeviceSynchronize();
    float best = 1e9f, sum = 0.f;
    for (int i = 0; i < 200; i++) {
        cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; sum += ms;
    }
    printf("%-40s best %6.2f us  mean %6.2f us  (%s)\n", name, best * 1e3, sum / 200 * 1e3, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    int* p; cudaMalloc(&p, 4096);
    int G; cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
    Big b{};
    for (int smem : {0, 100 * 1024, 184 * 1024, 220 * 1024}) {
        cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        char nm[64];
        snprintf(nm, 64, "small params, smem %d KB", smem / 1024);
        timeit(nm, [&] { k_small<<<G, 768, smem>>>(p); });
        snprintf(nm, 64, "760 B params, smem %d KB", smem / 1024);
        timeit(nm, [&] { k_big<<<G, 768, smem>>>(b, p); });
        snprintf(nm, 64, "coop small, smem %d KB", smem / 1024);
        timeit(nm, [&] { void* a[] = {&p}; cudaLaunchCooperativeKernel((void*)k_small, G, 768, a, smem, 0); });
        snprintf(nm, 64, "coop 760 B, smem %d KB", smem / 1024);
        timeit(nm, [&] { void* a[] = {&b, &p}; cudaLaunchCooperativeKernel((void*)k_big, G, 768, a, smem, 0); });
    }
    return 0;
}
