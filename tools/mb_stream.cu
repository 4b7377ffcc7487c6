// mb_stream.cu — microbenchmark of the fused tick's memory pipeline alone (no
// scoring): 3 fp32/int32 input arrays read, one int32 array written, 16 B per
// request, 10M requests, rotating 3 pool copies (480 MB > L2).  Variants:
//   ring<T, R>: per-warp cp.async (LDGSTS) ring of R 128-request tiles, T threads per
//               CTA, one CTA per SM, dynamic tile claims in batches of 4 (ftick's scheme)
//   direct<T, D>: LDG.128 straight into registers, D tiles in flight per warp
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb_stream tools/mb_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ void cp16(void* d, const void* s) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(s) : "memory");
}
template <int N> __device__ __forceinline__ void waitn() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int T, int R>
__global__ void __launch_bounds__(T, 1) ring(const int* __restrict__ len, const float* __restrict__ arr,
                                             const float* __restrict__ cost, int* __restrict__ qid, int64_t n,
                                             unsigned long long* ctr) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* ring = sm + warp * R * 3 * 512;
    const int ntiles = (int)(n / 128);
    // static first R tiles per warp, then dynamic claims of 4
    const int GW = gridDim.x * (T / 32);
    const int w = warp * gridDim.x + blockIdx.x;
    int tq[R];
    int seq = 0;
    unsigned long long cb = 0; int dc = 0, de = 0;
    auto next = [&]() -> int {
        if (seq < R) { int t = w + GW * seq++; return t < ntiles ? t : -1; }
        if (dc >= de) {
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(ctr, 4ull);
            b = __shfl_sync(0xffffffffu, b, 0);
            dc = (int)b + GW * R; de = dc + 4;
        }
        const int t = dc++;
        return t < ntiles ? t : -1;
    };
    auto issue = [&](int st, int t) {
        if (t >= 0) {
            const int64_t o = (int64_t)t * 128 + 4 * lane;
            cp16(ring + (st * 3 + 0) * 512 + 16 * lane, len + o);
            cp16(ring + (st * 3 + 1) * 512 + 16 * lane, arr + o);
            cp16(ring + (st * 3 + 2) * 512 + 16 * lane, cost + o);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int j = 0; j < R; j++) { tq[j] = next(); issue(j, tq[j]); }
    int st = 0;
    for (;;) {
        const int t = tq[0];
        if (t < 0) break;
        waitn<R - 1>();
        const int4 b = ((const int4*)(ring + (st * 3 + 0) * 512))[lane];
        const int4 a = ((const int4*)(ring + (st * 3 + 1) * 512))[lane];
        const int4 c = ((const int4*)(ring + (st * 3 + 2) * 512))[lane];
        __stcs((int4*)(qid + (int64_t)t * 128 + 4 * lane),
               make_int4(b.x ^ a.x ^ c.x, b.y ^ a.y ^ c.y, b.z ^ a.z ^ c.z, b.w ^ a.w ^ c.w));
        __syncwarp();
#pragma unroll
        for (int j = 0; j + 1 < R; j++) tq[j] = tq[j + 1];
        tq[R - 1] = next();
        issue(st, tq[R - 1]);
        st = st + 1 == R ? 0 : st + 1;
    }
}

template <int T, int D>
__global__ void __launch_bounds__(T, 1) direct(const int* __restrict__ len, const float* __restrict__ arr,
                                               const float* __restrict__ cost, int* __restrict__ qid, int64_t n,
                                               unsigned long long* ctr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ntiles = (int)(n / 128);
    const int GW = gridDim.x * (T / 32);
    const int w = warp * gridDim.x + blockIdx.x;
    // static round-robin: tile w + GW*i
    int4 b[D], a[D], c[D];
    int t0 = w;
#pragma unroll
    for (int j = 0; j < D; j++) {
        const int t = t0 + GW * j;
        if (t < ntiles) {
            const int64_t o = (int64_t)t * 128 + 4 * lane;
            b[j] = __ldcs((const int4*)(len + o)); a[j] = __ldcs((const int4*)(arr + o)); c[j] = __ldcs((const int4*)(cost + o));
        }
    }
    for (int base = t0; base < ntiles; base += GW * D) {
#pragma unroll
        for (int j = 0; j < D; j++) {
            const int t = base + GW * j;
            if (t < ntiles) {
                __stcs((int4*)(qid + (int64_t)t * 128 + 4 * lane),
                       make_int4(b[j].x ^ a[j].x ^ c[j].x, b[j].y ^ a[j].y ^ c[j].y, b[j].z ^ a[j].z ^ c[j].z,
                                 b[j].w ^ a[j].w ^ c[j].w));
            }
            const int tn = t + GW * D;
            if (tn < ntiles) {
                const int64_t o = (int64_t)tn * 128 + 4 * lane;
                b[j] = __ldcs((const int4*)(len + o)); a[j] = __ldcs((const int4*)(arr + o)); c[j] = __ldcs((const int4*)(cost + o));
            }
        }
    }
}


// direct loads with ftick's tile schedule: contiguous block per warp (blk = warp*G + cta),
// the first S0 tiles static, the rest claimed in batches of 4 from a counter (DYN), or the
// whole block static (!DYN).  P tiles after the D in flight are bulk-prefetched into L2 at
// launch, then every warp idles WAIT ns (the sample-bound wait of the tick) before streaming.
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
template <int T, int D, bool DYN>
__global__ void __launch_bounds__(T, 1) blockd(const int* __restrict__ len, const float* __restrict__ arr,
                                               const float* __restrict__ cost, int* __restrict__ qid, int64_t n,
                                               unsigned long long* ctr, int P, int wait_ns) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ntiles = (int)(n / 128);
    const int GW = gridDim.x * (T / 32);
    const int blk = warp * gridDim.x + blockIdx.x;
    const int stride = ntiles / GW;
    const int S0 = DYN ? min(1 + D + P, stride) : stride;
    const int dynb = stride - S0;
    const int ndyn = ntiles - GW * S0;
    int seq = 0, dc = 0, de = 0, tn = 0, rb = 0;
    unsigned long long nb = 0;
    if (DYN && lane == 0) nb = atomicAdd(ctr, 4ull);
    auto next = [&]() -> int {
        if (seq < S0) return blk * stride + seq++;
        if (!DYN) { return -1; }
        if (dc >= de) {
            unsigned long long b = 0;
            if (lane == 0) { b = nb; nb = b < (unsigned long long)ndyn ? atomicAdd(ctr, 4ull) : b; }
            b = __shfl_sync(0xffffffffu, b, 0);
            if (b >= (unsigned long long)ndyn) return -1;
            const int d = (int)b;
            dc = d; de = min(d + 4, ndyn);
            if (d < GW * dynb) { const int q = d / dynb, r = d - q * dynb; tn = q * stride + S0 + r; rb = dynb - r; }
            else { tn = GW * stride + (d - GW * dynb); rb = 1 << 30; }
        }
        const int t = tn; dc++; tn++;
        if (--rb == 0) { if (tn < GW * stride) { tn += S0; rb = dynb; } else rb = 1 << 30; }
        return t;
    };
    if (P > 0 && lane < 3 && S0 > 1 + D) {
        const int t0 = blk * stride + 1 + D, np = min(P, S0 - 1 - D);
        const void* src = lane == 0 ? (const void*)(len + (int64_t)t0 * 128) : lane == 1 ? (const void*)(arr + (int64_t)t0 * 128) : (const void*)(cost + (int64_t)t0 * 128);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(np * 512) : "memory");
    }
    int4 b[D], a[D], c[D];
    int tq[D];
#pragma unroll
    for (int j = 0; j < D; j++) {
        tq[j] = next();
        if (tq[j] >= 0) {
            const int64_t o = (int64_t)tq[j] * 128 + 4 * lane;
            b[j] = __ldcs((const int4*)(len + o)); a[j] = __ldcs((const int4*)(arr + o)); c[j] = __ldcs((const int4*)(cost + o));
        }
    }
    if (wait_ns) { const unsigned long long t0 = gt(); while (gt() - t0 < (unsigned long long)wait_ns) __nanosleep(200); }
    for (;;) {
        if (tq[0] < 0) break;
#pragma unroll
        for (int j = 0; j < D; j++) {
            const int t = tq[j];
            if (t >= 0) {
                __stcs((int4*)(qid + (int64_t)t * 128 + 4 * lane),
                       make_int4(b[j].x ^ a[j].x ^ c[j].x, b[j].y ^ a[j].y ^ c[j].y, b[j].z ^ a[j].z ^ c[j].z,
                                 b[j].w ^ a[j].w ^ c[j].w));
                const int tn2 = next();
                tq[j] = tn2;
                if (tn2 >= 0) {
                    const int64_t o = (int64_t)tn2 * 128 + 4 * lane;
                    b[j] = __ldcs((const int4*)(len + o)); a[j] = __ldcs((const int4*)(arr + o)); c[j] = __ldcs((const int4*)(cost + o));
                }
            }
        }
        // keep the order: tq[0] is always the oldest (rotate by D each round)
    }
}
template <typename K>
static int run2(const char* name, K k, int T, int G, int** L, float** A, float** C, int** Q, int64_t n,
                unsigned long long* ctr, int P, int wait_ns, bool coop) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9f, sum = 0.f;
    const int reps = 30;
    for (int i = 0; i < reps + 3; i++) {
        const int c = i % 3;
        CK(cudaMemsetAsync(ctr, 0, 8));
        cudaEventRecord(e0);
        if (coop) {
            const int* l = L[c]; const float* a = A[c]; const float* cc = C[c]; int* q = Q[c]; int64_t nn = n;
            void* args[] = {(void*)&l, (void*)&a, (void*)&cc, (void*)&q, (void*)&nn, (void*)&ctr, (void*)&P, (void*)&wait_ns};
            CK(cudaLaunchCooperativeKernel((const void*)k, dim3(G), dim3(T), args, 0, 0));
        } else {
            k<<<G, T>>>(L[c], A[c], C[c], Q[c], n, ctr, P, wait_ns);
        }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 3) { best = ms < best ? ms : best; sum += ms; }
    }
    CK(cudaGetLastError());
    const double bytes = 16.0 * n;
    printf("%-34s best %7.2f us (%5.2f TB/s)  mean %7.2f us (%5.2f TB/s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e12,
           sum / reps * 1e3, bytes / (sum / reps * 1e-3) / 1e12);
    return 0;
}


// ring (LDGSTS) or direct with a static round-robin schedule (tile w + GW*i) for the first
// `stat` rounds, then single-tile claims from a counter (dynamic tail); P round-robin tiles
// after the first R prefetched into L2 at launch; optional WAIT ns idle after the prologue
template <int T, int R>
__global__ void __launch_bounds__(T, 1) ringrr(const int* __restrict__ len, const float* __restrict__ arr,
                                               const float* __restrict__ cost, int* __restrict__ qid, int64_t n,
                                               unsigned long long* ctr, int P, int wait_ns, int stat) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* ring = sm + warp * R * 3 * 512;
    const int ntiles = (int)(n / 128);
    const int GW = gridDim.x * (T / 32);
    const int w = warp * gridDim.x + blockIdx.x;
    const int nstat = min(stat, ntiles / GW);      // static rounds
    int seq = 0;
    unsigned long long nb = 0;
    auto next = [&]() -> int {
        if (seq < nstat) return w + GW * seq++;
        unsigned long long b = 0;
        if (lane == 0) { b = nb; nb = atomicAdd(ctr, 1ull); }
        b = __shfl_sync(0xffffffffu, b, 0);
        const long long t = (long long)GW * nstat + (long long)b;
        return t < ntiles ? (int)t : -1;
    };
    if (lane == 0 && nstat < 3 + R) nb = atomicAdd(ctr, 1ull);
    if (P > 0 && lane < 3 * P) {
        const int i = R + lane / 3, a = lane % 3;
        if (i < nstat) {
            const int64_t o = (int64_t)(w + GW * i) * 128;
            const void* src = a == 0 ? (const void*)(len + o) : a == 1 ? (const void*)(arr + o) : (const void*)(cost + o);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;" ::"l"(src) : "memory");
        }
    }
    auto issue = [&](int st, int t) {
        if (t >= 0) {
            const int64_t o = (int64_t)t * 128 + 4 * lane;
            cp16(ring + (st * 3 + 0) * 512 + 16 * lane, len + o);
            cp16(ring + (st * 3 + 1) * 512 + 16 * lane, arr + o);
            cp16(ring + (st * 3 + 2) * 512 + 16 * lane, cost + o);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int tq[R];
#pragma unroll
    for (int j = 0; j < R; j++) { tq[j] = next(); issue(j, tq[j]); }
    if (seq == nstat && lane == 0) nb = atomicAdd(ctr, 1ull);
    if (wait_ns) { const unsigned long long t0 = gt(); while (gt() - t0 < (unsigned long long)wait_ns) __nanosleep(200); }
    int st = 0;
    for (;;) {
        const int t = tq[0];
        if (t < 0) break;
        waitn<R - 1>();
        const int4 b = ((const int4*)(ring + (st * 3 + 0) * 512))[lane];
        const int4 a = ((const int4*)(ring + (st * 3 + 1) * 512))[lane];
        const int4 c = ((const int4*)(ring + (st * 3 + 2) * 512))[lane];
        __stcs((int4*)(qid + (int64_t)t * 128 + 4 * lane),
               make_int4(b.x ^ a.x ^ c.x, b.y ^ a.y ^ c.y, b.z ^ a.z ^ c.z, b.w ^ a.w ^ c.w));
        __syncwarp();
#pragma unroll
        for (int j = 0; j + 1 < R; j++) tq[j] = tq[j + 1];
        const bool was_stat = seq < nstat;
        tq[R - 1] = next();
        if (was_stat && seq == nstat && lane == 0) nb = atomicAdd(ctr, 1ull);   // first claim one tile ahead
        issue(st, tq[R - 1]);
        st = st + 1 == R ? 0 : st + 1;
    }
}
template <typename K>
static int run3(const char* name, K k, int T, size_t smem, int G, int** L, float** A, float** C, int** Q, int64_t n,
                unsigned long long* ctr, int P, int wait_ns, int stat) {
    if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9f, sum = 0.f;
    const int reps = 30;
    for (int i = 0; i < reps + 3; i++) {
        const int c = i % 3;
        CK(cudaMemsetAsync(ctr, 0, 8));
        cudaEventRecord(e0);
        k<<<G, T, smem>>>(L[c], A[c], C[c], Q[c], n, ctr, P, wait_ns, stat);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 3) { best = ms < best ? ms : best; sum += ms; }
    }
    CK(cudaGetLastError());
    const double bytes = 16.0 * n;
    printf("%-34s best %7.2f us (%5.2f TB/s)  mean %7.2f us (%5.2f TB/s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e12,
           sum / reps * 1e3, bytes / (sum / reps * 1e-3) / 1e12);
    return 0;
}


// CTA-level TMA pipeline: chunks of CH = 24*128 requests (contiguous per CTA, chunk
// cta + G*i), S stages of 3 bulk copies, a producer warp (warp 24) and 24 consumer warps
__device__ __forceinline__ void mbi(unsigned long long* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbwait(unsigned long long* b, unsigned ph) {
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbarrive(unsigned long long* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory"); }
__device__ __forceinline__ void mbexpect(unsigned long long* b, unsigned bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned bytes, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(s), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
template <int S>
__global__ void __launch_bounds__(800, 1) tmas(const int* __restrict__ len, const float* __restrict__ arr,
                                               const float* __restrict__ cost, int* __restrict__ qid, int64_t n,
                                               unsigned long long* ctr) {
    constexpr int CH = 24 * 128;
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned long long* full = (unsigned long long*)sm;
    unsigned long long* empty = full + S;
    unsigned char* buf = sm + 1024;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nch = (int)(n / CH);
    if (threadIdx.x == 0) { for (int s = 0; s < S; s++) { mbi(&full[s], 1); mbi(&empty[s], 24); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    if (warp == 24) {
        if (lane == 0) {
            int i = 0;
            for (int c = blockIdx.x; c < nch; c += gridDim.x, i++) {
                const int s = i % S;
                if (i >= S) mbwait(&empty[s], ((i / S) - 1) & 1);
                mbexpect(&full[s], 3 * CH * 4);
                const int64_t o = (int64_t)c * CH;
                bulk(buf + (s * 3 + 0) * CH * 4, len + o, CH * 4, &full[s]);
                bulk(buf + (s * 3 + 1) * CH * 4, arr + o, CH * 4, &full[s]);
                bulk(buf + (s * 3 + 2) * CH * 4, cost + o, CH * 4, &full[s]);
            }
        }
        return;
    }
    int i = 0;
    for (int c = blockIdx.x; c < nch; c += gridDim.x, i++) {
        const int s = i % S;
        mbwait(&full[s], (i / S) & 1);
        const int e = warp * 128 + 4 * lane;
        const int4 b = *(const int4*)(buf + (s * 3 + 0) * CH * 4 + e * 4);
        const int4 a = *(const int4*)(buf + (s * 3 + 1) * CH * 4 + e * 4);
        const int4 cc = *(const int4*)(buf + (s * 3 + 2) * CH * 4 + e * 4);
        __syncwarp();
        if (lane == 0) mbarrive(&empty[s]);
        __stcs((int4*)(qid + (int64_t)c * CH + e),
               make_int4(b.x ^ a.x ^ cc.x, b.y ^ a.y ^ cc.y, b.z ^ a.z ^ cc.z, b.w ^ a.w ^ cc.w));
    }
}


// CTA TMA pipeline split into groups of GWP warps (each group its own S stages, refilled by
// its last releasing warp), no producer warp; consumers optionally spin a pseudo-random
// 0..jit cycles per tile on about half of the tiles (the fused tick's rare path)
template <int S, int GWP>
__global__ void __launch_bounds__(768, 1) tmag(const int* __restrict__ len, const float* __restrict__ arr,
                                               const float* __restrict__ cost, int* __restrict__ qid, int64_t n,
                                               unsigned long long* ctr, int jit) {
    constexpr int CH = 24 * 128, GC = GWP * 128, NG = 24 / GWP;
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned long long* full = (unsigned long long*)sm;          // [NG][S]
    unsigned* rel = (unsigned*)(sm + 8 * NG * S);                 // [NG][S]
    unsigned char* buf = sm + 2048;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = warp / GWP;
    const int nch = (int)(n / CH);
    const int iters = blockIdx.x < nch ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto gbuf = [&](int s, int a) { return buf + ((size_t)(g * S + s) * 3 + a) * GC * 4; };
    auto issue = [&](int i) {
        if (i >= iters) return;
        const int s = i % S;
        const int64_t o = (int64_t)(blockIdx.x + (int64_t)gridDim.x * i) * CH + g * GC;
        unsigned long long* b = &full[g * S + s];
        mbexpect(b, 3 * GC * 4);
        bulk(gbuf(s, 0), len + o, GC * 4, b);
        bulk(gbuf(s, 1), arr + o, GC * 4, b);
        bulk(gbuf(s, 2), cost + o, GC * 4, b);
    };
    if (threadIdx.x == 0) { for (int s = 0; s < NG * S; s++) { mbi(&full[s], 1); rel[s] = 0; } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    if (warp % GWP == 0 && lane == 0) for (int i = 0; i < S; i++) issue(i);
    if (jit >= 100000) { const unsigned long long t0 = gt(); while (gt() - t0 < (unsigned long long)(jit - 100000)) __nanosleep(200); jit = 0; }
    for (int i = 0; i < iters; i++) {
        const int s = i % S;
        mbwait(&full[g * S + s], (i / S) & 1);
        const int e = (warp % GWP) * 128 + 4 * lane;
        const int4 b = *(const int4*)(gbuf(s, 0) + e * 4);
        const int4 a = *(const int4*)(gbuf(s, 1) + e * 4);
        const int4 cc = *(const int4*)(gbuf(s, 2) + e * 4);
        const int64_t c = blockIdx.x + (int64_t)gridDim.x * i;
        __stcs((int4*)(qid + c * CH + g * GC + e),
               make_int4(b.x ^ a.x ^ cc.x, b.y ^ a.y ^ cc.y, b.z ^ a.z ^ cc.z, b.w ^ a.w ^ cc.w));
        if (jit) {
            const unsigned h = (unsigned)(c * 24 + warp) * 2654435761u;
            if (h & 0x10000u) { const long long t0 = clock64(); while (clock64() - t0 < (long long)((h >> 20) % jit)) {} }
        }
        __syncwarp();
        if (lane == 0) { const unsigned o = atomicAdd(&rel[g * S + s], 1u); if (o % GWP == GWP - 1) issue(i + S); }
    }
}
template <typename K>
static int run4(const char* name, K k, size_t smem, int G, int** L, float** A, float** C, int** Q, int64_t n,
                unsigned long long* ctr, int jit) {
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9f, sum = 0.f;
    const int reps = 30;
    for (int i = 0; i < reps + 3; i++) {
        const int c = i % 3;
        cudaEventRecord(e0);
        k<<<G, 768, smem>>>(L[c], A[c], C[c], Q[c], n, ctr, jit);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 3) { best = ms < best ? ms : best; sum += ms; }
    }
    CK(cudaGetLastError());
    const double bytes = 16.0 * n;
    printf("%-34s best %7.2f us (%5.2f TB/s)  mean %7.2f us (%5.2f TB/s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e12,
           sum / reps * 1e3, bytes / (sum / reps * 1e-3) / 1e12);
    return 0;
}

template <typename K>
static int run(const char* name, K k, int T, size_t smem, int G, int** L, float** A, float** C, int** Q, int64_t n,
               unsigned long long* ctr) {
    if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9f, sum = 0.f;
    const int reps = 30;
    for (int i = 0; i < reps + 3; i++) {
        const int c = i % 3;
        CK(cudaMemsetAsync(ctr, 0, 8));
        cudaEventRecord(e0);
        k<<<G, T, smem>>>(L[c], A[c], C[c], Q[c], n, ctr);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 3) { best = ms < best ? ms : best; sum += ms; }
    }
    CK(cudaGetLastError());
    const double bytes = 16.0 * n;
    printf("%-22s best %7.2f us (%5.2f TB/s)  mean %7.2f us (%5.2f TB/s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e12,
           sum / reps * 1e3, bytes / (sum / reps * 1e-3) / 1e12);
    return 0;
}

int main() {
    const int64_t n = 10000000;
    int G = 0;
    cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
    int *L[3], *Q[3];
    float *A[3], *C[3];
    for (int c = 0; c < 3; c++) {
        CK(cudaMalloc(&L[c], n * 4)); CK(cudaMalloc(&A[c], n * 4)); CK(cudaMalloc(&C[c], n * 4)); CK(cudaMalloc(&Q[c], n * 4));
        CK(cudaMemset(L[c], 1, n * 4)); CK(cudaMemset(A[c], 2, n * 4)); CK(cudaMemset(C[c], 3, n * 4));
    }
    unsigned long long* ctr;
    CK(cudaMalloc(&ctr, 8));
    const size_t CHB = 3 * 24 * 128 * 4;
    char nm[64];
    run4("tmag<4,24>", tmag<4, 24>, 2048 + 4 * CHB, G, L, A, C, Q, n, ctr, 0);
    run4("tmag<4,24> smem220K", tmag<4, 24>, 220 * 1024, G, L, A, C, Q, n, ctr, 0);
    run4("tmag<4,24> wait12", tmag<4, 24>, 2048 + 4 * CHB, G, L, A, C, Q, n, ctr, 112000);
    run4("tmag<4,24> smem220K wait12", tmag<4, 24>, 220 * 1024, G, L, A, C, Q, n, ctr, 112000);
    run4("tmag<3,24> smem220K", tmag<3, 24>, 220 * 1024, G, L, A, C, Q, n, ctr, 0);
    return 0;
}
