// common.cuh — device helpers shared by the libewsjf kernels (sm_100a only).
//
// Keys, the Eq. 4 score, TMA bulk-copy / mbarrier wrappers and warp
// reductions.  Nothing here is shared with oracle/ (the CPU oracle has its own
// arithmetic); see DESIGN.md §5 for the kernel map.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "ewsjf.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libewsjf targets sm_100a (B200) only"
#endif

// Every device / pinned allocation and free of the library goes through these
// counters (ewsjf_alloc_count): the tests check that no hot call allocates.
extern "C" void ewsjf_count_alloc_(void);
static inline cudaError_t ewsjf_counted_malloc_(void** p, size_t n) { ewsjf_count_alloc_(); return cudaMalloc(p, n); }
static inline cudaError_t ewsjf_counted_malloc_host_(void** p, size_t n) { ewsjf_count_alloc_(); return cudaMallocHost(p, n); }
static inline cudaError_t ewsjf_counted_free_(void* p) { ewsjf_count_alloc_(); return cudaFree(p); }
#define cudaMalloc(p, n) ewsjf_counted_malloc_((void**)(p), (n))
#define cudaMallocHost(p, n) ewsjf_counted_malloc_host_((void**)(p), (n))
#define cudaFree(p) ewsjf_counted_free_((void*)(p))

// Device bounds checks of the bounds-checked build (EWSJF_CHECKED=1 builds
// libewsjf_check.so with -DEWSJF_BOUNDS_CHECK; compute-sanitizer is not available on
// the GPU pool): a failed check prints its site and traps (the call returns
// EWSJF_ERR_CUDA).  Compiled out of libewsjf.so.
#ifdef EWSJF_BOUNDS_CHECK
#include <cstdio>
#define EWSJF_CHECK(c)                                                                        \
    do {                                                                                      \
        if (!(c)) {                                                                           \
            printf("EWSJF_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,    \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                                    \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define EWSJF_CHECK(c) do { } while (0)
#endif

namespace ewsjf {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int kMaxSlots = EWSJF_MAX_QUEUES;   // 256
constexpr int kThreads = 512;                 // persistent tick CTA
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 2048;                   // requests per pipeline stage (4 per thread)
constexpr int kStages = 3;
constexpr int kLutCap = 32784;                // bytes of the length->slot LUT (lengths < 32784)
constexpr uint32_t kGapSlot = 0x1000u;        // slot code: gap-falling length (> any position)
constexpr unsigned char kLutGap = 0xFE;       // LUT byte for a gap (LUT used only when nslots <= 250)
constexpr uint32_t kBadSlot = 0xFFFFu;        // invalid (len < 1 / unknown qid)

// ---------------------------------------------------------------- policy ---
// Per-queue tables of the active policy (partition + weights), passed by value
// as a __grid_constant__ kernel parameter (≈6 KB).  Index = queue position.
struct Policy {
    int32_t nslots;
    int32_t pad[3];                // every table 16-byte aligned (the fused tick stages them with cp.async)
    int32_t min_len[kMaxSlots];
    int32_t max_len[kMaxSlots];
    int32_t sid[kMaxSlots];        // stable id
    float wb[kMaxSlots];           // w_base
    float wu[kMaxSlots];           // w_urg
    float wf[kMaxSlots];           // w_fair * ln 2  (the score uses log2)
};

// Score inputs shared by all kernels.
struct ScoreParams {
    float now, c0, c1, c2;
    int32_t mode;                  // EWSJF_SELECT_SCORE / FIFO
    int32_t k;
};

// ---------------------------------------------------------------- keys -----
// SCORE key: hi = bits(s') (s' >= +0 so the IEEE bits are monotone), lo = ~id:
// larger key = better, ties -> lower id (R24).  FIFO key: hi = ~ord(arrival),
// lo = ~id: larger = earlier arrival, ties -> lower id (R26).  0 = empty.
__device__ __forceinline__ u32 ord_f32(float f) {
    u32 u = __float_as_uint(f);
    u = (u == 0x80000000u) ? 0u : u;           // -0 -> +0 (integer ops: exact under -ftz)
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ u64 score_key(float sp, u32 gid) {
    return ((u64)__float_as_uint(sp) << 32) | (u64)(~gid);
}
__device__ __forceinline__ u64 fifo_key(float arrival, u32 gid) {
    return ((u64)(~ord_f32(arrival)) << 32) | (u64)(~gid);
}
__device__ __forceinline__ u32 key_gid(u64 k) { return ~(u32)(k & 0xffffffffull); }
__device__ __forceinline__ float key_sp(u64 k) { return __uint_as_float((u32)(k >> 32)); }

// ------------------------------------------------------------- Eq. 4 -------
// s' = (w_base + w_urg W/C + w_fair ln(b+1)) / (b+1), so Φ = q_i · s' (Eq. 4,
// P:335-343; qf = q_i/(b+1) P:348; cs = W/C P:347).  Evaluated as
//   s' = ((w_base + w_fair' log2(b+1)) C + w_urg W) / ((b+1) C)
// with w_fair' = w_fair ln 2: one MUFU.LG2 + one MUFU.RCP per request.
// Returns false (excluded) when W < 0, C <= 0 or NaN (R5).
__device__ __forceinline__ bool score_sp(int b, float arrival, float cost, bool has_cost,
                                         const ScoreParams& P, float wb, float wu, float wf,
                                         float* sp) {
    float W = P.now - arrival;
    float bf = (float)b;
    float C = has_cost ? cost : fmaf(fmaf(P.c2, bf, P.c1), bf, P.c0);
    float b1 = bf + 1.0f;
    float lg = __log2f(b1);
    float num = fmaf(fmaf(wf, lg, wb), C, wu * W);
    *sp = __fdividef(num, b1 * C);
    return (W >= 0.0f) && (C > 0.0f);
}

// ------------------------------------------------------ TMA + mbarrier -----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(addr), "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).  SASS: UBLKCP.S.G.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// --------------------------------------------------------------- warps -----
__device__ __forceinline__ u64 shfl_xor_u64(u64 v, int m) {
    u32 lo = __shfl_xor_sync(0xffffffffu, (u32)v, m);
    u32 hi = __shfl_xor_sync(0xffffffffu, (u32)(v >> 32), m);
    return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ u64 shfl_idx_u64(u64 v, int src) {
    const u32 lo = __shfl_sync(0xffffffffu, (u32)v, src);
    const u32 hi = __shfl_sync(0xffffffffu, (u32)(v >> 32), src);
    return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ u64 shfl_up_u64(u64 v, int d) {
    const u32 lo = __shfl_up_sync(0xffffffffu, (u32)v, d);
    const u32 hi = __shfl_up_sync(0xffffffffu, (u32)(v >> 32), d);
    return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ u64 warp_max_u64(u64 v) {
#pragma unroll
    for (int m = 16; m; m >>= 1) {
        u64 o = shfl_xor_u64(v, m);
        v = o > v ? o : v;
    }
    return v;
}
__device__ __forceinline__ u64 warp_min_u64(u64 v) {
#pragma unroll
    for (int m = 16; m; m >>= 1) {
        u64 o = shfl_xor_u64(v, m);
        v = o < v ? o : v;
    }
    return v;
}

}  // namespace ewsjf
