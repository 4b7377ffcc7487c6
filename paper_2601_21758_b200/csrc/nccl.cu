// nccl.cu — the NCCL communicator of a ctx (SURVEY §8b ewsjf_ctx_attach_nccl,
// §8e): the index-sharded tick all-gathers the ranks' fixed-size exchange
// records (tick_local -> ncclAllGather -> tick_merge) on the ctx stream, inside
// ewsjf_tick, so a C caller runs the multi-GPU tick with no Python in the loop
// and the three steps are capturable in one CUDA graph.
//
// NCCL is resolved at run time: dlopen("libnccl.so.2") returns the copy the
// process already loaded (PyTorch's, when torch is imported first) and falls
// back to the system library; libewsjf has no link-time NCCL dependency.
// Only the types come from <nccl.h>.
#include <dlfcn.h>
#include <mutex>
#include <nccl.h>
#include "merge.cuh"
#include "ctx.h"

namespace ewsjf {

struct NcclApi {
    bool ok = false;
    char why[256] = {0};
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

static NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            snprintf(api.why, sizeof api.why, "dlopen(libnccl.so.2) failed: %s", dlerror());
            return;
        }
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.error_string;
        if (!api.ok) snprintf(api.why, sizeof api.why, "libnccl.so.2 lacks a required symbol");
    });
    return api;
}

// Exchange buffers for the largest record this ctx can produce (256 queues x max_k).
static ewsjf_status alloc_exchange(ewsjf_ctx* ctx, int world) {
    const int64_t per = ex_layout(kMaxSlots, ctx->max_k, ctx->ex_gap).total;
    if (cudaMalloc(&ctx->ex_local, per) != cudaSuccess ||
        cudaMalloc(&ctx->ex_all, per * world) != cudaSuccess)
        return fail(ctx, EWSJF_ERR_CUDA, "exchange buffers (%lld x %d bytes)", (long long)per, world);
    ctx->ex_cap = per;
    return EWSJF_OK;
}

ewsjf_status nccl_allgather(ewsjf_ctx* ctx, int64_t bytes) {
    NcclApi& api = nccl_api();
    const ncclResult_t r = api.all_gather(ctx->ex_local, ctx->ex_all, (size_t)bytes, ncclUint8,
                                          (ncclComm_t)ctx->nccl_comm, ctx->stream);
    if (r != ncclSuccess) return fail(ctx, EWSJF_ERR_NCCL, "ncclAllGather: %s", api.error_string(r));
    return EWSJF_OK;
}

void nccl_release(ewsjf_ctx* ctx) {
    if (ctx->nccl_comm && ctx->nccl_owned && nccl_api().ok) nccl_api().comm_destroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
    if (ctx->ex_local) cudaFree(ctx->ex_local);
    if (ctx->ex_all) cudaFree(ctx->ex_all);
    ctx->ex_local = ctx->ex_all = nullptr;
}

}  // namespace ewsjf

using namespace ewsjf;

extern "C" ewsjf_status ewsjf_nccl_get_unique_id(uint8_t* id_out) {
    if (!id_out) return EWSJF_ERR_INVALID_ARG;
    NcclApi& api = nccl_api();
    if (!api.ok) return EWSJF_ERR_NCCL;
    ncclUniqueId id;
    if (api.get_unique_id(&id) != ncclSuccess) return EWSJF_ERR_NCCL;
    memcpy(id_out, id.internal, sizeof id.internal);
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_ctx_init_nccl(ewsjf_ctx* ctx, const uint8_t* id, int32_t rank, int32_t world) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (!id || world < 1 || world > 1024 || rank < 0 || rank >= world)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad NCCL rank/world");
    if (ctx->nccl_comm) return fail(ctx, EWSJF_ERR_INVALID_ARG, "ctx already has a communicator");
    NcclApi& api = nccl_api();
    if (!api.ok) return fail(ctx, EWSJF_ERR_NCCL, "%s", api.why);
    CU(cudaSetDevice(ctx->device));
    ncclUniqueId uid;
    memcpy(uid.internal, id, sizeof uid.internal);
    ncclComm_t comm = nullptr;
    const ncclResult_t r = api.comm_init_rank(&comm, world, uid, rank);
    if (r != ncclSuccess) return fail(ctx, EWSJF_ERR_NCCL, "ncclCommInitRank: %s", api.error_string(r));
    ctx->nccl_comm = comm;
    ctx->nccl_owned = true;
    ctx->nccl_rank = rank;
    ctx->nccl_world = world;
    ewsjf_status s = alloc_exchange(ctx, world);
    if (s != EWSJF_OK) nccl_release(ctx);
    return s;
}

extern "C" ewsjf_status ewsjf_ctx_attach_nccl(ewsjf_ctx* ctx, void* nccl_comm, int32_t rank, int32_t world) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (!nccl_comm || world < 1 || world > 1024 || rank < 0 || rank >= world)
        return fail(ctx, EWSJF_ERR_INVALID_ARG, "bad NCCL comm/rank/world");
    if (ctx->nccl_comm) return fail(ctx, EWSJF_ERR_INVALID_ARG, "ctx already has a communicator");
    if (!nccl_api().ok) return fail(ctx, EWSJF_ERR_NCCL, "%s", nccl_api().why);
    CU(cudaSetDevice(ctx->device));
    ctx->nccl_comm = nccl_comm;
    ctx->nccl_owned = false;
    ctx->nccl_rank = rank;
    ctx->nccl_world = world;
    ewsjf_status s = alloc_exchange(ctx, world);
    if (s != EWSJF_OK) nccl_release(ctx);
    return s;
}

extern "C" ewsjf_status ewsjf_ctx_set_exchange_gap_cap(ewsjf_ctx* ctx, int32_t gap_cap) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    if (gap_cap < 1 || gap_cap > (1 << 26)) return fail(ctx, EWSJF_ERR_INVALID_ARG, "gap_cap out of [1, 2^26]");
    CU(cudaSetDevice(ctx->device));
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->ex_gap = gap_cap;
    if (ctx->ex_local) {               // an attached communicator: its buffers follow the new record size
        cudaFree(ctx->ex_local);
        cudaFree(ctx->ex_all);
        ctx->ex_local = ctx->ex_all = nullptr;
        ctx->ex_cap = 0;
        return alloc_exchange(ctx, ctx->nccl_world);
    }
    return EWSJF_OK;
}

extern "C" ewsjf_status ewsjf_ctx_detach_nccl(ewsjf_ctx* ctx) {
    if (!ctx) return EWSJF_ERR_INVALID_ARG;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    nccl_release(ctx);
    ctx->nccl_rank = 0;
    ctx->nccl_world = 0;
    return EWSJF_OK;
}
