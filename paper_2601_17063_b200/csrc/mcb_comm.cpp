// The context's NCCL communicator ("a device context per GPU
// set owns the NCCL communicator"): the single collective of the sharded
// engine -- one in-place sum of the int64 counter / latency-bit buffer in
// which every slot is written by exactly one rank (distributed.py) -- for
// callers that are not Python.  NCCL is opened at run time (dlopen of
// libnccl.so.2, RTLD_LOCAL), so libmcb.so has no link-time dependency on it
// and does not collide with another NCCL already loaded in the process (e.g.
// torch's); without NCCL these entry points fail with MCB_ERR_UNSUPPORTED.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>

#include <cstring>
#include <mutex>

#include "mcb_internal.h"

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy;
    });
    return api;
}

int nccl_error(ncclResult_t r) {
    const char *m = nccl().error_string ? nccl().error_string(r) : "NCCL error";
    return mcb_set_error(MCB_ERR_CUDA, m);
}

}  // namespace

// (mcb_api.cu) the context's communicator slot and device
ncclComm_t *mcb_ctx_comm(mcb_ctx *ctx);
int mcb_ctx_device(mcb_ctx *ctx);

extern "C" int mcb_comm_unique_id(uint8_t *out, int32_t n) {
    mcb_clear_error();
    if (!out || n < NCCL_UNIQUE_ID_BYTES) return mcb_set_error(MCB_ERR_INVALID, "need a 128-byte buffer");
    if (!nccl().ok) return mcb_set_error(MCB_ERR_UNSUPPORTED, "libnccl.so.2 is not available");
    ncclUniqueId id;
    if (ncclResult_t r = nccl().get_unique_id(&id)) return nccl_error(r);
    memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return MCB_OK;
}

extern "C" int mcb_comm_init(mcb_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t *unique_id) {
    mcb_clear_error();
    if (!ctx || !unique_id) return mcb_set_error(MCB_ERR_INVALID, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return mcb_set_error(MCB_ERR_INVALID, "need 0 <= rank < nranks");
    if (!nccl().ok) return mcb_set_error(MCB_ERR_UNSUPPORTED, "libnccl.so.2 is not available");
    ncclComm_t *slot = mcb_ctx_comm(ctx);
    if (*slot) return mcb_set_error(MCB_ERR_INVALID, "the context already owns a communicator");
    if (cudaSetDevice(mcb_ctx_device(ctx)) != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, "cudaSetDevice");
    ncclUniqueId id;
    memcpy(id.internal, unique_id, NCCL_UNIQUE_ID_BYTES);
    if (ncclResult_t r = nccl().comm_init_rank(slot, nranks, id, rank)) {
        *slot = nullptr;
        return nccl_error(r);
    }
    return MCB_OK;
}

extern "C" int mcb_comm_allreduce_i64(mcb_ctx *ctx, int64_t *buf, int64_t count, void *stream) {
    mcb_clear_error();
    if (!ctx || (!buf && count > 0)) return mcb_set_error(MCB_ERR_INVALID, "NULL argument");
    ncclComm_t comm = *mcb_ctx_comm(ctx);
    if (!comm) return mcb_set_error(MCB_ERR_INVALID, "the context has no communicator (mcb_comm_init)");
    if (count == 0) return MCB_OK;
    if (ncclResult_t r = nccl().all_reduce(buf, buf, (size_t)count, ncclInt64, ncclSum, comm, (cudaStream_t)stream))
        return nccl_error(r);
    return MCB_OK;
}

int mcb_comm_release(ncclComm_t *slot) {
    if (slot && *slot && nccl().ok) nccl().comm_destroy(*slot);
    if (slot) *slot = nullptr;
    return MCB_OK;
}

extern "C" int mcb_comm_destroy(mcb_ctx *ctx) {
    mcb_clear_error();
    if (!ctx) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    return mcb_comm_release(mcb_ctx_comm(ctx));
}
