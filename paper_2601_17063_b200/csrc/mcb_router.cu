// K1 placeholder: the tcgen05/TMA router GEMM lands in a later milestone.
#include "mcb_internal.h"

extern "C" int mcb_router_topk(mcb_ctx *, const void *, const void *, int64_t, int32_t, int32_t, int32_t,
                               int32_t, uint8_t *, float *, void *) {
    return mcb_set_error(MCB_ERR_UNSUPPORTED, "router top-k generator not built yet");
}
