// C ABI of libmcb.so (include/mcb.h): context, scratch, orchestration of the
// K2 -> K3 -> K4 -> K5 pipeline, and the host-buffer entry point.
//
// mcb_replay mirrors engine.sweep (pkg/src/moecache/engine.py:439-465) over
// the policies x capacities cross product for every trace of a packed batch;
// the per-cell arithmetic is engine.run_simulation (engine.py:300-380).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "mcb_internal.h"

#define MCB_MAX_UPLOAD_PIECES 16
#include "mcb_kernels.cuh"

// ---------------------------------------------------------------- errors ---
static thread_local std::string g_err;

int mcb_set_error(int code, const char *msg) {
    g_err = msg ? msg : "";
    return code;
}
void mcb_clear_error() { g_err.clear(); }

extern "C" int mcb_last_error(char *buf, size_t n) {
    if (!buf || n == 0) return (int)g_err.size();
    const size_t k = g_err.size() < n - 1 ? g_err.size() : n - 1;
    memcpy(buf, g_err.data(), k);
    buf[k] = 0;
    return (int)g_err.size();
}

extern "C" int mcb_abi_version(void) { return MCB_ABI_VERSION; }

#define CUDA_TRY(expr)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            char b_[256];                                                                          \
            snprintf(b_, sizeof b_, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, \
                     __LINE__, cudaGetErrorString(e_));                                            \
            return mcb_set_error(MCB_ERR_CUDA, b_);                                                \
        }                                                                                          \
    } while (0)

// ---------------------------------------------------------------- context --
int mcb_router_preload();   // mcb_router.cu
struct DevBuf {
    void *p = nullptr;
    size_t n = 0;
    int ensure(size_t bytes) {
        if (bytes <= n) return MCB_OK;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        const size_t want = bytes + bytes / 8 + 256;
        if (cudaMalloc(&p, want) != cudaSuccess) {
            cudaGetLastError();
            return mcb_set_error(MCB_ERR_NOMEM, "device scratch allocation failed");
        }
        n = want;
        return MCB_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

#define MCB_MAX_ML_CHUNKS 8

#include <nccl.h>

int mcb_comm_release(ncclComm_t *slot);   // mcb_comm.cpp

struct mcb_ctx {
    ncclComm_t comm = nullptr;         // sharded engine's communicator (mcb_comm_init), owned
    int device = 0;
    std::mutex mu;
    DevBuf next_pos, ranks[2], inst_out, inst_lat, wt, snaps, tile_off, stats, pol_caps;
    // host path staging
    DevBuf h_acc, h_acc_off, h_ev_off, h_rt_off, h_ev_info, h_routed, h_params, h_reports, h_latency,
        h_chain_reports, h_hashes, h_outcomes, h_chain_latency;
    cudaStream_t stream = nullptr;
    int64_t last_kernels = 0;
    int64_t last_uncertain = 0;
    bool timing = false;
    cudaStream_t side = nullptr;       // non-ML replay runs here concurrently with K3
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaStream_t side2 = nullptr;      // ML replay chunks, pipelined behind the K3 chunks; the ML replay after K3
    cudaStream_t side_lo = nullptr;    // the non-ML replay after K3 (least priority: the ML replay's blocks go first)
    cudaEvent_t join_lo = nullptr;
    cudaEvent_t chunk_ev[MCB_MAX_ML_CHUNKS] = {};
    cudaEvent_t join2 = nullptr;
    cudaEvent_t pre = nullptr;         // the side stream's replay preparation is done
    cudaEvent_t nets_ev = nullptr;     // host path: the nets' upload (on side2) is done
    // host path, uniform batches: the trace arrives in trace-range pieces on
    // copy_stream (up_ev[k] = piece k landed) and the trace-only stages (K2,
    // snapshots, K3) of piece k start as soon as it is there
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t up_ev[MCB_MAX_UPLOAD_PIECES] = {};
    int n_pieces = 0;                  // > 0 only inside one mcb_replay_host call
    int64_t piece_chain[MCB_MAX_UPLOAD_PIECES + 1] = {};
    int64_t upload_pieces = 8;         // MCB_TUNE_UPLOAD_PIECES
    bool pieces_next = false;          // the pieced K3 loop also runs K2 per piece
    std::function<int()> before_rescore;   // replay_locked: start the non-ML replay under the re-score
    size_t pieces_nu_sw = 0;
    bool nets_pending = false;         // the scorer must wait for nets_ev before using the nets
    int64_t ml_chunks = 1;             // K3 / ML replay pipeline depth (MCB_TUNE_ML_CHUNKS)
    int k3_ctas = -1;                  // K3 grid mode (MCB_TUNE_K3_CTAS)
    int overlap = 0;                   // non-ML replay: 0 after K3 (next to the ML replay), 1 during K3
    int64_t solo_min_instances = 0;   // thread-per-instance whenever E <= 16 (MCB_SOLO_MIN overrides)
    int64_t wide_min_instances = 8192;    // thread-per-instance for 16 < E <= 128 from this many (MCB_WIDE_MIN)
    int64_t seg_ev = 0;               // segmented replay: 0 auto, <0 off, >0 events per segment (MCB_SEG_EV)
    int64_t seg_nw = 0;               // warm-up events before each segment: 0 auto (MCB_SEG_NW)
    int64_t seg_passes = 0;           // speculation passes (MCB_SEG_PASSES): 0 auto, 1 or 2
    int seg_tspec = 0;                // E > 16 speculation: 0 auto, 1 thread, -1 warp (MCB_SEG_TSPEC)
    int64_t group_lanes = 0;          // lanes per instance of the E > 16 replay: 0 auto, 8 / 16 / 32
    int64_t scratch_bytes = 0;        // per-call scratch budget (MCB_TUNE_SCRATCH_BYTES): 0 = 40% of free
    int64_t fit_need = 0;             // largest scratch estimate replayed in one range (its buffers are held)
    int64_t mem_total = 0;            // device memory (cudaDeviceProp::totalGlobalMem)
    int64_t last_chunks = 1;          // trace ranges of the last mcb_replay
    bool serial = false;              // one stream for every stage (per-stage attribution timing)
    DevBuf seg_snap, seg_summ, seg_out, seg_codes, nu_scratch;
    DevBuf tc_wimg, tc_bias, tc_flag_cnt, tc_flag_list;   // K3-TC scratch
    int k3_tc = 1;                    // tensor-core scorer when eligible (MCB_TUNE_K3_TC)
    int64_t k3_tau_ppb = 4000;        // its certification threshold tau in 1e-9 (MCB_TUNE_K3_TAU_PPB)
    int k3_groups = 3;                // its epilogue groups for E <= 64 (MCB_TUNE_K3_GROUPS)
    // LeCaR (mcb_set_lecar): parameters, the shared random() stream (cached
    // per seed, grown on demand) and the per-call regret factor table
    double lecar_lr = 0.45, lecar_base = 0.005;
    int64_t lecar_seed = 0, lecar_u_seed = -1, lecar_u_n = 0;
    DevBuf lecar_u, lecar_f;
    DevBuf diag;                       // K8 duel tables
    DevBuf train_ws[2];                // K10 training / evaluation workspaces
    cublasHandle_t cublas = nullptr;   // K10 batched DGEMMs
    std::vector<double> lecar_host;
    cudaEvent_t ev[10] = {};          // start/stop per stage: K2, K3, K4 non-ML, K4 ML, K5
    nvtxRangeId_t nvtx[5] = {};       // open NVTX range per stage
    bool ran[5] = {};
};

// Stage boundaries: CUDA events for mcb_last_timings (when timing is on) and
// NVTX ranges around the enqueue of each stage (K2 next-use, K3 scorer, K4
// non-ML / ML replay, K5 fold) for Nsight timelines; NVTX calls are no-ops
// unless a tool is attached.
static const char *const kStageNames[5] = {"mcb K2 next-use scan", "mcb K3 scorer", "mcb K4 replay (non-ML)",
                                          "mcb K4 replay (ML)", "mcb K5 fold"};
static void mark(mcb_ctx *c, int i, cudaStream_t s) {
    if (c->timing) cudaEventRecord(c->ev[i], s);
    if (i % 2 == 0) c->nvtx[i / 2] = nvtxRangeStartA(kStageNames[i / 2]);
    else nvtxRangeEnd(c->nvtx[i / 2]);
}
static const int N_STAGES = 5;

extern "C" int mcb_set_timing(mcb_ctx *c, int32_t enable) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    CUDA_TRY(cudaSetDevice(c->device));
    if (enable && !c->ev[0])
        for (auto &e : c->ev) CUDA_TRY(cudaEventCreate(&e));
    c->timing = enable != 0;
    return MCB_OK;
}

extern "C" int mcb_set_lecar(mcb_ctx *c, double learning_rate, double discount_base, int64_t seed) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (!(discount_base >= 0.0))
        return mcb_set_error(MCB_ERR_UNSUPPORTED, "LeCaR discount_base must be >= 0");
    std::lock_guard<std::mutex> lk(c->mu);
    c->lecar_lr = learning_rate;
    c->lecar_base = discount_base;
    c->lecar_seed = seed < 0 ? -seed : seed;   // random.seed(int) uses abs(n)
    return MCB_OK;
}

// LeCaR inputs for one call: the random() stream (at least one draw per
// access of the longest chain) and the regret factors of these capacities.
static int lecar_prepare(mcb_ctx *c, const DevTrace &d, const int32_t *caps, int n_cap, ReplayParams &P,
                         cudaStream_t s) {
    int64_t maxlen = 0;
    if (d.uniform) {
        maxlen = d.T * d.K;
    } else {
        std::vector<int64_t> off((size_t)d.n_chains + 1);
        CUDA_TRY(cudaMemcpyAsync(off.data(), d.acc_off, off.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (int64_t i = 0; i < d.n_chains; ++i) maxlen = std::max(maxlen, off[i + 1] - off[i]);
    }
    maxlen = std::max<int64_t>(maxlen, 1);
    if (c->lecar_u_seed != c->lecar_seed || c->lecar_u_n < maxlen) {
        const int64_t n = std::max(maxlen, c->lecar_u_seed == c->lecar_seed ? 2 * c->lecar_u_n : 0);
        c->lecar_host.resize((size_t)n);
        mcb_lecar_stream(c->lecar_seed, n, c->lecar_host.data());
        if (int rc = c->lecar_u.ensure((size_t)n * sizeof(double))) return rc;
        CUDA_TRY(cudaMemcpyAsync(c->lecar_u.p, c->lecar_host.data(), (size_t)n * sizeof(double),
                                 cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        c->lecar_u_seed = c->lecar_seed;
        c->lecar_u_n = n;
    }
    const int64_t tlen = mcb_lecar_factor_len(caps, n_cap, c->lecar_lr, c->lecar_base, maxlen);
    std::vector<double> f((size_t)(n_cap * tlen));
    mcb_lecar_factors(caps, n_cap, c->lecar_lr, c->lecar_base, tlen, f.data());
    if (int rc = c->lecar_f.ensure(f.size() * sizeof(double))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->lecar_f.p, f.data(), f.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    P.lecar_u = (const double *)c->lecar_u.p;
    P.lecar_f = (const double *)c->lecar_f.p;
    P.lecar_tlen = tlen;
    return MCB_OK;
}

extern "C" int mcb_set_tuning(mcb_ctx *c, int32_t knob, int64_t value) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    if (knob == MCB_TUNE_SOLO_MIN) {
        c->solo_min_instances = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_SEG_EV) {
        c->seg_ev = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_SEG_NW) {
        c->seg_nw = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_SERIAL) {
        c->serial = value != 0;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_SEG_TSPEC) {
        c->seg_tspec = (int)value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_WIDE_MIN) {
        c->wide_min_instances = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_OVERLAP) {
        c->overlap = (int)value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_K3_TC) {
        c->k3_tc = value != 0;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_K3_TAU_PPB) {
        if (value < 0) return mcb_set_error(MCB_ERR_INVALID, "tau must be >= 0");
        c->k3_tau_ppb = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_UPLOAD_PIECES) {
        if (value < 0 || value > MCB_MAX_UPLOAD_PIECES)
            return mcb_set_error(MCB_ERR_INVALID, "upload pieces must be 0 .. 16");
        c->upload_pieces = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_K3_GROUPS) {
        if (value < 1 || value > 3) return mcb_set_error(MCB_ERR_INVALID, "K3 variant must be 1, 2 or 3");
        c->k3_groups = (int)value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_SCRATCH_BYTES) {
        if (value < 0) return mcb_set_error(MCB_ERR_INVALID, "scratch budget must be >= 0");
        c->scratch_bytes = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_ML_CHUNKS) {
        c->ml_chunks = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_K3_CTAS) {
        c->k3_ctas = (int)value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_GROUP_LANES) {
        if (value != 0 && value != 8 && value != 16 && value != 32)
            return mcb_set_error(MCB_ERR_INVALID, "lane group must be 0, 8, 16 or 32");
        c->group_lanes = value;
        return MCB_OK;
    }
    if (knob == MCB_TUNE_SEG_PASSES) {
        if (value < 0 || value > 8) return mcb_set_error(MCB_ERR_INVALID, "speculation passes must be 0 (auto) .. 8");
        c->seg_passes = value;
        return MCB_OK;
    }
    return mcb_set_error(MCB_ERR_INVALID, "unknown tuning knob");
}

extern "C" int mcb_last_timings(mcb_ctx *c, float *ms, int32_t n) {
    mcb_clear_error();
    if (!c || !ms) return mcb_set_error(MCB_ERR_INVALID, "ctx / ms is NULL");
    if (!c->timing) return mcb_set_error(MCB_ERR_INVALID, "timing is not enabled");
    for (int i = 0; i < n && i < N_STAGES; ++i) {
        ms[i] = 0.f;
        if (c->ran[i]) CUDA_TRY(cudaEventElapsedTime(&ms[i], c->ev[2 * i], c->ev[2 * i + 1]));
    }
    return MCB_OK;
}

extern "C" int mcb_ctx_create(int device, mcb_ctx **out) {
    mcb_clear_error();
    if (!out) return mcb_set_error(MCB_ERR_INVALID, "out is NULL");
    int n = 0;
    CUDA_TRY(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return mcb_set_error(MCB_ERR_INVALID, "no such CUDA device");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return mcb_set_error(MCB_ERR_UNSUPPORTED, "libmcb is built for sm_100a (B200); device is older");
    if (preload_kernels() != 0 || preload_segment_kernels() != 0 || preload_segment_warp_kernels() != 0 ||
        preload_wide_kernels() != 0 || preload_score_tc() != 0)
        return mcb_set_error(MCB_ERR_CUDA, "failed to load the replay kernels");
    if (int rc = mcb_router_preload()) return rc;
    auto *c = new (std::nothrow) mcb_ctx();
    if (!c) return mcb_set_error(MCB_ERR_NOMEM, "out of host memory");
    c->device = device;
    c->mem_total = (int64_t)prop.totalGlobalMem;
    if (const char *env = getenv("MCB_SOLO_MIN")) c->solo_min_instances = atoll(env);
    if (const char *env = getenv("MCB_WIDE_MIN")) c->wide_min_instances = atoll(env);
    if (const char *env = getenv("MCB_SEG_EV")) c->seg_ev = atoll(env);
    if (const char *env = getenv("MCB_SEG_NW")) c->seg_nw = atoll(env);
    if (const char *env = getenv("MCB_SEG_PASSES")) c->seg_passes = atoll(env);
    if (const char *env = getenv("MCB_SEG_TSPEC")) c->seg_tspec = atoi(env);
    if (const char *env = getenv("MCB_GROUP_LANES")) c->group_lanes = atoll(env);
    if (const char *env = getenv("MCB_K3_CTAS")) c->k3_ctas = atoi(env);
    if (const char *env = getenv("MCB_ML_CHUNKS")) c->ml_chunks = atoll(env);
    if (const char *env = getenv("MCB_OVERLAP")) c->overlap = atoi(env);
    if (const char *env = getenv("MCB_SCRATCH_BYTES")) c->scratch_bytes = atoll(env);
    if (const char *env = getenv("MCB_K3_TC")) c->k3_tc = atoi(env);
    if (const char *env = getenv("MCB_K3_TAU_PPB")) c->k3_tau_ppb = atoll(env);
    if (const char *env = getenv("MCB_UPLOAD_PIECES"))
        c->upload_pieces = std::max<int64_t>(0, std::min<int64_t>(MCB_MAX_UPLOAD_PIECES, atoll(env)));
    if (const char *env = getenv("MCB_K3_GROUPS")) c->k3_groups = std::max(1, std::min(3, atoi(env)));
    for (auto &e : c->up_ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            delete c;
            return mcb_set_error(MCB_ERR_CUDA, "event creation failed");
        }
    for (auto &e : c->chunk_ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            delete c;
            return mcb_set_error(MCB_ERR_CUDA, "event creation failed");
        }
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);   // replay warps dispatch ahead of K3 blocks
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->side2, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->side_lo, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->join_lo, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->join2, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->pre, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->nets_ev, cudaEventDisableTiming) != cudaSuccess ||

        cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return mcb_set_error(MCB_ERR_CUDA, "stream creation failed");
    }

    *out = c;
    return MCB_OK;
}

ncclComm_t *mcb_ctx_comm(mcb_ctx *c) { return &c->comm; }
int mcb_ctx_device(mcb_ctx *c) { return c->device; }

extern "C" int mcb_ctx_destroy(mcb_ctx *c) {
    if (!c) return MCB_OK;
    cudaSetDevice(c->device);
    mcb_comm_release(&c->comm);
    DevBuf *all[] = {&c->next_pos, &c->ranks[0], &c->ranks[1], &c->inst_out, &c->inst_lat, &c->wt, &c->snaps,
                     &c->tile_off, &c->stats, &c->pol_caps, &c->h_acc, &c->h_acc_off, &c->h_ev_off,
                     &c->h_rt_off, &c->h_ev_info, &c->h_routed, &c->h_params, &c->h_reports, &c->h_latency,
                     &c->h_chain_reports, &c->h_hashes, &c->h_outcomes, &c->h_chain_latency, &c->seg_snap,
                     &c->seg_summ, &c->tc_wimg, &c->tc_bias, &c->tc_flag_cnt, &c->tc_flag_list,
                     &c->seg_out, &c->seg_codes, &c->nu_scratch, &c->lecar_u, &c->lecar_f, &c->diag,
                     &c->train_ws[0], &c->train_ws[1]};
    for (DevBuf *b : all) b->release();
    if (c->cublas) cublasDestroy(c->cublas);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->side2) cudaStreamDestroy(c->side2);
    if (c->side_lo) cudaStreamDestroy(c->side_lo);
    if (c->join_lo) cudaEventDestroy(c->join_lo);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (auto &e : c->up_ev)
        if (e) cudaEventDestroy(e);
    if (c->join2) cudaEventDestroy(c->join2);
    if (c->pre) cudaEventDestroy(c->pre);
    if (c->nets_ev) cudaEventDestroy(c->nets_ev);
    for (auto &e : c->chunk_ev)
        if (e) cudaEventDestroy(e);

    if (c->fork) cudaEventDestroy(c->fork);
    if (c->join) cudaEventDestroy(c->join);
    for (auto &e : c->ev)
        if (e) cudaEventDestroy(e);
    delete c;
    return MCB_OK;
}

extern "C" int mcb_read_stats(mcb_ctx *c, int64_t *out, int32_t n) {
    mcb_clear_error();
    if (!c || !out) return mcb_set_error(MCB_ERR_INVALID, "ctx / out is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    CUDA_TRY(cudaSetDevice(c->device));
    if (int rc = c->stats.ensure(64)) return rc;
    unsigned long long v[8];
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(v, c->stats.p, sizeof v, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n && i < 8; ++i) out[i] = (int64_t)v[i];
    return MCB_OK;
}

extern "C" int mcb_last_chunks(mcb_ctx *c, int64_t *chunks) {
    if (!c || !chunks) return mcb_set_error(MCB_ERR_INVALID, "ctx / chunks is NULL");
    *chunks = c->last_chunks;
    return MCB_OK;
}

extern "C" int mcb_last_stats(mcb_ctx *c, int64_t *kernels, int64_t *uncertain) {
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (kernels) *kernels = c->last_kernels;
    if (uncertain) *uncertain = c->last_uncertain;
    return MCB_OK;
}

// ------------------------------------------------------------ validation --
static int check_trace(const mcb_trace *t) {
    if (!t) return mcb_set_error(MCB_ERR_INVALID, "trace is NULL");
    if (t->num_layers < 1 || t->num_experts < 1 || t->top_k < 1 || t->top_k > t->num_experts ||
        t->num_traces < 0)
        return mcb_set_error(MCB_ERR_INVALID, "invalid trace header");
    if (t->num_experts > MCB_MAX_EXPERTS)
        return mcb_set_error(MCB_ERR_UNSUPPORTED, "num_experts > 128 is not supported by the B200 engine");
    if (!t->acc) return mcb_set_error(MCB_ERR_INVALID, "trace.acc is NULL");
    if (!t->uniform && (!t->chain_acc_off || !t->chain_ev_off || !t->chain_rt_off || !t->ev_info || !t->routed))
        return mcb_set_error(MCB_ERR_INVALID, "general-mode trace needs chain offsets, ev_info and routed");
    if (t->uniform && t->events_per_chain < 0) return mcb_set_error(MCB_ERR_INVALID, "events_per_chain < 0");
    return MCB_OK;
}

static DevTrace make_dev_trace(const mcb_trace *t) {
    DevTrace d;
    d.L = t->num_layers;
    d.E = t->num_experts;
    d.K = t->top_k;
    d.uniform = t->uniform;
    d.T = t->events_per_chain;
    d.n_chains = (int64_t)t->num_layers * t->num_traces;
    d.total_acc = t->uniform ? d.n_chains * d.T * d.K : t->total_acc;
    d.total_events = t->uniform ? d.n_chains * d.T : t->total_events;
    d.acc = t->acc;
    d.acc_off = t->chain_acc_off;
    d.ev_off = t->chain_ev_off;
    d.rt_off = t->chain_rt_off;
    d.ev_info = t->ev_info;
    d.routed = t->routed;
    return d;
}

// A uniform trace's chains [lo, hi) as a trace of their own (chain-major
// layout: every per-chain output is offset by lo times its per-chain size)
static DevTrace sub_trace(const DevTrace &d, int64_t lo, int64_t hi) {
    DevTrace s = d;
    s.acc = d.acc + lo * d.T * d.K;
    s.n_chains = hi - lo;
    s.total_acc = s.n_chains * d.T * d.K;
    s.total_events = s.n_chains * d.T;
    return s;
}

static int64_t max_score_tiles(const DevTrace &d) {
    if (d.uniform) return d.n_chains * ((d.T + MCB_TILE_EV - 1) / MCB_TILE_EV);
    return d.total_events / MCB_TILE_EV + d.n_chains;  // upper bound of sum(ceil(n_c / TILE))
}

// All device allocations of K3 happen here, before anything is launched.
static int ensure_score_buffers(mcb_ctx *c, const DevTrace &d, const mcb_nets *nets) {
    const int E = d.E, H = nets->hidden;
    const size_t per = prepared_net_doubles(E, H);
    if (int rc = c->wt.ensure(per * nets->num_nets * sizeof(double))) return rc;
    const int64_t tiles = max_score_tiles(d);
    if (int rc = c->snaps.ensure((size_t)(tiles + 1) * (4 * E + 8) * sizeof(int32_t))) return rc;
    if (int rc = c->tile_off.ensure((size_t)(d.n_chains + 1) * sizeof(int64_t))) return rc;
    return MCB_OK;
}

static int check_nets(const DevTrace &d, const mcb_nets *nets) {
    const int H = nets->hidden;
    if (nets->num_experts != d.E) return mcb_set_error(MCB_ERR_SHAPE, "net num_experts does not match the trace");
    if (H < 1 || H > 256) return mcb_set_error(MCB_ERR_UNSUPPORTED, "net hidden size must be in [1, 256]");
    if (nets->num_nets != 1 && nets->num_nets != d.L)
        return mcb_set_error(MCB_ERR_INVALID, "num_nets must be 1 or num_layers");
    if (!nets->params) return mcb_set_error(MCB_ERR_INVALID, "nets.params is NULL");
    return MCB_OK;
}

static int run_score(mcb_ctx *c, const DevTrace &d, const mcb_nets *nets, int include_prefill, uint8_t *ranks,
                     double *scores, cudaStream_t s, int64_t *launched, float *tc_scores = nullptr) {
    const int E = d.E, H = nets->hidden;
    if (int rc = check_nets(d, nets)) return rc;
    if (int rc = ensure_score_buffers(c, d, nets)) return rc;
    if (c->nets_pending) CUDA_TRY(cudaStreamWaitEvent(s, c->nets_ev, 0));   // host path: nets copied on side2
    *launched += launch_prepare_nets(nets->params, E, H, nets->num_nets, (double *)c->wt.p, s);
    const int64_t tiles = max_score_tiles(d);
    if (c->k3_tc && !scores && score_tc_eligible(d, H)) {
        // K3-TC: fp16x2 tcgen05 scorer; events it cannot certify are re-scored in float64
        const int nn = nets->num_nets;
        const int64_t cap = nn == 1 ? d.total_events : d.total_events / d.L;
        if (int rc = c->tc_wimg.ensure(score_tc_net_bytes(E) * nn)) return rc;
        if (int rc = c->tc_bias.ensure((size_t)score_tc_bias_stride(E) * nn * sizeof(float))) return rc;
        if (int rc = c->tc_flag_cnt.ensure((size_t)nn * sizeof(int32_t))) return rc;
        if (int rc = c->tc_flag_list.ensure((size_t)(nn * cap + 1) * sizeof(int32_t))) return rc;
        // one pass, or one per uploaded piece (trace ranges; each waits for its
        // bytes): K2 (when the call needs it) + snapshots + the scorer per
        // piece on this stream, the float64 re-score once over all pieces
        const int np = c->n_pieces > 0 ? c->n_pieces : 1;
        const int64_t tpc32 = (d.T + MCB_TILE_EV - 1) / MCB_TILE_EV, SN = 2 * E + 4;
        for (int k = 0; k < np; ++k) {
            const int64_t lo = c->n_pieces > 0 ? c->piece_chain[k] : 0;
            const int64_t hi = c->n_pieces > 0 ? c->piece_chain[k + 1] : d.n_chains;
            const DevTrace dk = c->n_pieces > 0 ? sub_trace(d, lo, hi) : d;
            if (c->n_pieces > 0) {
                CUDA_TRY(cudaStreamWaitEvent(s, c->up_ev[k], 0));
                if (c->pieces_next)
                    *launched += launch_next_use(dk, (uint32_t *)c->next_pos.p + lo * d.T * d.K,
                                                 c->pieces_nu_sw ? (uint32_t *)c->nu_scratch.p : nullptr, s);
            }
            int32_t *snk = (int32_t *)c->snaps.p + lo * tpc32 * SN;
            *launched += launch_score_prep(dk, include_prefill, snk, (int64_t *)c->tile_off.p, max_score_tiles(dk), s);
            const int n_tc = launch_score_tc(dk, nets->params, nn, snk, (uint8_t *)c->tc_wimg.p, (float *)c->tc_bias.p,
                                             ranks + lo * d.T * E, (float)(c->k3_tau_ppb * 1e-9),
                                             (int32_t *)c->tc_flag_cnt.p, (int32_t *)c->tc_flag_list.p, cap,
                                             (unsigned long long *)c->stats.p,
                                             tc_scores ? tc_scores + lo * d.T * E : nullptr, c->k3_groups, s, k == 0,
                                             lo * d.T);
            if (n_tc < 0) return MCB_ERR_CUDA;
            *launched += n_tc;
        }
        if (c->before_rescore) {   // (the float64 re-score leaves most of the GPU to the non-ML replay)
            if (int rc = c->before_rescore()) return rc;
            c->before_rescore = nullptr;
        }
        *launched += launch_rescore(d, (const double *)c->wt.p, H, nn, (const int32_t *)c->snaps.p,
                                    (const int32_t *)c->tc_flag_cnt.p, (const int32_t *)c->tc_flag_list.p, cap, ranks,
                                    (unsigned long long *)c->stats.p, s);
        return MCB_OK;
    }
    const int n = launch_score(d, (const double *)c->wt.p, H, nets->num_nets, include_prefill, ranks, scores,
                               (int32_t *)c->snaps.p, (int64_t *)c->tile_off.p, tiles,
                               (unsigned long long *)c->stats.p, c->k3_ctas, s);
    *launched += n;
    return MCB_OK;
}

extern "C" int mcb_next_use(mcb_ctx *c, const mcb_trace *t, uint32_t *next_pos, void *stream) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (int rc = check_trace(t)) return rc;
    if (!next_pos) return mcb_set_error(MCB_ERR_INVALID, "next_pos is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    CUDA_TRY(cudaSetDevice(c->device));
    const DevTrace d = make_dev_trace(t);
    const size_t sw = next_use_scratch_words(d);
    if (sw)
        if (int rc = c->nu_scratch.ensure(sw * sizeof(uint32_t))) return rc;
    launch_next_use(d, next_pos, sw ? (uint32_t *)c->nu_scratch.p : nullptr, (cudaStream_t)stream);
    CUDA_TRY(cudaGetLastError());
    return MCB_OK;
}

extern "C" int mcb_score(mcb_ctx *c, const mcb_trace *t, const mcb_nets *nets, int32_t include_prefill,
                         uint8_t *ranks, double *scores, void *stream) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (int rc = check_trace(t)) return rc;
    if (!nets || !ranks) return mcb_set_error(MCB_ERR_INVALID, "nets / ranks is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = c->stats.ensure(64)) return rc;
    CUDA_TRY(cudaMemsetAsync(c->stats.p, 0, 64, s));
    const DevTrace d = make_dev_trace(t);
    int64_t launched = 0;
    if (int rc = run_score(c, d, nets, include_prefill, ranks, scores, s, &launched)) return rc;
    CUDA_TRY(cudaGetLastError());
    return MCB_OK;
}

extern "C" int mcb_score_tc_scores(mcb_ctx *c, const mcb_trace *t, const mcb_nets *nets, uint8_t *ranks,
                                   float *scores, void *stream) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (int rc = check_trace(t)) return rc;
    if (!nets || !ranks || !scores) return mcb_set_error(MCB_ERR_INVALID, "nets / ranks / scores is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = c->stats.ensure(64)) return rc;
    CUDA_TRY(cudaMemsetAsync(c->stats.p, 0, 64, s));
    const DevTrace d = make_dev_trace(t);
    if (!score_tc_eligible(d, nets->hidden))
        return mcb_set_error(MCB_ERR_UNSUPPORTED, "trace / net shape not eligible for the tensor-core scorer");
    const int keep = c->k3_tc;
    c->k3_tc = 1;
    int64_t launched = 0;
    const int rc = run_score(c, d, nets, 1, ranks, nullptr, s, &launched, scores);
    c->k3_tc = keep;
    if (rc) return rc;
    CUDA_TRY(cudaGetLastError());
    return MCB_OK;
}

// shared with the other translation units (mcb_diag.cu)
DevTrace mcb_dev_trace(const mcb_trace *t) { return make_dev_trace(t); }
int mcb_check_trace(const mcb_trace *t) { return check_trace(t); }
int mcb_ctx_scratch_named(mcb_ctx *c, int slot, size_t bytes, void **p) {
    std::lock_guard<std::mutex> lk(c->mu);
    if (int rc = c->train_ws[slot].ensure(bytes)) return rc;
    *p = c->train_ws[slot].p;
    return MCB_OK;
}
cublasHandle_t mcb_ctx_cublas(mcb_ctx *c) {
    std::lock_guard<std::mutex> lk(c->mu);
    if (!c->cublas && cublasCreate(&c->cublas) != CUBLAS_STATUS_SUCCESS) c->cublas = nullptr;
    return c->cublas;
}
int mcb_ctx_scratch(mcb_ctx *c, size_t bytes, void **p) {
    std::lock_guard<std::mutex> lk(c->mu);
    if (int rc = c->diag.ensure(bytes)) return rc;
    *p = c->diag.p;
    return MCB_OK;
}

static int replay_locked(mcb_ctx *c, const mcb_trace *t, const int32_t *pols, int32_t n_pol, const int32_t *caps,
                         int32_t n_cap, const mcb_cost *cost, const mcb_nets *nets, const mcb_outputs *out,
                         cudaStream_t s, bool reset_stats = true) {
    if (int rc = check_trace(t)) return rc;
    if (!pols || !caps || !cost || !out || !out->reports || !out->latency)
        return mcb_set_error(MCB_ERR_INVALID, "NULL policies / capacities / cost / outputs");
    if (n_pol < 1 || n_pol > MCB_MAX_POL) return mcb_set_error(MCB_ERR_UNSUPPORTED, "1..8 policies per call");
    if (n_cap < 1 || n_cap > MCB_MAX_CAP) return mcb_set_error(MCB_ERR_UNSUPPORTED, "1..64 capacities per call");
    // CostModel.validate (engine.py:51-55)
    if (!(cost->t_load_s > 0) || !(cost->t_compute_s > 0))
        return mcb_set_error(MCB_ERR_INVALID, "cost durations must be positive");
    if (!(cost->ml_score_cost_s >= 0)) return mcb_set_error(MCB_ERR_INVALID, "ml_score_cost_s must be >= 0");
    // capacity >= top_k (engine.py:312-316, 449-453)
    for (int i = 0; i < n_cap; ++i)
        if (caps[i] < t->top_k) {
            char b[128];
            snprintf(b, sizeof b, "capacity %d < top_k %d: a decode event cannot fit in the cache", caps[i], t->top_k);
            return mcb_set_error(MCB_ERR_CAPACITY, b);
        }
    bool need_next = false, need_lecar = false, need_ml[2] = {false, false};
    for (int i = 0; i < n_pol; ++i) {
        switch (pols[i]) {
            case MCB_LRU: case MCB_LFU: case MCB_FIFO: case MCB_ARC: break;
            case MCB_LECAR: need_lecar = true; break;
            case MCB_BELADY: need_next = true; break;
            case MCB_ML: need_ml[0] = true; break;
            case MCB_ML_NO_PREFILL: need_ml[1] = true; break;
            default: return mcb_set_error(MCB_ERR_UNSUPPORTED, "policy not supported by the B200 engine");
        }
    }
    if ((need_ml[0] || need_ml[1]) && (!nets || !nets->params))
        return mcb_set_error(MCB_ERR_INVALID, "ml policy requires trained eviction nets");

    const DevTrace d = make_dev_trace(t);
    int64_t launched = 0;
    if (int rc = c->stats.ensure(64)) return rc;
    if (reset_stats) CUDA_TRY(cudaMemsetAsync(c->stats.p, 0, 64, s));

    ReplayParams P;
    memset(&P, 0, sizeof P);
    P.tr = d;
    P.n_pol = n_pol;
    P.n_cap = n_cap;
    for (int i = 0; i < n_pol; ++i) P.pol[i] = pols[i];
    for (int i = 0; i < n_cap; ++i) P.cap[i] = caps[i];
    P.t_load = cost->t_load_s;
    P.t_compute = cost->t_compute_s;
    P.ml_cost = cost->ml_score_cost_s;
    P.loads_serial = cost->loads_serial;
    P.window = cost->window;
    P.solo_min_instances = c->solo_min_instances;
    P.wide_min_instances = c->wide_min_instances;
    P.stats = (unsigned long long *)c->stats.p;
    P.chain_lo = 0;
    P.chain_hi = d.n_chains;
    P.group_lanes = (int)c->group_lanes;
    if (need_lecar)
        if (int rc = lecar_prepare(c, d, caps, n_cap, P, s)) return rc;

    // Orchestration.  K3 (ML scores) is only needed by ML instances.  When
    // both kinds are present (default, MCB_TUNE_OVERLAP = 0) K3 runs alone
    // while the side stream prepares the replays, then the two replays --
    // both latency-bound -- run side by side:
    //     s:    +-- K3 ---------------+-- (wait pre) K4(ml) --+-- K5
    //     side: +-- K2 -- snapshot    +-- K4(lru/lfu/belady) -+
    // With MCB_TUNE_OVERLAP = 1 the non-ML replay runs under K3 instead
    // (measured slower: it competes with the scorer for issue slots).
    const int64_t n_inst = d.n_chains * n_pol * n_cap;
    if (out->chain_reports) {
        P.inst_out = out->chain_reports;
    } else {
        if (int rc = c->inst_out.ensure((size_t)(n_inst + 1) * MCB_R_N * sizeof(int64_t))) return rc;
        P.inst_out = (int64_t *)c->inst_out.p;
    }
    if (int rc = c->inst_lat.ensure((size_t)(n_inst + 1) * 2 * sizeof(double))) return rc;
    P.inst_lat = (double *)c->inst_lat.p;
    P.hashes = out->hashes;
    P.outcomes = out->outcomes;
    ReplayParams Pn = P, Pm = P;   // non-ML and ML launches
    Pn.n_pol_launch = Pm.n_pol_launch = 0;
    for (int i = 0; i < n_pol; ++i) {
        if (pols[i] == MCB_ML || pols[i] == MCB_ML_NO_PREFILL) Pm.pol_map[Pm.n_pol_launch++] = i;
        else Pn.pol_map[Pn.n_pol_launch++] = i;
    }
    const bool split = Pn.n_pol_launch > 0 && Pm.n_pol_launch > 0 && !c->serial;
    cudaStream_t sn = split ? c->side : s;
    for (bool &r : c->ran) r = false;

    // Segmented speculative replay (mcb_segment.cu) when the instances are
    // too few to fill the GPU; every buffer is sized here, before any launch.
    {
        const int64_t n_launch = d.n_chains * n_cap * (Pn.n_pol_launch > Pm.n_pol_launch ? Pn.n_pol_launch
                                                                                         : Pm.n_pol_launch);
        ReplayParams probe = P;
        probe.seg.n_seg = 2;
        const bool solo_ok = n_launch >= c->solo_min_instances;
        const bool paired = split && c->overlap == 0;   // ML and non-ML replays side by side after K3
        // E > 16: speculation by one thread per (instance, segment) for long
        // chains (segments sized like the E <= 16 replay's), else one warp
        const bool tspec = d.E > 16 && d.T * d.K < (1ll << 25) &&
                           (c->seg_tspec > 0 || (c->seg_tspec == 0 && d.T >= 65536));
        const int se = (c->seg_ev >= 0 && solo_ok && d.uniform)
                           ? seg_events_per_segment(d.T, n_launch, c->seg_ev, tspec ? 16 : d.E, paired) : 0;
        if (se > 0 && seg_eligible(probe)) {
            P.seg.SE = se;
            P.seg.n_seg = (int)((d.T + se - 1) / se);
            P.seg.NW = seg_warmup_events(se, c->seg_nw, d.E);
            P.seg.thread_spec = tspec ? 1 : 0;
            // one pass for E <= 16 (measured best on C2); two for E > 16, whose states
            // coalesce more slowly (C3 with thread speculation: 1 / 2 passes = 333 / 141
            // ms per step, the second pass removing almost all fix-up walking)
            P.seg.passes = c->seg_passes > 0 ? (int)c->seg_passes : (d.E <= 16 ? 1 : 2);
            if (d.E <= 16) P.seg.passes = std::min(P.seg.passes, 2);   // (mcb_segment.cu: two record buffers, two passes)
            P.seg.n_snap = (int)((d.T + MCB_SNAP_EV - 1) / MCB_SNAP_EV);
            P.seg.Tpad = (d.T + 15) / 16 * 16;
            P.seg.snap_e = seg_snap_stride(d.E);
            if (int rc = c->seg_snap.ensure(seg_snap_bytes(d.n_chains, P.seg.n_snap, d.E))) return rc;
            if (int rc = c->seg_summ.ensure(seg_snap_bytes(d.n_chains, P.seg.n_snap, d.E))) return rc;
            if (int rc = c->seg_out.ensure(2 * seg_out_bytes(n_inst, P.seg.n_seg, d.E))) return rc;
            if (int rc = c->seg_codes.ensure(seg_codes_bytes(n_inst, P.seg.Tpad))) return rc;
            P.seg.snap = (int2 *)c->seg_snap.p;
            P.seg.summ = (int2 *)c->seg_summ.p;
            P.seg.out[0] = (SegOut *)c->seg_out.p;
            P.seg.out[1] = (SegOut *)((char *)c->seg_out.p + seg_out_bytes(n_inst, P.seg.n_seg, d.E));
            P.seg.codes = (uint8_t *)c->seg_codes.p;
            Pn.seg = Pm.seg = P.seg;
        }
    }
    if (Pm.n_pol_launch > 0) {
        if (int rc = ensure_score_buffers(c, d, nets)) return rc;
        for (int v = 0; v < 2; ++v)
            if (need_ml[v])
                if (int rc = c->ranks[v].ensure((size_t)d.total_events * d.E + 64)) return rc;
        prepare_launch_attributes(d, nets->hidden);
    }
    const size_t nu_sw = need_next ? next_use_scratch_words(d) : 0;
    if (nu_sw)
        if (int rc = c->nu_scratch.ensure(nu_sw * sizeof(uint32_t))) return rc;
    const bool chunked = Pm.n_pol_launch > 0 && d.uniform && !c->serial && !(need_ml[0] && need_ml[1]) &&
                         std::min<int64_t>(std::min<int64_t>(c->ml_chunks, MCB_MAX_ML_CHUNKS), d.n_chains) > 1;
    const bool after_k3 = split && c->overlap == 0 && Pm.n_pol_launch > 0 && !chunked;
    // Piecewise upload (mcb_replay_host): the pieced schedule needs K3-TC on a
    // uniform trace with the replays after it; otherwise wait for the whole trace.
    if (c->n_pieces > 0) {
        const bool pieced = after_k3 && d.uniform && P.seg.n_seg <= 1 && !(need_ml[0] && need_ml[1]) && nets &&
                            c->k3_tc && score_tc_eligible(d, nets->hidden);
        if (!pieced) {
            for (int k = 0; k < c->n_pieces; ++k) CUDA_TRY(cudaStreamWaitEvent(s, c->up_ev[k], 0));
            c->n_pieces = 0;
        }
    }
    // With the replays after K3, the replays' own preparation (K2 next-use scan,
    // key snapshots) runs on the side stream under K3; the ML replay waits for it.
    cudaStream_t sp = after_k3 ? c->side : s;
    if (after_k3) {
        CUDA_TRY(cudaEventRecord(c->fork, s));
        CUDA_TRY(cudaStreamWaitEvent(c->side, c->fork, 0));
    }
    if (need_next) {
        if (int rc = c->next_pos.ensure((size_t)(d.total_acc + 64) * sizeof(uint32_t))) return rc;
        Pn.next_pos = Pm.next_pos = (const uint32_t *)c->next_pos.p;
        mark(c, 0, sp);
        if (c->n_pieces > 0) {   // piece by piece in the scorer's loop (run_score), as the trace arrives
            c->pieces_next = true;
            c->pieces_nu_sw = nu_sw;
        } else {
            launched += launch_next_use(d, (uint32_t *)c->next_pos.p, nu_sw ? (uint32_t *)c->nu_scratch.p : nullptr,
                                        sp);
        }
        mark(c, 1, sp);
        c->ran[0] = true;
    }
    if (P.seg.n_seg > 1) launched += launch_seg_snapshot(P, sp);
    if (after_k3) CUDA_TRY(cudaEventRecord(c->pre, c->side));
    for (int i = 0; i < Pn.n_pol_launch; ++i)
        if (pols[Pn.pol_map[i]] == MCB_FIFO || pols[Pn.pol_map[i]] == MCB_ARC || pols[Pn.pol_map[i]] == MCB_LECAR)
            Pn.seg.n_seg = 0;   // their eviction order depends on the cache state
    // Where the non-ML replay overlaps: during K3 (it then competes with the
    // scorer for issue slots), or after it, next to the ML replay (both are
    // latency-bound and leave most of the GPU idle).  See MCB_TUNE_OVERLAP.
    // After K3 the two replays run side by side for the rest of the step; the
    // ML replay (side2, highest priority) is the longer chain of the two, so its
    // blocks are dispatched ahead of the non-ML replay's (side_lo, least
    // priority) -- at equal priority the launch order decides, and a non-ML
    // grid queued first delayed the ML replay by up to 80 ms on C4.
    auto launch_non_ml = [&]() -> int {
        cudaStream_t sx = after_k3 ? c->side_lo : sn;
        if (split) {
            CUDA_TRY(cudaEventRecord(c->fork, s));
            CUDA_TRY(cudaStreamWaitEvent(sx, c->fork, 0));
            if (after_k3) CUDA_TRY(cudaStreamWaitEvent(sx, c->pre, 0));
        }
        if (Pn.n_pol_launch > 0) {
            mark(c, 4, sx);
            launched += seg_eligible(Pn) ? launch_replay_segmented(Pn, sx) : launch_replay(Pn, sx);
            mark(c, 5, sx);
            c->ran[2] = true;
        }
        if (after_k3) CUDA_TRY(cudaEventRecord(c->join_lo, sx));
        return MCB_OK;
    };
    if (!after_k3)
        if (int rc = launch_non_ml()) return rc;
    // K3 / ML-replay pipeline: the chains are cut into ml_chunks ranges; K3
    // scores them in order on s and the ML replay of a range starts on side2
    // as soon as its ranks are written, overlapping K3 on the next range
    // (uniform traces, one ML variant).  Off by default: measured on C2
    // (tools/chunk_sweep.sh) 1 / 2 / 4 / 8 chunks = 6.09 / 6.12 / 6.34 / 8.28 ms
    // per step -- a chunk's segmented ML replay is latency-bound (its finish
    // walk is sequential over the segments), so it costs nearly as much as
    // the whole replay and the overlap does not pay.
    const int n_chunks = (Pm.n_pol_launch > 0 && d.uniform && !c->serial && !(need_ml[0] && need_ml[1]))
                             ? (int)std::min<int64_t>(std::min<int64_t>(c->ml_chunks, MCB_MAX_ML_CHUNKS), d.n_chains)
                             : 1;
    if (Pm.n_pol_launch > 0 && n_chunks > 1) {
        const int v = need_ml[0] ? 0 : 1;
        if (int rc = check_nets(d, nets)) return rc;
        mark(c, 2, s);
        if (c->nets_pending) CUDA_TRY(cudaStreamWaitEvent(s, c->nets_ev, 0));
        launched += launch_prepare_nets(nets->params, d.E, nets->hidden, nets->num_nets, (double *)c->wt.p, s);
        const int64_t tiles = max_score_tiles(d);
        launched += launch_score_prep(d, v == 0 ? 1 : 0, (int32_t *)c->snaps.p, (int64_t *)c->tile_off.p, tiles, s);
        Pm.rank[v] = (const uint8_t *)c->ranks[v].p;
        const int64_t tpc = (d.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
        for (int k = 0; k < n_chunks; ++k) {
            const int64_t lo = d.n_chains * k / n_chunks, hi = d.n_chains * (k + 1) / n_chunks;
            launched += launch_score_tiles(d, (const double *)c->wt.p, nets->hidden, nets->num_nets, v == 0 ? 1 : 0,
                                           (uint8_t *)c->ranks[v].p, nullptr, (const int32_t *)c->snaps.p,
                                           (const int64_t *)c->tile_off.p, lo * tpc, hi * tpc,
                                           (unsigned long long *)c->stats.p, c->k3_ctas, s);
            CUDA_TRY(cudaEventRecord(c->chunk_ev[k], s));
            CUDA_TRY(cudaStreamWaitEvent(c->side2, c->chunk_ev[k], 0));
            if (k == 0) mark(c, 6, c->side2);
            ReplayParams Pk = Pm;
            Pk.chain_lo = lo;
            Pk.chain_hi = hi;
            launched += seg_eligible(Pk) ? launch_replay_segmented(Pk, c->side2) : launch_replay(Pk, c->side2);
        }
        mark(c, 3, s);
        mark(c, 7, c->side2);
        CUDA_TRY(cudaEventRecord(c->join2, c->side2));
        CUDA_TRY(cudaStreamWaitEvent(s, c->join2, 0));
        c->ran[1] = true;
        c->ran[3] = true;
    } else if (Pm.n_pol_launch > 0) {
        // The ML replay needs K3's ranks; it follows K3 on the same stream.
        // With the replays after K3, the non-ML replay starts between the
        // tensor-core scorer and its float64 re-score (run_score's hook).
        mark(c, 2, s);
        bool non_ml_started = false;
        if (after_k3)
            c->before_rescore = [&]() -> int {
                non_ml_started = true;
                return launch_non_ml();
            };
        for (int v = 0; v < 2; ++v) {
            if (!need_ml[v]) continue;
            const int rc = run_score(c, d, nets, v == 0 ? 1 : 0, (uint8_t *)c->ranks[v].p, nullptr, s, &launched);
            if (rc) {
                c->before_rescore = nullptr;
                return rc;
            }
            Pm.rank[v] = (const uint8_t *)c->ranks[v].p;
        }
        c->before_rescore = nullptr;
        mark(c, 3, s);
        cudaStream_t sm = s;
        if (after_k3) {
            if (!non_ml_started)
                if (int rc = launch_non_ml()) return rc;
            sm = c->side2;
            CUDA_TRY(cudaEventRecord(c->fork, s));
            CUDA_TRY(cudaStreamWaitEvent(sm, c->fork, 0));
            CUDA_TRY(cudaStreamWaitEvent(sm, c->pre, 0));   // key snapshots / next-use for the ML replay
        }
        mark(c, 6, sm);
        launched += seg_eligible(Pm) ? launch_replay_segmented(Pm, sm) : launch_replay(Pm, sm);
        mark(c, 7, sm);
        if (after_k3) {
            CUDA_TRY(cudaEventRecord(c->join2, sm));
            CUDA_TRY(cudaStreamWaitEvent(s, c->join2, 0));
            CUDA_TRY(cudaStreamWaitEvent(s, c->join_lo, 0));
        }
        c->ran[1] = true;
        c->ran[3] = true;
    }
    if (split) {
        CUDA_TRY(cudaEventRecord(c->join, c->side));
        CUDA_TRY(cudaStreamWaitEvent(s, c->join, 0));
    }
    mark(c, 8, s);
    launched += launch_fold(P, t->num_traces, out->reports, out->latency, s);
    if (out->chain_latency && n_inst > 0)
        CUDA_TRY(cudaMemcpyAsync(out->chain_latency, P.inst_lat, (size_t)n_inst * 2 * sizeof(double),
                                 cudaMemcpyDeviceToDevice, s));
    mark(c, 9, s);
    c->ran[4] = true;
    CUDA_TRY(cudaGetLastError());
    c->last_kernels = launched;
    return MCB_OK;
}

// Belady-labelled training data (dataset.py:35-96): features [event][2E]
// (float64), targets [event][E] (float64) and masks [event][E] (0/1 bytes)
// for every event of every chain (chain-major, mcb_trace event order); the
// reference's samples are the decode events.  Device pointers, asynchronous.
extern "C" int mcb_training_data(mcb_ctx *c, const mcb_trace *t, int32_t capacity, int32_t distance_cap,
                                 int32_t include_prefill, double *features, double *targets, uint8_t *masks,
                                 void *stream) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (int rc = check_trace(t)) return rc;
    if (capacity < t->top_k) return mcb_set_error(MCB_ERR_CAPACITY, "capacity is below top_k");
    if (distance_cap < 1) return mcb_set_error(MCB_ERR_INVALID, "distance_cap must be >= 1");
    if (!features || !targets || !masks) return mcb_set_error(MCB_ERR_INVALID, "NULL output");
    std::lock_guard<std::mutex> lk(c->mu);
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    const DevTrace d = make_dev_trace(t);
    // Belady residency at the label capacity (whole-chain replay, masks at every event start)
    const size_t nu_sw = next_use_scratch_words(d);
    if (nu_sw)
        if (int rc = c->nu_scratch.ensure(nu_sw * sizeof(uint32_t))) return rc;
    if (int rc = c->next_pos.ensure((size_t)(d.total_acc + 64) * sizeof(uint32_t))) return rc;
    if (int rc = c->inst_out.ensure((size_t)(d.n_chains + 1) * MCB_R_N * sizeof(int64_t))) return rc;
    if (int rc = c->inst_lat.ensure((size_t)(d.n_chains + 1) * 2 * sizeof(double))) return rc;
    if (int rc = c->tile_off.ensure((size_t)(d.n_chains + 1) * sizeof(int64_t))) return rc;
    const int64_t tiles = max_score_tiles(d);
    if (int rc = c->snaps.ensure((size_t)(tiles + 1) * (4 * d.E + 8) * sizeof(int32_t))) return rc;
    launch_next_use(d, (uint32_t *)c->next_pos.p, nu_sw ? (uint32_t *)c->nu_scratch.p : nullptr, s);
    ReplayParams P;
    memset(&P, 0, sizeof P);
    P.tr = d;
    P.n_pol = 1;
    P.n_cap = 1;
    P.n_pol_launch = 1;
    P.pol[0] = MCB_BELADY;
    P.cap[0] = capacity;
    P.t_load = 1.0;
    P.t_compute = 1.0;
    P.window = 5;
    P.inst_out = (int64_t *)c->inst_out.p;
    P.inst_lat = (double *)c->inst_lat.p;
    P.next_pos = (const uint32_t *)c->next_pos.p;
    P.chain_lo = 0;
    P.chain_hi = d.n_chains;
    P.res_masks = masks;
    launch_replay(P, s);
    // features and targets
    launch_score_prep(d, include_prefill ? 1 : 0, (int32_t *)c->snaps.p, (int64_t *)c->tile_off.p, tiles, s);
    launch_train_features(d, (const int32_t *)c->snaps.p, (const int64_t *)c->tile_off.p, tiles,
                          include_prefill ? 1 : 0, features, s);
    launch_train_targets(d, distance_cap, targets, s);
    CUDA_TRY(cudaGetLastError());
    return MCB_OK;
}

// Device scratch of one replay of a uniform batch, per trace: K2 next-use
// positions, the ML rank rows (one per ML variant), K3 feature snapshots,
// per-instance outputs.  The segmented replay's records are only used when
// the instances are too few to fill the GPU, i.e. never for large batches.
static int64_t scratch_per_trace(const mcb_trace *t, const int32_t *pols, int n_pol, int n_cap) {
    const int64_t ev = (int64_t)t->num_layers * t->events_per_chain;
    bool ml[2] = {false, false}, nx = false;
    for (int i = 0; i < n_pol; ++i) {
        if (pols[i] == MCB_ML) ml[0] = true;
        if (pols[i] == MCB_ML_NO_PREFILL) ml[1] = true;
        if (pols[i] == MCB_BELADY) nx = true;
    }
    const int64_t E = t->num_experts;
    int64_t b = (int64_t)t->num_layers * n_pol * n_cap * (MCB_R_N + 2) * 8;
    if (nx) b += ev * t->top_k * 4;
    if (ml[0] || ml[1]) b += ev * E * ((ml[0] ? 1 : 0) + (ml[1] ? 1 : 0)) + ev / MCB_TILE_EV * (4 * E + 8) * 4 + ev * 4 + 64;
    return b;
}

// Caller holds c->mu.
static int replay_chunked(mcb_ctx *c, const mcb_trace *t, const int32_t *pols, int32_t n_pol, const int32_t *caps,
                          int32_t n_cap, const mcb_cost *cost, const mcb_nets *nets, const mcb_outputs *out,
                          void *stream) {
    c->last_chunks = 1;
    if (int rc = check_trace(t)) return rc;
    if (!pols || n_pol < 1 || n_pol > MCB_MAX_POL || !caps || n_cap < 1 || n_cap > MCB_MAX_CAP || !out)
        return replay_locked(c, t, pols, n_pol, caps, n_cap, cost, nets, out, (cudaStream_t)stream);
    // Large uniform batches (e.g. C5: 4,096 Qwen3-shaped traces x 4,096 tokens,
    // ~135 GB of rank rows and next-use positions at once) are replayed in
    // consecutive trace ranges that share one bounded scratch.  Every chain
    // is independent, so the results are those of one call.
    int64_t per = t->uniform && t->num_traces > 1 ? scratch_per_trace(t, pols, n_pol, n_cap) : 0;
    int64_t budget = c->scratch_bytes;
    // cudaMemGetInfo is a driver round trip that took 3-76 ms on the GPU box
    // (measured, tools/var_probe.py): a call whose whole scratch is below 10%
    // of the device does not ask for the free memory.
    if (per > 0 && budget == 0 && per * t->num_traces <= c->mem_total / 10) budget = per * t->num_traces;
    // cudaMemGetInfo is a driver round trip that took 3-80 ms on the GPU box
    // (tools/var_probe.py, host-side stalls of the whole step); a call whose
    // scratch fits the buffers an earlier one-range call left does not ask.
    const int64_t need = per * t->num_traces;
    if (per > 0 && budget == 0 && need <= c->fit_need) budget = need;
    if (per > 0 && budget == 0) {
        size_t fr = 0, tot = 0;
        CUDA_TRY(cudaMemGetInfo(&fr, &tot));
        budget = (int64_t)(fr * 0.4);
    }
    const int64_t per_chunk = per > 0 ? std::max<int64_t>(1, budget / per) : t->num_traces;
    if (per == 0 || per_chunk >= t->num_traces || out->outcomes) {
        const int rc = replay_locked(c, t, pols, n_pol, caps, n_cap, cost, nets, out, (cudaStream_t)stream);
        if (rc == MCB_OK && per > 0 && c->scratch_bytes == 0) c->fit_need = std::max(c->fit_need, need);
        return rc;
    }
    for (int k = 0; k < c->n_pieces; ++k)   // trace ranges of their own: the whole upload first
        CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, c->up_ev[k], 0));
    c->n_pieces = 0;
    const int64_t n_cells = (int64_t)n_pol * n_cap, L = t->num_layers;
    const int64_t chain_acc = t->events_per_chain * t->top_k;
    int64_t kernels = 0, chunks = 0;
    for (int64_t t0 = 0; t0 < t->num_traces; t0 += per_chunk) {
        const int64_t n = std::min<int64_t>(per_chunk, t->num_traces - t0);
        mcb_trace sub = *t;
        sub.num_traces = (int32_t)n;
        sub.acc = t->acc + t0 * L * chain_acc;
        mcb_outputs o = *out;
        o.reports = out->reports + t0 * n_cells * MCB_R_N;
        o.latency = out->latency + t0 * n_cells * 2;
        if (out->chain_reports) o.chain_reports = out->chain_reports + t0 * L * n_cells * MCB_R_N;
        if (out->hashes) o.hashes = out->hashes + t0 * L * n_cells;
        if (out->chain_latency) o.chain_latency = out->chain_latency + t0 * L * n_cells * 2;
        if (int rc = replay_locked(c, &sub, pols, n_pol, caps, n_cap, cost, nets, &o, (cudaStream_t)stream,
                                   t0 == 0))
            return rc;
        kernels += c->last_kernels;
        ++chunks;
    }
    c->last_kernels = kernels;
    c->last_chunks = chunks;
    return MCB_OK;
}

extern "C" int mcb_replay(mcb_ctx *c, const mcb_trace *t, const int32_t *pols, int32_t n_pol, const int32_t *caps,
                          int32_t n_cap, const mcb_cost *cost, const mcb_nets *nets, const mcb_outputs *out,
                          void *stream) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    CUDA_TRY(cudaSetDevice(c->device));
    return replay_chunked(c, t, pols, n_pol, caps, n_cap, cost, nets, out, stream);
}

template <typename T>
static int upload(DevBuf &b, const T *src, size_t count, size_t pad_bytes, cudaStream_t s, const T **dst) {
    const size_t bytes = count * sizeof(T);
    if (int rc = b.ensure(bytes + pad_bytes)) return rc;
    if (bytes) CUDA_TRY(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, s));
    if (pad_bytes) CUDA_TRY(cudaMemsetAsync((char *)b.p + bytes, 0, pad_bytes, s));
    *dst = (const T *)b.p;
    return MCB_OK;
}

extern "C" int mcb_replay_host(mcb_ctx *c, const mcb_trace *t, const int32_t *pols, int32_t n_pol,
                               const int32_t *caps, int32_t n_cap, const mcb_cost *cost, const mcb_nets *nets,
                               const mcb_outputs *out, void *stream) {
    mcb_clear_error();
    if (!c) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (int rc = check_trace(t)) return rc;
    if (!out || !out->reports || !out->latency) return mcb_set_error(MCB_ERR_INVALID, "outputs are NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
    mcb_trace dt = *t;
    const DevTrace d = make_dev_trace(t);
    const int64_t n_chains = d.n_chains;
    mcb_nets dn;
    const mcb_nets *npn = nullptr;
    if (nets && nets->params) {
        // the nets' copy runs on side2 while the trace-only stages (K2, key and
        // feature snapshots) start; the scorer waits for it (nets_ev).  It is
        // submitted before the trace: copies in one direction share the copy
        // engine in submission order, and the scorer must not wait for the trace.
        dn = *nets;
        const size_t cnt = net_param_doubles(nets->num_experts, nets->hidden) * (size_t)nets->num_nets;
        CUDA_TRY(cudaEventRecord(c->nets_ev, s));                 // after the previous call's use of h_params
        CUDA_TRY(cudaStreamWaitEvent(c->side2, c->nets_ev, 0));
        if (int rc = upload(c->h_params, nets->params, cnt, 0, c->side2, &dn.params)) return rc;
        CUDA_TRY(cudaEventRecord(c->nets_ev, c->side2));
        c->nets_pending = true;
        npn = &dn;
    }
    // Uniform batches of many traces: upload in trace-range pieces on the copy
    // stream so that the trace-only stages of piece k overlap the copy of k+1
    // (whole traces per piece: a piece's first chain is layer 0).  Batches that
    // will be replayed in scratch-bounded trace ranges take the plain upload.
    c->n_pieces = 0;
    const int np = t->uniform ? (int)std::min<int64_t>(c->upload_pieces, t->num_traces / 8) : 0;
    if (np >= 2) {
        if (int rc = c->h_acc.ensure((size_t)d.total_acc + 256)) return rc;
        uint8_t *dst = (uint8_t *)c->h_acc.p;
        const int64_t per_trace = (int64_t)t->num_layers * t->events_per_chain * t->top_k;
        CUDA_TRY(cudaEventRecord(c->fork, s));   // after the previous call's use of the buffer
        CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->fork, 0));
        CUDA_TRY(cudaMemsetAsync(dst + d.total_acc, 0, 256, c->copy_stream));
        for (int k = 0; k <= np; ++k) c->piece_chain[k] = (int64_t)t->num_traces * k / np * t->num_layers;
        for (int k = 0; k < np; ++k) {
            const int64_t b0 = c->piece_chain[k] / t->num_layers * per_trace;
            const int64_t b1 = c->piece_chain[k + 1] / t->num_layers * per_trace;
            CUDA_TRY(cudaMemcpyAsync(dst + b0, t->acc + b0, (size_t)(b1 - b0), cudaMemcpyHostToDevice, c->copy_stream));
            CUDA_TRY(cudaEventRecord(c->up_ev[k], c->copy_stream));
        }
        dt.acc = dst;
        c->n_pieces = np;
    } else if (int rc = upload(c->h_acc, t->acc, (size_t)d.total_acc, 256, s, &dt.acc)) {
        return rc;
    }
    if (!t->uniform) {
        int64_t total_rt = 0;
        if (n_chains > 0) total_rt = t->chain_rt_off[n_chains];
        if (int rc = upload(c->h_acc_off, t->chain_acc_off, (size_t)n_chains + 1, 0, s, &dt.chain_acc_off)) return rc;
        if (int rc = upload(c->h_ev_off, t->chain_ev_off, (size_t)n_chains + 1, 0, s, &dt.chain_ev_off)) return rc;
        if (int rc = upload(c->h_rt_off, t->chain_rt_off, (size_t)n_chains + 1, 0, s, &dt.chain_rt_off)) return rc;
        if (int rc = upload(c->h_ev_info, t->ev_info, (size_t)d.total_events, 64, s, &dt.ev_info)) return rc;
        if (int rc = upload(c->h_routed, t->routed, (size_t)total_rt, 64, s, &dt.routed)) return rc;
    }
    const int64_t n_cells = (int64_t)t->num_traces * n_pol * n_cap;
    const int64_t n_inst = n_chains * n_pol * n_cap;
    mcb_outputs dout;
    memset(&dout, 0, sizeof dout);
    if (int rc = c->h_reports.ensure((size_t)(n_cells + 1) * MCB_R_N * sizeof(int64_t))) return rc;
    if (int rc = c->h_latency.ensure((size_t)(n_cells + 1) * 2 * sizeof(double))) return rc;
    dout.reports = (int64_t *)c->h_reports.p;
    dout.latency = (double *)c->h_latency.p;
    if (out->chain_reports) {
        if (int rc = c->h_chain_reports.ensure((size_t)(n_inst + 1) * MCB_R_N * sizeof(int64_t))) return rc;
        dout.chain_reports = (int64_t *)c->h_chain_reports.p;
    }
    if (out->hashes) {
        if (int rc = c->h_hashes.ensure((size_t)(n_inst + 1) * sizeof(uint64_t))) return rc;
        dout.hashes = (uint64_t *)c->h_hashes.p;
    }
    if (out->outcomes) {
        if (int rc = c->h_outcomes.ensure((size_t)(n_pol * n_cap * d.total_acc + 1) * sizeof(uint16_t))) return rc;
        dout.outcomes = (uint16_t *)c->h_outcomes.p;
    }
    if (out->chain_latency) {
        if (int rc = c->h_chain_latency.ensure((size_t)(n_inst + 1) * 2 * sizeof(double))) return rc;
        dout.chain_latency = (double *)c->h_chain_latency.p;
    }
    const int rc_replay = replay_chunked(c, &dt, pols, n_pol, caps, n_cap, cost, npn, &dout, s);
    for (int k = 0; k < c->n_pieces; ++k) cudaStreamWaitEvent(s, c->up_ev[k], 0);   // (a path that did not wait)
    c->n_pieces = 0;
    c->pieces_next = false;
    if (c->nets_pending) {   // the stream must not outrun the copy even if no scorer ran
        cudaStreamWaitEvent(s, c->nets_ev, 0);
        c->nets_pending = false;
    }
    if (rc_replay) {
        cudaStreamSynchronize(s);
        return rc_replay;
    }
    CUDA_TRY(cudaMemcpyAsync(out->reports, dout.reports, (size_t)n_cells * MCB_R_N * sizeof(int64_t),
                             cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(out->latency, dout.latency, (size_t)n_cells * 2 * sizeof(double),
                             cudaMemcpyDeviceToHost, s));
    if (out->chain_reports)
        CUDA_TRY(cudaMemcpyAsync(out->chain_reports, dout.chain_reports, (size_t)n_inst * MCB_R_N * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, s));
    if (out->hashes)
        CUDA_TRY(cudaMemcpyAsync(out->hashes, dout.hashes, (size_t)n_inst * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    if (out->outcomes)
        CUDA_TRY(cudaMemcpyAsync(out->outcomes, dout.outcomes, (size_t)n_pol * n_cap * d.total_acc * sizeof(uint16_t),
                                 cudaMemcpyDeviceToHost, s));
    if (out->chain_latency)
        CUDA_TRY(cudaMemcpyAsync(out->chain_latency, dout.chain_latency, (size_t)n_inst * 2 * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
    unsigned long long unc = 0;
    CUDA_TRY(cudaMemcpyAsync(&unc, c->stats.p, sizeof unc, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->last_uncertain = (int64_t)unc;
    return MCB_OK;
}
