// K8: eviction_quality_duel on the GPU (engine.py:404-436; SURVEY.md §8f
// item 4).  Inputs are two policies' per-access outcome streams (the
// engine's outcomes output: victim id, MCB_OUT_HIT or MCB_OUT_MISS) and K2's
// next_pos.  At every access where both policies evict, the victim whose
// next use (OracleIndex.next_use(layer, victim, position), policies.py:65-76)
// is strictly farther wins; ties (both never used again included) drop out.
//
// next_use(v, p) for a victim v at position p: v is resident, so it was
// accessed at some q < p, and with q its last access before p,
// next_use(v, p) = next_pos[q] (v is not the expert accessed at p).  The
// last-access positions come from a blocked scan over each chain:
//   k_duel_tables  warp per (chain, piece): last access of every expert
//                  inside the piece (shared-memory atomicMax);
//   k_duel_scan    thread per (chain, expert): exclusive max-scan over pieces;
//   k_duel_walk    warp per (chain, piece): 32 positions at a time, the last
//                  access before each lane's position from the lanes below
//                  it, else from the running table; compare, count, reduce.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "mcb_internal.h"
#include "mcb_kernels.cuh"

namespace diag {

#define DUEL_PIECE 1024
#define DUEL_WARPS 4

struct Params {
    DevTrace tr;
    const uint16_t *out_a, *out_b;
    const uint32_t *next_pos;
    int32_t *tab;               // [chain][piece][E] last access in piece (-1 none), then exclusive scan
    int64_t max_pieces;
    unsigned long long *wins;   // [2]
};

__device__ __forceinline__ int64_t chain_len(const DevTrace &t, int64_t c) { return t.acc_end(c) - t.acc_begin(c); }

__global__ void __launch_bounds__(32 * DUEL_WARPS) k_duel_tables(const __grid_constant__ Params P) {
    extern __shared__ int32_t s_last[];   // [DUEL_WARPS][E]
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int E = P.tr.E;
    int32_t *last = s_last + w * E;
    const int64_t item = (int64_t)blockIdx.x * DUEL_WARPS + w;
    const int64_t chain = item / P.max_pieces, piece = item % P.max_pieces;
    if (chain >= P.tr.n_chains) return;
    for (int e = lane; e < E; e += 32) last[e] = -1;
    __syncwarp();
    const int64_t a0 = P.tr.acc_begin(chain);
    const int64_t n = chain_len(P.tr, chain);
    const int64_t p0 = piece * DUEL_PIECE, p1 = min(n, p0 + DUEL_PIECE);
    for (int64_t p = p0 + lane; p < p1; p += 32) atomicMax(&last[P.tr.acc[a0 + p]], (int32_t)p);
    __syncwarp();
    int32_t *dst = P.tab + (chain * P.max_pieces + piece) * E;
    for (int e = lane; e < E; e += 32) dst[e] = last[e];
}

__global__ void k_duel_scan(const __grid_constant__ Params P) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int E = P.tr.E;
    if (i >= P.tr.n_chains * E) return;
    const int64_t chain = i / E;
    const int e = (int)(i % E);
    int32_t run = -1;
    int32_t *t = P.tab + chain * P.max_pieces * E + e;
    for (int64_t k = 0; k < P.max_pieces; ++k) {
        const int32_t v = t[k * E];
        t[k * E] = run;
        run = max(run, v);
    }
}

__global__ void __launch_bounds__(32 * DUEL_WARPS) k_duel_walk(const __grid_constant__ Params P) {
    extern __shared__ int32_t s_last[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int E = P.tr.E;
    int32_t *last = s_last + w * E;
    const int64_t item = (int64_t)blockIdx.x * DUEL_WARPS + w;
    const int64_t chain = item / P.max_pieces, piece = item % P.max_pieces;
    uint32_t a_win = 0, b_win = 0;
    if (chain < P.tr.n_chains) {
        const int64_t a0 = P.tr.acc_begin(chain);
        const int64_t n = chain_len(P.tr, chain);
        const int64_t p0 = piece * DUEL_PIECE, p1 = min(n, p0 + DUEL_PIECE);
        const int32_t *src = P.tab + (chain * P.max_pieces + piece) * E;
        for (int e = lane; e < E; e += 32) last[e] = src[e];
        __syncwarp();
        for (int64_t base = p0; base < p1; base += 32) {
            const int64_t p = base + lane;
            const bool in = p < p1;
            const uint32_t x = in ? P.tr.acc[a0 + p] : 0xFFu;
            const uint32_t ca = in ? P.out_a[a0 + p] : MCB_OUT_HIT;
            const uint32_t cb = in ? P.out_b[a0 + p] : MCB_OUT_HIT;
            const bool duel = ca < MCB_OUT_MISS && cb < MCB_OUT_MISS;
            // last access of ca / cb before p: the highest lane below with that id, else the table
            int32_t qa = -1, qb = -1;
            for (int j = 0; j < 32; ++j) {
                const uint32_t xj = __shfl_sync(0xFFFFFFFFu, x, j);
                if (j < lane) {
                    if (xj == ca) qa = (int32_t)(base + j);
                    if (xj == cb) qb = (int32_t)(base + j);
                }
            }
            if (duel) {
                if (qa < 0) qa = last[ca];
                if (qb < 0) qb = last[cb];
                const uint32_t na = qa >= 0 ? __ldg(P.next_pos + a0 + qa) : MCB_NEXT_INF;
                const uint32_t nb = qb >= 0 ? __ldg(P.next_pos + a0 + qb) : MCB_NEXT_INF;
                a_win += na > nb ? 1u : 0u;
                b_win += nb > na ? 1u : 0u;
            }
            __syncwarp();
            if (in) atomicMax(&last[x], (int32_t)p);
            __syncwarp();
        }
    }
    a_win = __reduce_add_sync(0xFFFFFFFFu, a_win);
    b_win = __reduce_add_sync(0xFFFFFFFFu, b_win);
    if (lane == 0 && (a_win | b_win)) {
        atomicAdd(P.wins, (unsigned long long)a_win);
        atomicAdd(P.wins + 1, (unsigned long long)b_win);
    }
}

}  // namespace diag

// defined in mcb_api.cu
DevTrace mcb_dev_trace(const mcb_trace *t);
int mcb_check_trace(const mcb_trace *t);
int mcb_ctx_scratch(mcb_ctx *c, size_t bytes, void **p);

extern "C" int mcb_eviction_duel(mcb_ctx *ctx, const mcb_trace *trace, const uint16_t *outcomes_a,
                                 const uint16_t *outcomes_b, const uint32_t *next_pos, int64_t *wins, void *stream) {
    mcb_clear_error();
    if (!ctx) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (int rc = mcb_check_trace(trace)) return rc;
    if (!outcomes_a || !outcomes_b || !next_pos || !wins) return mcb_set_error(MCB_ERR_INVALID, "NULL pointer");
    cudaStream_t s = (cudaStream_t)stream;
    diag::Params P;
    P.tr = mcb_dev_trace(trace);
    P.out_a = outcomes_a;
    P.out_b = outcomes_b;
    P.next_pos = next_pos;
    P.wins = (unsigned long long *)wins;
    cudaError_t e = cudaMemsetAsync(wins, 0, 2 * sizeof(int64_t), s);
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    int64_t maxlen = 0;
    if (P.tr.uniform) {
        maxlen = P.tr.T * P.tr.K;
    } else {
        std::vector<int64_t> off((size_t)P.tr.n_chains + 1);
        e = cudaMemcpyAsync(off.data(), P.tr.acc_off, off.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
        for (int64_t i = 0; i < P.tr.n_chains; ++i) maxlen = std::max(maxlen, off[i + 1] - off[i]);
    }
    if (maxlen == 0 || P.tr.n_chains == 0) return MCB_OK;
    if (maxlen >= (1ll << 31)) return mcb_set_error(MCB_ERR_UNSUPPORTED, "chains of >= 2^31 accesses");
    P.max_pieces = (maxlen + DUEL_PIECE - 1) / DUEL_PIECE;
    void *tab = nullptr;
    if (int rc = mcb_ctx_scratch(ctx, (size_t)(P.tr.n_chains * P.max_pieces * P.tr.E) * sizeof(int32_t), &tab))
        return rc;
    P.tab = (int32_t *)tab;
    const int64_t items = P.tr.n_chains * P.max_pieces;
    const unsigned blocks = (unsigned)((items + DUEL_WARPS - 1) / DUEL_WARPS);
    const size_t smem = (size_t)DUEL_WARPS * P.tr.E * sizeof(int32_t);
    diag::k_duel_tables<<<blocks, 32 * DUEL_WARPS, smem, s>>>(P);
    const int64_t ne = P.tr.n_chains * P.tr.E;
    diag::k_duel_scan<<<(unsigned)((ne + 127) / 128), 128, 0, s>>>(P);
    diag::k_duel_walk<<<blocks, 32 * DUEL_WARPS, smem, s>>>(P);
    e = cudaGetLastError();
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    return MCB_OK;
}
