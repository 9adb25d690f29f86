// K7: GPU validate + pack of decode-only trace batches.
//
// Input: ids uint8 [n_traces][T][L][K] in the reference's event order
// (trace.py:121-127: one sequence per trace, step-major, then layer) -- the
// payload of a batch-kind .mcbt file.  Output: the engine's chain-major
// uniform layout acc[n_traces * L][T][K] (mcb.h mcb_trace) and the index of
// the first invalid event in event order (AccessEvent.validate,
// trace.py:80-106: an expert outside [0, E) or a duplicate within the
// event), or -1.
//
// HBM-bound transpose: each CTA stages TT consecutive tokens of one trace
// (TT * L * K contiguous bytes, 16-byte vector loads when aligned) in shared
// memory, validates its events there, and writes L runs of TT * K bytes (one
// per layer chain) with 4-byte stores.  Algorithmic traffic 2 B per id.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mcb_internal.h"

namespace tpack {

struct Params {
    const uint8_t *ids;
    uint8_t *acc;
    unsigned long long *first_bad;
    int64_t n, T;
    int L, K, E, TT;
    int vec;   // 16-byte loads legal (every tile starts 16-byte aligned)
};

__global__ void __launch_bounds__(256) k_pack_decode_ids(const __grid_constant__ Params P) {
    extern __shared__ __align__(16) uint8_t tile[];
    const int64_t tiles_per_trace = (P.T + P.TT - 1) / P.TT;
    const int64_t tr = blockIdx.x / tiles_per_trace;
    const int64_t t0 = (blockIdx.x % tiles_per_trace) * P.TT;
    const int tt = (int)min((int64_t)P.TT, P.T - t0);
    const int LK = P.L * P.K;
    const int bytes = tt * LK;
    const uint8_t *src = P.ids + (tr * P.T + t0) * LK;
    if (P.vec && (bytes & 15) == 0) {
        const uint4 *s4 = (const uint4 *)src;
        uint4 *d4 = (uint4 *)tile;
        for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) d4[i] = __ldcs(s4 + i);
    } else {
        for (int i = threadIdx.x; i < bytes; i += blockDim.x) tile[i] = __ldcs(src + i);
    }
    __syncthreads();

    // validate: one thread per event
    for (int ev = threadIdx.x; ev < tt * P.L; ev += blockDim.x) {
        const uint8_t *e = tile + ev * P.K;
        uint32_t seen[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        bool bad = false;
        for (int k = 0; k < P.K; ++k) {
            const uint32_t x = e[k];
            bad |= x >= (uint32_t)P.E;
            const uint32_t w = x >> 5, b = 1u << (x & 31u);
            uint32_t cur = 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q) cur |= (q == (int)w) ? seen[q] : 0u;
            bad |= (cur & b) != 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q) seen[q] |= (q == (int)w) ? b : 0u;
        }
        if (bad) atomicMin(P.first_bad, (unsigned long long)((tr * P.T + t0) * P.L + ev));
    }

    // chain-major stores: layer l's run is out[((tr * L + l) * T + t0) * K ..][tt * K]
    const int run = tt * P.K;
    const int words = (run + 3) / 4;
    for (int i = threadIdx.x; i < P.L * words; i += blockDim.x) {
        const int l = i / words;
        const int j0 = (i % words) * 4;
        uint8_t *dst = P.acc + ((tr * P.L + l) * P.T + t0) * P.K;
        uint32_t w = 0u;
        int nb = 0;
        for (int q = 0; q < 4 && j0 + q < run; ++q, ++nb) {
            const int j = j0 + q;
            const int t = j / P.K, k = j - t * P.K;
            w |= (uint32_t)tile[(t * P.L + l) * P.K + k] << (8 * q);
        }
        if (nb == 4 && (((uintptr_t)(dst + j0)) & 3u) == 0u) {
            __stcs((unsigned int *)(dst + j0), w);
        } else {
            for (int q = 0; q < nb; ++q) dst[j0 + q] = (uint8_t)(w >> (8 * q));
        }
    }
}

}  // namespace tpack

extern "C" int mcb_pack_decode_ids(mcb_ctx *ctx, const uint8_t *ids, int64_t num_traces, int64_t decode_steps,
                                   int32_t num_layers, int32_t top_k, int32_t num_experts, uint8_t *acc,
                                   int64_t *first_bad, void *stream) {
    mcb_clear_error();
    (void)ctx;
    if (num_layers < 1 || num_experts < 1 || top_k < 1 || top_k > num_experts || num_traces < 0 || decode_steps < 0)
        return mcb_set_error(MCB_ERR_INVALID, "invalid batch shape");
    if (num_experts > 256) return mcb_set_error(MCB_ERR_UNSUPPORTED, "num_experts > 256 is not supported");
    if (!first_bad || ((num_traces * decode_steps) > 0 && (!ids || !acc)))
        return mcb_set_error(MCB_ERR_INVALID, "NULL pointer");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(first_bad, 0xFF, sizeof(int64_t), s);
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    if (num_traces * decode_steps == 0) return MCB_OK;
    tpack::Params P;
    P.ids = ids;
    P.acc = acc;
    P.first_bad = (unsigned long long *)first_bad;
    P.n = num_traces;
    P.T = decode_steps;
    P.L = num_layers;
    P.K = top_k;
    P.E = num_experts;
    const int64_t lk = (int64_t)num_layers * top_k;
    int tt = (int)((32 * 1024) / lk);                 // <= 32 KB of tile
    tt = tt >= 16 ? tt / 16 * 16 : (tt < 1 ? 1 : tt);
    if (tt > 1024) tt = 1024;
    if ((int64_t)tt > decode_steps) tt = (int)decode_steps;
    P.TT = tt;
    P.vec = ((uintptr_t)ids % 16 == 0) && ((int64_t)tt * lk % 16 == 0) && (decode_steps * lk % 16 == 0);
    const int64_t tiles = num_traces * ((decode_steps + tt - 1) / tt);
    const size_t smem = (size_t)tt * lk;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(tpack::k_pack_decode_ids, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    }
    tpack::k_pack_decode_ids<<<(unsigned)tiles, 256, smem, s>>>(P);
    e = cudaGetLastError();
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    return MCB_OK;
}
