// K1: synthetic routing-trace generator = router-logits GEMM on the 5th-gen
// tensor cores with a fused per-(token, layer) top-k epilogue (sm_100a).
//
//   logits[t][n] = sum_k hidden[t][k] * weight[n][k]      (bf16 x bf16 -> fp32)
//   acc[l][t][0..K) = the K largest logits of columns [l*Ep, l*Ep + E),
//                     sorted descending, ties to the lower expert id
//
// which is the torch.topk semantics of the HF routers the reference's
// extractor records (pkg/extractor/src/trace_extractor/extractor.py:162-183;
// softmax is monotone, so top-k of logits == top-k of router probabilities).
// The reference has no GEMM generator: parity is against
// torch (tests/test_router_gpu.py).
//
// Persistent kernel, one CTA per SM, 256-token x 128-column tiles:
//   warp 0      TMA producer: 256x64 hidden tile + 128x64 weight tile per
//               stage (SWIZZLE_128B, K-major), 4-stage mbarrier ring (48 KB
//               per stage; the weight tile is shared by both token halves)
//   warp 1      TMEM allocator (512 columns) + the single tcgen05.mma issuer:
//               per K step, M=128 N=128 K=16 for each 128-token half into
//               its own 128-column fp32 accumulator; two accumulator sets
//               (2 x 256 columns) so the MMAs of tile i+1 run while the
//               epilogue drains tile i
//   warps 2..9  epilogue (warp w: TMEM lane quarter w % 4, token half
//               (w - 2) / 4): tcgen05.ld 32 columns at a time; every logit
//               becomes a 32-bit key (order-preserving float bits, low 7
//               bits = 127 - expert) and is inserted branch-free into the
//               running top-K of its layer segment (max/min exchange chain:
//               no divergence between the lanes' tokens); uint8 ids to HBM.
// Tiles are taken round-robin (tile = k * grid + blockIdx.x), n fastest, so
// the ~150 tiles in flight share a few hidden m-blocks and the whole gate
// matrix in L2.
//
// Keys keep the top 25 bits of the order-preserving logit (2^-16 relative):
// logits closer than that are ordered by expert id.  That is far below the
// difference between this kernel's fp32 summation order and torch's (the
// near-tie bound of tests/test_router_gpu.py is 4e-3 absolute).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "mcb_internal.h"

namespace k1 {

constexpr int BM = 256, BN = 128, BK = 64, STAGES = 4;   // BM = two M=128 MMA halves
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int HALF_A = 128 * BK * 2;   // 16 KB: rows 128..255 of the A tile
constexpr int KMAX = 8;             // top-k capacity of the epilogue (K <= 8)
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms of 1024 B
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)1 << 16;                          // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                          // layout: SWIZZLE_128B
    return d;
}

// instruction descriptor, kind::f16: D=f32, A=B=bf16, both K-major, M=128, N=BN
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// order-preserving map of fp32 to uint32 (-0.0 canonicalised to +0.0)
__device__ __forceinline__ uint32_t okey(float x) {
    const uint32_t b = __float_as_uint(x + 0.0f);
    return b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
}

// Running top-K of packed keys, descending; insertion is a max/min exchange
// chain (the same instructions whatever the lane's data).
struct TopK {
    uint32_t v[KMAX];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < KMAX; ++k) v[k] = 0u;
    }
    __device__ __forceinline__ void push(uint32_t x) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const uint32_t hi = max(x, v[k]);
            x = min(x, v[k]);
            v[k] = hi;
        }
    }
};

__global__ void __launch_bounds__(THREADS, 1)
router_topk_kernel(const __grid_constant__ CUtensorMap map_h, const __grid_constant__ CUtensorMap map_w, int T, int Dp,
                   int L, int E, int lgEp, int K, uint8_t *__restrict__ acc, float *__restrict__ logits, int N_total) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the swizzle atoms
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + STAGES * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;     // [2] accumulator set ready
    uint64_t *tempty = tfull + 2;         // [2] accumulator set drained (EPI_WARPS arrivals)
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = Dp / BK;
    const int tiles_n = (N_total + BN - 1) / BN;
    const int64_t n_tiles = (int64_t)((T + BM - 1) / BM) * tiles_n;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], EPI_WARPS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_h)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                const int m0 = (int)(t / tiles_n) * BM, n0 = (int)(t % tiles_n) * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
                    uint8_t *sa = smem + s * STAGE_BYTES;
                    tma_load_2d(sa, &map_h, &full[s], kb * BK, m0);
                    tma_load_2d(sa + A_BYTES, &map_w, &full[s], kb * BK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            uint32_t it = 0, ti = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++ti) {
                const uint32_t buf = ti & 1, d = tmem + 256 * buf;
                mbar_wait(&tempty[buf], ((ti >> 1) & 1) ^ 1);   // the epilogue drained this set
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
                    const uint32_t sb = sa + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // advance 16 bf16 = 32 B along K inside the swizzled rows
                        const uint64_t db = make_desc(sb + k * 32);
                        const uint32_t accum = (kb > 0 || k > 0) ? 1u : 0u;
                        mma_bf16(d, make_desc(sa + k * 32), db, accum);
                        mma_bf16(d + 128, make_desc(sa + HALF_A + k * 32), db, accum);
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&tfull[buf]);
            }
        }
    } else {
        const int q = warp & 3, h = (warp - 2) >> 2;   // TMEM lane quarter, token half
        const uint32_t Ep1 = (1u << lgEp) - 1u;
        uint32_t ti = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++ti) {
            const uint32_t buf = ti & 1;
            const int m0 = (int)(t / tiles_n) * BM, n0 = (int)(t % tiles_n) * BN;
            const int tok = m0 + h * 128 + q * 32 + lane;
            mbar_wait(&tfull[buf], (ti >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            TopK tk;
            tk.reset();
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                float v[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 256 * buf + 128 * h + (uint32_t)c0, v);
                if (logits != nullptr && tok < T) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (n0 + c0 + j < N_total) logits[(int64_t)tok * N_total + n0 + c0 + j] = v[j];
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const uint32_t n = (uint32_t)(n0 + c0 + j);
                    const uint32_t e = n & Ep1;
                    if ((int)e < E) tk.push((okey(v[j]) & ~127u) | (127u - e));
                    if (e == Ep1) {   // end of a layer segment
                        const int layer = (int)(n >> lgEp);
                        if (layer < L && tok < T) {
                            uint8_t *dst = acc + ((int64_t)layer * T + tok) * K;
#pragma unroll
                            for (int k = 0; k < KMAX; ++k)   // static indices: tk stays in registers
                                if (k < K) dst[k] = (uint8_t)(127u - (tk.v[k] & 127u));
                        }
                        tk.reset();
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

int make_map(CUtensorMap *map, const void *base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    auto enc = get_encode();
    if (!enc) return mcb_set_error(MCB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {BK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char b[96];
        snprintf(b, sizeof b, "cuTensorMapEncodeTiled failed (%d)", (int)r);
        return mcb_set_error(MCB_ERR_CUDA, b);
    }
    return MCB_OK;
}

}  // namespace k1

static int k1_num_sms = 0;

int mcb_router_preload() {
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, (const void *)k1::router_topk_kernel) != cudaSuccess)
        return mcb_set_error(MCB_ERR_CUDA, "failed to load the router kernel");
    cudaFuncSetAttribute(k1::router_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, k1::SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&k1_num_sms, cudaDevAttrMultiProcessorCount, dev);
    return MCB_OK;
}

// hidden: bf16 [T][d] (d a multiple of 64, 16-B aligned rows); weight: bf16
// [L*Ep][d] with Ep = num_experts rounded up to a divisor of 256 (rows of
// padding experts are ignored); acc: uint8 [L][T][K].
extern "C" int mcb_router_topk(mcb_ctx *ctx, const void *hidden, const void *weight, int64_t T, int32_t d, int32_t L,
                               int32_t E, int32_t K, uint8_t *acc, float *logits, void *stream) {
    mcb_clear_error();
    if (!ctx || !hidden || !weight || !acc) return mcb_set_error(MCB_ERR_INVALID, "NULL argument");
    if (T < 1 || T > (1ll << 31) - 1) return mcb_set_error(MCB_ERR_INVALID, "T out of range");
    if (d < k1::BK || d % k1::BK) return mcb_set_error(MCB_ERR_INVALID, "hidden dim must be a multiple of 64");
    if (L < 1 || E < 1 || E > MCB_MAX_EXPERTS || K < 1 || K > E || K > k1::KMAX)
        return mcb_set_error(MCB_ERR_INVALID, "need 1 <= K <= min(E, 8), E <= 128");
    int Ep = 8, lgEp = 3;
    while (Ep < E) { Ep *= 2; ++lgEp; }  // power of two, divides the 128-column tile
    const int64_t N = (int64_t)L * Ep;
    CUtensorMap mh, mw;
    if (int rc = k1::make_map(&mh, hidden, (uint64_t)T, (uint64_t)d, k1::BM)) return rc;   // 256-row boxes
    if (int rc = k1::make_map(&mw, weight, (uint64_t)N, (uint64_t)d, k1::BN)) return rc;   // 128-row boxes
    const int64_t tiles = ((T + k1::BM - 1) / k1::BM) * ((N + k1::BN - 1) / k1::BN);
    const int sms = k1_num_sms > 0 ? k1_num_sms : 148;
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
    k1::router_topk_kernel<<<grid, k1::THREADS, k1::SMEM, (cudaStream_t)stream>>>(mh, mw, (int)T, d, L, E, lgEp, K, acc,
                                                                                  logits, (int)N);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    return MCB_OK;
}

// ---- K1 input synthesis: AR(1) hidden states over tokens (bf16) ------------
// h[0][j] = n(0, j), h[t][j] = rho h[t-1][j] + sqrt(1 - rho^2) n(t, j), with
// n a counter-based standard normal (splitmix64 hash of (seed, t, j) -> two
// uniforms -> Box-Muller), so any token chunk can be generated independently:
// pass 1 runs each 512-token chunk from zero, pass 2 carries the chunk ends
// across chunks (h_end[c] = g_end[c] + rho^len h_end[c-1]), pass 3 reruns
// each chunk from its carry and writes bf16 rows [T][d_pad] (column d = 1,
// the bias input of the gate rows; columns > d = 0).
namespace ar1 {

constexpr int CHUNK = 512;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ float normal(uint64_t seed, int64_t t, int j) {
    const uint64_t r = mix64(seed ^ mix64(((uint64_t)t << 20) ^ (uint64_t)j));
    const float u1 = ((float)(uint32_t)(r >> 40) + 0.5f) * (1.0f / 16777216.0f);   // (0, 1)
    const float u2 = (float)(uint32_t)(r & 0xFFFFFFu) * (1.0f / 16777216.0f);
    return sqrtf(-2.0f * logf(u1)) * __cosf(6.283185307179586f * u2);
}

// pass 1 (write_out == false): chunk-end values from a zero start;
// pass 3 (write_out == true): the chunk again from its carry, bf16 rows out
template <bool WRITE>
__global__ void k_ar1_chunk(int64_t T, int d, int d_pad, float rho, float c, uint64_t seed, const float *carry_in,
                            float *chunk_end, __nv_bfloat16 *out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ch = blockIdx.y;
    const int64_t t0 = ch * CHUNK, t1 = min(T, t0 + CHUNK);
    if (j >= d_pad) return;
    if (j >= d) {   // bias column and padding
        if (WRITE)
            for (int64_t t = t0; t < t1; ++t) out[t * d_pad + j] = __float2bfloat16(j == d ? 1.0f : 0.0f);
        return;
    }
    float h = WRITE ? carry_in[ch * d + j] : 0.0f;
    for (int64_t t = t0; t < t1; ++t) {
        const float n = normal(seed, t, j);
        h = t == 0 ? n : fmaf(rho, h, c * n);   // stationary start: h_0 ~ N(0, 1)
        if (WRITE) out[t * d_pad + j] = __float2bfloat16(h);
    }
    if (!WRITE) chunk_end[ch * d + j] = h;
}

// pass 2: carry_in[c] = the true h before chunk c (one thread per column)
__global__ void k_ar1_carry(int64_t T, int d, float rho, const float *chunk_end, float *carry_in) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d) return;
    const int64_t n_ch = (T + CHUNK - 1) / CHUNK;
    const float rho_full = powf(rho, (float)CHUNK);
    float carry = 0.0f;
    for (int64_t ch = 0; ch < n_ch; ++ch) {
        carry_in[ch * d + j] = carry;
        carry = chunk_end[ch * d + j] + (ch == 0 ? 0.0f : rho_full * carry);   // chunk 0 starts at h_0
    }
}

}  // namespace ar1

extern "C" int mcb_ar1_hidden(mcb_ctx *ctx, int64_t T, int32_t d, int32_t d_pad, double rho, uint64_t seed,
                              void *out_bf16, void *stream) {
    mcb_clear_error();
    if (!ctx || !out_bf16) return mcb_set_error(MCB_ERR_INVALID, "NULL argument");
    if (T < 1 || d < 1 || d_pad < d + 1 || !(rho >= 0.0 && rho < 1.0))
        return mcb_set_error(MCB_ERR_INVALID, "need T >= 1, d >= 1, d_pad > d, 0 <= rho < 1");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n_ch = (T + ar1::CHUNK - 1) / ar1::CHUNK;
    float *scratch = nullptr;
    if (cudaMallocAsync((void **)&scratch, sizeof(float) * 2 * (size_t)n_ch * d, s) != cudaSuccess)
        return mcb_set_error(MCB_ERR_NOMEM, "ar1 scratch");
    float *chunk_end = scratch, *carry_in = scratch + (size_t)n_ch * d;
    const float fr = (float)rho, fc = (float)std::sqrt(1.0 - rho * rho);
    const dim3 g1((unsigned)((d + 127) / 128), (unsigned)n_ch), g3((unsigned)((d_pad + 127) / 128), (unsigned)n_ch);
    ar1::k_ar1_chunk<false><<<g1, 128, 0, s>>>(T, d, d_pad, fr, fc, seed, nullptr, chunk_end, nullptr);
    ar1::k_ar1_carry<<<(d + 127) / 128, 128, 0, s>>>(T, d, fr, chunk_end, carry_in);
    ar1::k_ar1_chunk<true><<<g3, 128, 0, s>>>(T, d, d_pad, fr, fc, seed, carry_in, nullptr, (__nv_bfloat16 *)out_bf16);
    cudaFreeAsync(scratch, s);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    return MCB_OK;
}
