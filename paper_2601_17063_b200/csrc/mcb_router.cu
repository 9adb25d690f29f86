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
// One CTA per 128-token x 256-column output tile:
//   warp 0      TMA producer: 128x64 hidden tile + 256x64 weight tile per
//               stage (SWIZZLE_128B, K-major), 4-stage mbarrier ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=256, K=16 per instruction, fp32 accumulator in
//               256 TMEM columns), tcgen05.commit frees smem stages
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time, running top-k per
//               layer segment in registers, uint8 ids to HBM
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>

#include "mcb_internal.h"

namespace k1 {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int KMAX = 8;             // top-k capacity of the epilogue (K <= 8)
constexpr int THREADS = 192;

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

// instruction descriptor, kind::f16: D=f32, A=B=bf16, both K-major, M=128, N=256
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

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

struct TopK {
    float v[KMAX];
    int i[KMAX];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < KMAX; ++k) { v[k] = -INFINITY; i[k] = 0x7FFFFFFF; }
    }
    // columns arrive in ascending id order: strict '>' keeps the lower id on ties
    __device__ __forceinline__ void push(float x, int id) {
        if (x > v[KMAX - 1]) {
            v[KMAX - 1] = x;
            i[KMAX - 1] = id;
#pragma unroll
            for (int k = KMAX - 1; k > 0; --k) {
                if (v[k] > v[k - 1]) {
                    const float tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
                    const int ti = i[k]; i[k] = i[k - 1]; i[k - 1] = ti;
                }
            }
        }
    }
};

__global__ void __launch_bounds__(THREADS, 1)
router_topk_kernel(const __grid_constant__ CUtensorMap map_h, const __grid_constant__ CUtensorMap map_w, int T, int Dp,
                   int L, int E, int Ep, int K, uint8_t *__restrict__ acc, float *__restrict__ logits, int N_total) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the swizzle atoms
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + STAGES * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tmem_full = empty + STAGES;
    uint32_t *tmem_slot = (uint32_t *)(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int nk = Dp / BK;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_h)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
                uint8_t *sa = smem + s * STAGE_BYTES;
                tma_load_2d(sa, &map_h, &full[s], kb * BK, m0);
                tma_load_2d(sa + A_BYTES, &map_w, &full[s], kb * BK, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                mbar_wait(&full[s], (kb / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
                const uint32_t sb = sa + A_BYTES;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    // advance 16 bf16 = 32 B along K inside the swizzled rows
                    mma_bf16(tmem, make_desc(sa + k * 32), make_desc(sb + k * 32), (kb > 0 || k > 0) ? 1u : 0u);
                }
                mma_commit(&empty[s]);
            }
            mma_commit(tmem_full);
        }
    } else {
        // epilogue: warp (2..5) owns TMEM lanes 32*(warp%4) .. +31 = tokens of the tile
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int t = m0 + row;
        mbar_wait(tmem_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        TopK tk;
        tk.reset();
        for (int c0 = 0; c0 < BN; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
            if (logits != nullptr && t < T) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (n0 + c0 + j < N_total) logits[(int64_t)t * N_total + n0 + c0 + j] = v[j];
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = n0 + c0 + j;
                const int layer = n / Ep, e = n - layer * Ep;
                if (e < E && layer < L) tk.push(v[j], e);
                if (e == Ep - 1) {
                    if (layer < L && t < T) {
                        uint8_t *dst = acc + ((int64_t)layer * T + t) * K;
                        for (int k = 0; k < K; ++k) dst[k] = (uint8_t)tk.i[k];
                    }
                    tk.reset();
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
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

int mcb_router_preload() {
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, (const void *)k1::router_topk_kernel) != cudaSuccess)
        return mcb_set_error(MCB_ERR_CUDA, "failed to load the router kernel");
    const size_t smem = (size_t)k1::STAGES * k1::STAGE_BYTES + 1024 + 256;
    cudaFuncSetAttribute(k1::router_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
    int Ep = 8;
    while (Ep < E) Ep *= 2;  // power of two, divides 256
    const int64_t N = (int64_t)L * Ep;
    CUtensorMap mh, mw;
    if (int rc = k1::make_map(&mh, hidden, (uint64_t)T, (uint64_t)d, k1::BM)) return rc;
    if (int rc = k1::make_map(&mw, weight, (uint64_t)N, (uint64_t)d, k1::BN)) return rc;
    const size_t smem = (size_t)k1::STAGES * k1::STAGE_BYTES + 1024 + 256;
    cudaFuncSetAttribute(k1::router_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)((T + k1::BM - 1) / k1::BM), (unsigned)((N + k1::BN - 1) / k1::BN));
    k1::router_topk_kernel<<<grid, k1::THREADS, smem, (cudaStream_t)stream>>>(mh, mw, (int)T, d, L, E, Ep, K, acc, logits,
                                                                               (int)N);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    return MCB_OK;
}
