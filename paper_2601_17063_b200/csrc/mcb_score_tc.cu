// K3-TC: the ML scorer (EvictionNet.forward, pkg/src/moecache/net.py:88-105,
// fed by FeatureTracker, features.py:34-52) on the 5th-gen tensor cores, with
// certified per-event ranks.
//
// The reference scores every event with a float64 3-layer MLP 2E -> 128 ->
// 128 -> E (SiLU) and evicts the arg-max score over resident \ pinned,
// lowest id on ties (mlpolicy.py:15-26).  The replay only needs the ORDER of
// each event's scores (the rank row, shared by every capacity), so:
//
//   1. this kernel evaluates the MLP on tcgen05 in "fp16 x 2" arithmetic:
//      every operand is split into two fp16 parts, a = a0 + a1 with
//      a0 = rn(a), a1 = rn(a - a0) (11 + 1 + 11 + 1 = 24 significant bits,
//      |a - a0 - a1| <= 2^-24 |a|), and the three products a0*w0 + a1*w0 +
//      a0*w1 are accumulated in fp32 in TMEM (the dropped a1*w1 is below
//      2^-22 of a product).  fp16's range is handled with exact powers of
//      two: each layer's weights are scaled per net so that max|w| lies in
//      [2^13, 2^14), layer-1 features (in [0, 1]) by 2^14 and the hidden
//      activations by 2^8; the epilogue folds the inverse scale into one
//      FFMA with the bias.  An activation that would overflow (|h| > 255)
//      marks its event uncertified;
//   2. it sorts each event's E scores (one thread per event, bitonic network
//      on order-preserving keys carrying the expert id in their low bits)
//      and writes the rank row;
//   3. an event is CERTIFIED only if every pair of adjacent scores in that
//      order is separated by more than 2 * tau * max|s| (tau = 4e-6 by
//      default, an order of magnitude above the largest deviation from the
//      float64 forward measured over the test corpus, tests/test_score_tc_gpu.py)
//      and all scores are finite; any other event is appended to a per-net
//      list and RE-SCORED in float64 by k_rescore (mcb_kernels.cu: the fp64
//      DMMA scorer on gathered events), whose ranks overwrite the row.
//
// So every rank row equals the float64 scorer's (the round-1 K3), and ML
// decisions equal the reference's whenever the float64 scores order the
// experts like the reference's BLAS float64 scores.
//
// Kernel shape: persistent, one CTA per SM, 2 + 4 * GROUPS warps:
//   warp 0     weight producer: cp.async.bulk of pre-swizzled fp16 weight
//              blocks (one part x one 64-wide K block) into a ring
//   warp 1     TMEM allocator + the single MMA-issuing thread
//              (tcgen05.mma kind::f16 with fp16 operands, M=128, N=128 / E, K=16)
//   warps 2..  GROUPS epilogue groups of 4 warps: each group owns one
//              128-event tile at a time (one event per thread: TMEM lane =
//              event row), its A buffer (2 parts x 128 x 128 fp16 = 64 KB,
//              plus the score staging) and 128 TMEM columns.
// The groups take turns on the tensor pipe: while one group runs its
// epilogue (features, bias + SiLU + split, or the rank sort), the MMAs of the
// others' layers run.  E <= 64 runs 3 groups (2 weight stages), E = 128 two
// groups (its score staging needs 84 KB) with the activations as the MMA's A
// operand in TMEM (tcgen05.st by the epilogue; 3 weight stages).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <stdio.h>
#include <stdlib.h>

#include "mcb_kernels.cuh"

namespace k3tc {

constexpr int H = 128;                    // EvictionNet hidden size (net.py:64 default)
constexpr int BM = 128;                   // events per tile (MMA M)
constexpr int ROWB = 128;                 // bytes per swizzled row: 64 fp16 (SWIZZLE_128B atom)
constexpr int KBLK = BM * ROWB;           // [128 rows x 64 K] block: 16 KB
constexpr int A_PART = 2 * KBLK;          // one fp16 part of a [128 x 128] operand: 32 KB
constexpr int NPART = 2;                  // fp16 parts per operand
constexpr int W_STAGE = 128 * ROWB;       // one weight block [<= 128 rows x 64 K]: 16 KB
constexpr float FEAT_SCALE = 16384.0f;    // layer-1 features in [0, 1] -> [0, 2^14]
constexpr float ACT_SCALE = 256.0f;       // hidden activations -> x 2^8 (|h| <= 255 certified)
constexpr int NSCALE = 8;                 // per net: 2^s of layers 1..3, then their epilogue multipliers

// TA = activations (the MMA's A operand) in TMEM instead of shared memory:
// 2 groups x (128 accumulator + 128 operand columns), and the shared memory
// left to the score staging goes to a deep weight ring.
template <int GROUPS, int E, bool TA = false>
struct Shape {
    static constexpr int STAGING = ((BM * (E + 1) * 4 + BM * (E + 16)) + 1023) / 1024 * 1024;
    static constexpr int REGION = TA ? STAGING : (E == 128 ? 88 * 1024 : 64 * 1024);   // [A parts +] staging
    static constexpr int SMEM_MAX = 232448;                             // opt-in shared memory per block
    static constexpr int W_STAGES_FIT = (SMEM_MAX - GROUPS * REGION - 1024 - 256) / W_STAGE;
    static constexpr int W_STAGES = W_STAGES_FIT > 8 ? 8 : W_STAGES_FIT;
    static constexpr int THREADS = 64 + 128 * GROUPS;
    static constexpr int SMEM = GROUPS * REGION + W_STAGES * W_STAGE + 1024 + 256;
    static constexpr int TMEM_COLS = (TA ? 256 : 128) * GROUPS > 256 ? 512 : 256;
    static constexpr int D_STRIDE = TA ? 256 : 128;                     // TMEM columns per group
    static_assert(W_STAGES >= 2, "the MMA order holds a job's two part-0 blocks at once");
    static_assert(!TA || GROUPS * 256 <= 512, "TMEM: 256 columns per group");
};

struct Params {
    DevTrace tr;
    const uint8_t *wimg;        // per net: swizzled fp16 weight blocks (k_prep_tc)
    int64_t net_bytes;
    const float *bias;          // per net: b1[128] b2[128] b3[N3] scales[NSCALE] -log2(e)*b1[128] -log2(e)*b2[128]
    int bias_stride;
    int num_nets;
    int N3, KB1, P1;            // layer-3 N (E rounded up to 16), layer-1 K blocks, layer-1 passes
    int64_t n_tiles, tpc, tpc32;
    int64_t ev_base;            // event index of this launch's first chain in the flag lists (trace pieces)
    const int32_t *snaps;       // K3 tracker snapshots every 32 events (k_snap_scan)
    uint8_t *ranks;             // [event][E]
    float tau;
    int32_t *flag_cnt;          // [num_nets]
    int32_t *flag_list;         // [num_nets][bucket_cap]
    int64_t bucket_cap;
    unsigned long long *stats;  // [5] += events flagged for the float64 re-score
    float *dbg_scores;          // optional [event][E]: the fp32 scores (tests / calibration)
};

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
// the same, letting the thread sleep until the phase completes (the producer
// and the MMA issuer: their polling would steal issue slots from epilogue warps)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms of 1024 B
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
// kind::f16 instruction descriptor: D = f32 (bit 4), A = B = f16 (format 0),
// K-major, N >> 3 at bit 17, M >> 4 at bit 24
__device__ __forceinline__ uint32_t idesc(int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(id), "r"(acc));
}
// A operand from TMEM (tcgen05.mma ... [d], [a], b_desc): M=128 rows = lanes,
// two fp16 K values per 32-bit column (lower K in the low half)
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// one lane of the (converged) warp -- the same lane every time, so the
// tcgen05.commit that tracks a job's MMAs is issued by the thread that issued them
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// 32 consecutive fp32 TMEM columns of this thread's lane (no wait)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// st.shared writes become visible to the tensor core's async proxy
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr float LOG2E = 1.4426950408889634f;
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// byte offset of the 16-B chunk `ch` (0..7) of row `row` inside a
// [rows x 64] fp16 block in the SWIZZLE_128B K-major layout
__host__ __device__ __forceinline__ uint32_t sw128(int row, int ch) {
    return (uint32_t)row * ROWB + ((uint32_t)(ch ^ (row & 7)) << 4);
}

// (a, b) = (a0 + a1, b0 + b1), fp16 parts rounded to nearest, two values per
// cvt.rn.f16x2.f32 (the remainders a - a0 are exact in fp32)
__device__ __forceinline__ void split2x2(float a, float b, uint32_t &w0, uint32_t &w1) {
    const __half2 p0 = __floats2half2_rn(a, b);
    const float2 f0 = __half22float2(p0);
    const __half2 p1 = __floats2half2_rn(a - f0.x, b - f0.y);
    w0 = *(const uint32_t *)&p0;
    w1 = *(const uint32_t *)&p1;
}

// eight consecutive K values of one row -> the two parts' 16-B chunks
__device__ __forceinline__ void store_chunk8(uint8_t *abuf, int row, int k0, const float (&v)[8]) {
    uint32_t w[NPART][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) split2x2(v[2 * j], v[2 * j + 1], w[0][j], w[1][j]);
    const uint32_t off = (uint32_t)(k0 >> 6) * KBLK + sw128(row, (k0 & 63) >> 3);
#pragma unroll
    for (int p = 0; p < NPART; ++p)
        *(uint4 *)(abuf + p * A_PART + off) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

// order-preserving map of fp32 to uint32 (-0.0 canonicalised to +0.0)
__device__ __forceinline__ uint32_t okey(float x) {
    const uint32_t b = __float_as_uint(x + 0.0f);
    return b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
}

// ascending sort network: Batcher's odd-even merge sort (543 comparators for
// 64 keys against the bitonic network's 672), recursive templates so every
// index is a compile-time constant (the keys stay in registers)
template <int N>
__device__ __forceinline__ void cswap(uint32_t (&v)[N], int a, int b) {
    const uint32_t x = v[a], y = v[b];
    v[a] = min(x, y);
    v[b] = max(x, y);
}
template <int LO, int N, int R, int NV>
__device__ __forceinline__ void oem_merge(uint32_t (&v)[NV]) {
    constexpr int M = R * 2;
    if constexpr (M < N) {
        oem_merge<LO, N, M, NV>(v);
        oem_merge<LO + R, N, M, NV>(v);
#pragma unroll
        for (int i = LO + R; i + R < LO + N; i += M) cswap(v, i, i + R);
    } else {
        cswap(v, LO, LO + R);
    }
}
template <int LO, int N, int NV>
__device__ __forceinline__ void oem_sort_range(uint32_t (&v)[NV]) {
    if constexpr (N > 1) {
        constexpr int M = N / 2;
        oem_sort_range<LO, M, NV>(v);
        oem_sort_range<LO + M, M, NV>(v);
        oem_merge<LO, N, 1, NV>(v);
    }
}
template <int N>
__device__ __forceinline__ void oem_sort(uint32_t (&v)[N]) {
    oem_sort_range<0, N, N>(v);
}
// bitonic network (E = 128: the odd-even network's live ranges spill there)
template <int N>
__device__ __forceinline__ void bitonic_sort(uint32_t (&v)[N]) {
#pragma unroll
    for (int k = 2; k <= N; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const uint32_t a = v[i], b = v[l];
                    const bool up = (i & k) == 0;
                    v[i] = up ? min(a, b) : max(a, b);
                    v[l] = up ? max(a, b) : min(a, b);
                }
            }
}

// Tile order shared by the producer, the MMA issuer and the epilogue groups:
// the k-th tile set of CTA b is tiles (k * G + b) * GROUPS + g, g = epilogue
// group; per tile set the jobs (layer-1 passes, layer 2, layer 3) run in
// order, the groups interleaved within each job.
template <int E, int GROUPS, bool TA>
__global__ void __launch_bounds__(Shape<GROUPS, E, TA>::THREADS, 1) k_score_tc(const __grid_constant__ Params P) {
    using S = Shape<GROUPS, E, TA>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *abuf0 = smem;                         // group regions (A operand + score staging)
    uint8_t *wring = smem + GROUPS * S::REGION;    // weight ring
    uint64_t *bars = (uint64_t *)(wring + S::W_STAGES * W_STAGE);
    uint64_t *w_full = bars, *w_empty = bars + S::W_STAGES;
    uint64_t *feat_ready = bars + 2 * S::W_STAGES, *acc_ready = feat_ready + GROUPS;
    uint32_t *tmem_slot = (uint32_t *)(acc_ready + GROUPS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P1 = P.P1, JOBS = P1 + 2;
    const int64_t G = gridDim.x, b = blockIdx.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S::W_STAGES; ++s) { mbar_init(&w_full[s], 1); mbar_init(&w_empty[s], 1); }
        for (int g = 0; g < GROUPS; ++g) { mbar_init(&feat_ready[g], 128); mbar_init(&acc_ready[g], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(S::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    const int64_t T = P.tr.T;
    const int L = P.tr.L;
    auto net_of_tile = [&](int64_t t) -> int {
        const int64_t c = t / P.tpc;
        return P.num_nets == 1 ? 0 : (int)(c % L);
    };
    auto job_kblocks = [&](int j) -> int { return j < P1 ? min(2, P.KB1 - 2 * j) : 2; };
    auto job_n = [&](int j) -> int { return j == P1 + 1 ? P.N3 : H; };
    // weight block (layer of job j, global K block, part) of a net
    auto wblock = [&](int net, int j, int kbl, int part) -> const uint8_t * {
        const uint8_t *base = P.wimg + (int64_t)net * P.net_bytes;
        if (j < P1) return base + (int64_t)((2 * j + kbl) * NPART + part) * KBLK;
        base += (int64_t)P.KB1 * NPART * KBLK;
        if (j == P1) return base + (int64_t)(kbl * NPART + part) * KBLK;
        base += (int64_t)2 * NPART * KBLK;
        return base + (int64_t)(kbl * NPART + part) * P.N3 * ROWB;
    };

    if (warp == 0) {
        // ---------------------------------------------------- weight producer
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t k = 0;; ++k) {
                const int64_t t0 = (k * G + b) * GROUPS;
                if (t0 >= P.n_tiles) break;
                for (int j = 0; j < JOBS; ++j)
                    for (int g = 0; g < GROUPS; ++g) {
                        const int64_t t = t0 + g;
                        if (t >= P.n_tiles) continue;
                        const int net = net_of_tile(t), nkb = job_kblocks(j);
                        const uint32_t bytes = (uint32_t)job_n(j) * ROWB;
                        // the job's weight blocks: part 1 of every K block, then part 0
                        for (int part = NPART - 1; part >= 0; --part)
                            for (int kbl = 0; kbl < nkb; ++kbl, ++it) {
                                const int s = it % S::W_STAGES;
                                mbar_wait_sleep(&w_empty[s], ((it / S::W_STAGES) & 1) ^ 1);
                                mbar_arrive_expect_tx(&w_full[s], bytes);
                                bulk_g2s(wring + s * W_STAGE, wblock(net, j, kbl, part), bytes, &w_full[s]);
                            }
                    }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer
        // The whole warp walks the schedule, so every operand (TMEM address,
        // smem descriptors, instruction descriptor) is warp-uniform and lives in
        // uniform registers; one elected lane issues each block's MMAs and
        // commits.  The issue rate matters: a group's job is 24 MMAs.
        {
            uint32_t it = 0, fr[GROUPS];
#pragma unroll
            for (int g = 0; g < GROUPS; ++g) fr[g] = 0u;
            const uint64_t wdesc0 = make_desc(smem_u32(wring));   // + (slot offset >> 4)
            const uint64_t adesc0 = make_desc(smem_u32(abuf0));   // + (A offset >> 4)
            for (int64_t k = 0;; ++k) {
                const int64_t t0 = (k * G + b) * GROUPS;
                if (t0 >= P.n_tiles) break;
                for (int j = 0; j < JOBS; ++j)
#pragma unroll
                    for (int g = 0; g < GROUPS; ++g) {
                        const int64_t t = t0 + g;
                        if (t >= P.n_tiles) continue;
                        mbar_wait_sleep(&feat_ready[g], fr[g] & 1);
                        ++fr[g];
                        __syncwarp();
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint32_t d = tmem + (uint32_t)(S::D_STRIDE * g);
                        const uint32_t id = idesc(job_n(j));
                        const uint64_t ag = adesc0 + (uint64_t)((g * S::REGION) >> 4);
                        const uint32_t a_tm = d + 128;   // TA: the group's operand columns
                        bool fresh = !(j > 0 && j < P1);   // layer-1 passes > 0 accumulate
                        const int nkb = job_kblocks(j);
                        // Small products first, the leading a0*w0 last: the cross terms
                        // a0*w1 (weight part 1) and a1*w0 are summed while the accumulator
                        // is still small, so the accumulator's alignment to its running
                        // magnitude costs them nothing; then a0*w0 over the same K blocks.
                        // The ring holds the job's <= 2 part-0 blocks at once (W_STAGES >= 2).
                        // layer-1 K steps stop at 2E (E = 8, 16: the rest of the block is padding)
                        constexpr int NS1 = 2 * E < 64 ? 2 * E / 16 : 4;
                        const bool short_k = NS1 < 4 && j < P1;
                        // (descriptor start addresses advance by 32 B = 2 units per K step)
                        auto issue_n = [&](auto ns_c, uint32_t a_part, int s, int kbl) {
                            constexpr int NS = decltype(ns_c)::value;
                            const uint64_t wd = wdesc0 + (uint64_t)((s * W_STAGE) >> 4);
                            if constexpr (TA) {
                                const uint32_t a0 = a_tm + a_part * 64 + kbl * 32;
#pragma unroll
                                for (int k4 = 0; k4 < NS; ++k4) {
                                    mma_f16_ts(d, a0 + k4 * 8, wd + 2 * k4, id, fresh ? 0u : 1u);
                                    fresh = false;
                                }
                            } else {
                                const uint64_t ad = ag + (uint64_t)((a_part * A_PART + kbl * KBLK) >> 4);
#pragma unroll
                                for (int k4 = 0; k4 < NS; ++k4) {
                                    mma_f16(d, ad + 2 * k4, wd + 2 * k4, id, fresh ? 0u : 1u);
                                    fresh = false;
                                }
                            }
                        };
                        auto issue = [&](uint32_t a_part, int s, int kbl) {
                            if (short_k) issue_n(std::integral_constant<int, NS1>{}, a_part, s, kbl);
                            else issue_n(std::integral_constant<int, 4>{}, a_part, s, kbl);
                        };
                        for (int kbl = 0; kbl < nkb; ++kbl, ++it) {   // part 1: a0 * w1
                            const int s = it % S::W_STAGES;
                            mbar_wait_sleep(&w_full[s], (it / S::W_STAGES) & 1);
                            __syncwarp();
                            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                            if (elect_one()) {
                                issue(0, s, kbl);
                                mma_commit(&w_empty[s]);
                            }
                            __syncwarp();
                            fresh = false;
                        }
                        const uint32_t it0 = it;
                        for (int kbl = 0; kbl < nkb; ++kbl) {          // part 0: a1 * w0
                            const uint32_t i2 = it0 + kbl;
                            const int s = i2 % S::W_STAGES;
                            mbar_wait_sleep(&w_full[s], (i2 / S::W_STAGES) & 1);
                            __syncwarp();
                            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                            if (elect_one()) issue(1, s, kbl);
                            __syncwarp();
                            fresh = false;
                        }
                        for (int kbl = 0; kbl < nkb; ++kbl, ++it) {   // part 0: a0 * w0
                            const int s = it % S::W_STAGES;
                            if (elect_one()) {
                                issue(0, s, kbl);
                                mma_commit(&w_empty[s]);
                            }
                            __syncwarp();
                        }
                        if (elect_one()) mma_commit(&acc_ready[g]);
                        __syncwarp();
                    }
            }
        }
    } else {
        // ---------------------------------------------------- epilogue groups
        // group g = 4 warps, one per TMEM lane quarter (32 event rows each)
        const int g = (warp - 2) >> 2;
        const int q = warp & 3;                 // TMEM lane quarter of this warp
        const int row = q * 32 + lane;          // event row of the tile = TMEM lane
        uint8_t *abuf = abuf0 + g * S::REGION;
        const uint32_t t_acc = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(S::D_STRIDE * g);
        const uint32_t t_a = t_acc + 128;   // TA: this lane quarter's operand columns (part p at + 64 p)
        // eight consecutive K values of this thread's row -> both fp16 parts of the A operand
        auto put8 = [&](int k0, const float (&v)[8]) {
            if constexpr (TA) {
                uint32_t w0[4], w1[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) split2x2(v[2 * j], v[2 * j + 1], w0[j], w1[j]);
                tmem_st4(t_a + (uint32_t)(k0 >> 1), w0);
                tmem_st4(t_a + 64 + (uint32_t)(k0 >> 1), w1);
            } else {
                store_chunk8(abuf, row, k0, v);
            }
        };
        // the A operand of the next MMA job is complete
        auto publish = [&]() {
            if constexpr (TA) tmem_wait_st();
            else fence_async_smem();
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&feat_ready[g]);
        };
        const int SN = 2 * E + 4;
        constexpr int IDB = E <= 8 ? 3 : E <= 16 ? 4 : E <= 32 ? 5 : E <= 64 ? 6 : 7;   // id bits in a key
        // staging (the region after the last layer's MMAs): fp32 scores
        // [row][E + 1] (odd stride: conflict-free columns), then rank rows [row][E + 16]
        static_assert(BM * (E + 1) * 4 + BM * (E + 16) <= S::REGION, "score staging");
        float *sc = (float *)abuf;
        uint32_t ar = 0;
        for (int64_t k = 0;; ++k) {
            const int64_t t = (k * G + b) * GROUPS + g;
            if (t >= P.n_tiles) break;
            const int64_t c = t / P.tpc, ev0 = (t % P.tpc) * BM, ev = ev0 + row;
            const bool valid = ev < T;
            const int net = P.num_nets == 1 ? 0 : (int)(c % L);
            const float *nb = P.bias + (int64_t)net * P.bias_stride;
            const float *mult = nb + 2 * H + P.N3 + 3;   // epilogue multipliers of layers 1..3
            bool bad = false;
            // this event's routed experts as a 128-bit mask
            uint32_t mine[4] = {0u, 0u, 0u, 0u};
            if (valid) {
                const uint8_t *ids = P.tr.acc + (c * T + ev) * P.tr.K;
                for (int kk = 0; kk < P.tr.K; ++kk) {
                    const int x = __ldg(ids + kk);
                    const uint32_t bit = 1u << (x & 31);
#pragma unroll
                    for (int w = 0; w < 4; ++w) mine[w] |= (x >> 5) == w ? bit : 0u;
                }
            }
            // tracker snapshot at the start of this warp's 32-event sub-tile,
            // distributed: lane l keeps last / f of experts l, l + 32, ...
            const int64_t s32 = (ev0 >> 5) + q;
            const bool has_snap = s32 < P.tpc32;
            const int32_t *sp = P.snaps + (c * P.tpc32 + (has_snap ? s32 : 0)) * SN;
            constexpr int NW = (E + 31) / 32;
            constexpr int EW = E < 32 ? E : 32;   // experts per mask word
            int32_t s_last[NW], s_f[NW];
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                const int e = lane + 32 * j;
                s_last[j] = (has_snap && e < E) ? __ldg(sp + e) : -1;
                s_f[j] = (has_snap && e < E) ? __ldg(sp + E + e) : 0;
            }
            const int32_t u0 = (int32_t)(s32 * 32);
            const int32_t u = u0 + lane + 1;   // this event's update index (1-based)
            const uint32_t upto = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);
            // max_f over experts at this event (features.py:44-52)
            int32_t maxf = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {   // 32-expert words: the word index is static
#pragma unroll 8
                for (int el = 0; el < EW; ++el) {
                    const uint32_t m = __ballot_sync(0xFFFFFFFFu, (mine[w] >> el) & 1u);
                    const int32_t f = __shfl_sync(0xFFFFFFFFu, s_f[w], el) + __popc(m & upto);
                    maxf = max(maxf, f);
                }
            }
            // f / max_f, pre-scaled by 2^14 for fp16
            const float rmaxf = maxf > 0 ? FEAT_SCALE / (float)maxf : 0.0f;
            named_sync(1 + g, 128);   // every thread is done with the previous tile's staging
            // ---- layer-1 input: [1/r || f / max_f] x 2^14 (K = 2E, zero padded to KB1 * 64).
            // E <= 64: one pass holds both halves; E = 128: recency, then frequency.
            constexpr int P1C = 2 * E <= 128 ? 1 : 2;   // == P.P1
#pragma unroll
            for (int p = 0; p < P1C; ++p) {
                if (p > 0) {   // the previous pass's MMAs have consumed the A buffer
                    mbar_wait(&acc_ready[g], ar & 1);
                    ++ar;
                }
                const bool want_r = P1C == 1 || p == 0, want_f = P1C == 1 || p == 1;   // static per pass
                const int kr = 2 * E <= 128 ? 0 : -128 * p, kf = 2 * E <= 128 ? E : E - 128 * p;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
#pragma unroll 1
                    for (int e8 = 0; e8 < EW; e8 += 8) {
                        float rv[8], fv[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int el = e8 + i;
                            const uint32_t m = __ballot_sync(0xFFFFFFFFu, (mine[w] >> el) & 1u);
                            const uint32_t seen = m & upto;
                            const int32_t sl = __shfl_sync(0xFFFFFFFFu, s_last[w], el);
                            const int32_t sf = __shfl_sync(0xFFFFFFFFu, s_f[w], el);
                            const int32_t lastu = seen ? u0 + 32 - __clz(seen) : sl;
                            rv[i] = lastu < 0 ? 0.0f : FEAT_SCALE * rcp_ftz((float)(u - lastu + 1));
                            fv[i] = (float)(sf + __popc(seen)) * rmaxf;
                        }
                        const int e0 = 32 * w + e8;
                        if (want_r) put8(kr + e0, rv);
                        if (want_f) put8(kf + e0, fv);
                    }
                }
                publish();   // (the MMAs read layer-1 K steps up to 2E only: no padding)
            }
            // ---- hidden layers: h = silu(acc * 2^-s + bias) -> next A operand (x 2^8)
            for (int layer = 0; layer < 2; ++layer) {
                mbar_wait(&acc_ready[g], ar & 1);
                ++ar;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                // u = -log2(e) * z in one FFMA (prescaled multiplier and bias),
                // h * 2^8 = u * (-2^8 / log2(e)) * 1 / (1 + 2^u)
                const float *nbias = nb + 2 * H + P.N3 + NSCALE + layer * H;
                const float mul = __ldg(mult + layer) * -LOG2E;
                float hmax = 0.0f;
#pragma unroll 1
                for (int c0 = 0; c0 < H; c0 += 32) {
                    uint32_t ra[32];
                    tmem_ld32_nowait(t_acc + c0, ra);
                    float4 b0 = __ldg((const float4 *)(nbias + c0)), b1 = __ldg((const float4 *)(nbias + c0) + 1);
                    tmem_wait_ld();
#pragma unroll
                    for (int c8 = 0; c8 < 32; c8 += 8) {
                        const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                        if (c8 + 8 < 32) {
                            b0 = __ldg((const float4 *)(nbias + c0 + c8 + 8));
                            b1 = __ldg((const float4 *)(nbias + c0 + c8 + 8) + 1);
                        }
                        float v[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float uu = fmaf(__uint_as_float(ra[c8 + i]), mul, bb[i]);
                            const float r = rcp_ftz(1.0f + ex2_ftz(uu));
                            v[i] = (uu * (-ACT_SCALE / LOG2E)) * r;
                            hmax = fmaxf(hmax, fabsf(v[i]));
                        }
                        put8(c0 + c8, v);
                    }
                }
                bad |= !(hmax <= 255.0f * ACT_SCALE);   // fp16 range of the scaled activations (and NaN)
                publish();
            }
            // ---- scores: s = acc * 2^-s + b3, one thread per event sorts
            // the E keys and certifies the order
            mbar_wait(&acc_ready[g], ar & 1);
            ++ar;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            constexpr int EP = E;   // E is a power of two
            constexpr uint32_t M = (1u << IDB) - 1u;
            {
                const float *b3 = nb + 2 * H;
                const float mul = __ldg(mult + 2);
                float *srow = sc + row * (E + 1);
                uint8_t *rrow = (uint8_t *)(sc + BM * (E + 1)) + row * (E + 16);
                uint32_t key[EP];
#pragma unroll
                for (int c0 = 0; c0 < EP; c0 += 32) {
                    uint32_t ra[32];
                    tmem_ld32_nowait(t_acc + c0, ra);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int e = c0 + i;
                        if (e < E) {
                            const float s = fmaf(__uint_as_float(ra[i]), mul, __ldg(b3 + e));
                            bad |= !isfinite(s);
                            srow[e] = s;
                            key[e] = (okey(s) & ~M) | (uint32_t)e;
                        }
                    }
                }
                if constexpr (E == 128) bitonic_sort<EP>(key); else oem_sort<EP>(key);
                // certify: adjacent scores apart by more than 2 tau max|s|, no
                // truncated-key collision (then the sorted order is the exact order)
                const float smin = srow[key[0] & M], smax = srow[key[E - 1] & M];
                const float thr = 2.0f * P.tau * fmaxf(fabsf(smin), fabsf(smax));
                float prev = smin;
#pragma unroll
                for (int n = 0; n < E; ++n) {
                    const int id = (int)(key[n] & M);
                    if (n > 0) {
                        const float cur = srow[id];
                        bad |= ((key[n] ^ key[n - 1]) >> IDB) == 0u;
                        bad |= !(cur - prev > thr);
                        prev = cur;
                    }
                    rrow[id] = (uint8_t)(n + 1);
                }
                if (valid) {
                    uint8_t *dst = P.ranks + (c * T + ev) * E;
                    if constexpr (E % 16 == 0) {
#pragma unroll
                        for (int i = 0; i < E; i += 16) *(uint4 *)(dst + i) = *(const uint4 *)(rrow + i);
                    } else {
#pragma unroll
                        for (int i = 0; i < E; i += 8) *(uint2 *)(dst + i) = *(const uint2 *)(rrow + i);
                    }
                    if (P.dbg_scores) {
                        float *ds = P.dbg_scores + (c * T + ev) * E;
                        for (int e = 0; e < E; ++e) ds[e] = srow[e];
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            {
                const bool flagged = valid && bad;
                if (flagged) {
                    const int slot = atomicAdd(P.flag_cnt + net, 1);
                    P.flag_list[(int64_t)net * P.bucket_cap + slot] = (int32_t)(P.ev_base + c * T + ev);
                }
                const unsigned nbad = __popc(__ballot_sync(0xFFFFFFFFu, flagged));
                if (lane == 0 && nbad) atomicAdd(P.stats + 5, (unsigned long long)nbad);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(S::TMEM_COLS));
    }
}

// Per (net, layer): the power of two 2^s with max|w| * 2^s in [2^13, 2^14)
// (fp16 range with headroom for the split; s clamped to +-100), and the
// epilogue multiplier 2^-(s + activation scale).  One block per (net, layer).
__global__ void k_wscale(const double *__restrict__ params, int E, int N3, float *__restrict__ bias, int bias_stride) {
    const int net = blockIdx.x / 3, layer = blockIdx.x % 3;
    const int D = 2 * E;
    const int64_t src_per = (int64_t)D * H + H + (int64_t)H * H + H + (int64_t)E * H + E;
    const double *src = params + net * src_per;
    const double *w = layer == 0 ? src : layer == 1 ? src + (int64_t)D * H + H : src + (int64_t)D * H + H + (int64_t)H * H + H;
    const int n = layer == 0 ? D * H : layer == 1 ? H * H : E * H;
    double m = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(w[i]));
    __shared__ double red[256];
    red[threadIdx.x] = m;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        m = red[0];
        int s = 0;
        if (m > 0.0 && isfinite(m)) s = 13 - ilogb(m);
        s = max(-100, min(100, s));
        const int act = layer == 0 ? 14 : 8;   // FEAT_SCALE, ACT_SCALE
        float *sc = bias + (int64_t)net * bias_stride + 2 * H + N3;
        sc[layer] = ldexpf(1.0f, s);
        sc[3 + layer] = ldexpf(1.0f, -(s + act));
    }
}

// Weight images: per net, the fp16 x 2 parts of 2^s * W1 (N = 128, K = 2E
// padded to a multiple of 64), 2^s * W2 (128 x 128) and 2^s * W3 (N3 x 128),
// as [N x 64] blocks in the SWIZZLE_128B K-major layout in MMA consumption
// order (layer, K block, part), and fp32 biases b1, b2, b3 (padded to N3).
// params: .evnet order.  Runs after k_wscale.
__global__ void k_prep_tc(const double *__restrict__ params, int E, int num_nets, int KB1, int N3,
                          int64_t net_bytes, uint8_t *__restrict__ wimg, float *__restrict__ bias, int bias_stride) {
    const int D = 2 * E;
    const int64_t src_per = (int64_t)D * H + H + (int64_t)H * H + H + (int64_t)E * H + E;
    // one thread per (net, layer, row n, 8-wide K chunk)
    const int64_t per_net_chunks = (int64_t)H * (KB1 * 8) + (int64_t)H * 16 + (int64_t)N3 * 16;
    const int64_t total = per_net_chunks * num_nets;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int net = (int)(i / per_net_chunks);
        int64_t r = i % per_net_chunks;
        const double *src = params + net * src_per;
        const double *w;
        int n, ch, ldw, kmax, nmax, layer;
        if (r < (int64_t)H * KB1 * 8) {
            layer = 0; n = (int)(r / (KB1 * 8)); ch = (int)(r % (KB1 * 8)); w = src; ldw = D; kmax = D; nmax = H;
        } else if ((r -= (int64_t)H * KB1 * 8) < (int64_t)H * 16) {
            layer = 1; n = (int)(r / 16); ch = (int)(r % 16); w = src + (int64_t)D * H + H; ldw = H; kmax = H; nmax = H;
        } else {
            r -= (int64_t)H * 16;
            layer = 2; n = (int)(r / 16); ch = (int)(r % 16);
            w = src + (int64_t)D * H + H + (int64_t)H * H + H; ldw = H; kmax = H; nmax = E;
        }
        const double scale = (double)bias[(int64_t)net * bias_stride + 2 * H + N3 + layer];
        const int kb = ch >> 3, c8 = ch & 7, Nl = layer == 2 ? N3 : H;
        uint32_t part[NPART][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint16_t h[NPART][2];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int kk = kb * 64 + c8 * 8 + 2 * j + hh;
                const double x = (n < nmax && kk < kmax) ? w[(int64_t)n * ldw + kk] * scale : 0.0;
                const __half p0 = __double2half(x);
                const __half p1 = __double2half(x - (double)__half2float(p0));
                h[0][hh] = __half_as_ushort(p0);
                h[1][hh] = __half_as_ushort(p1);
            }
#pragma unroll
            for (int p = 0; p < NPART; ++p) part[p][j] = (uint32_t)h[p][0] | ((uint32_t)h[p][1] << 16);
        }
        uint8_t *base = wimg + (int64_t)net * net_bytes;
        int64_t blk0;
        if (layer == 0) blk0 = (int64_t)(kb * NPART) * KBLK;
        else if (layer == 1) blk0 = (int64_t)KB1 * NPART * KBLK + (int64_t)(kb * NPART) * KBLK;
        else blk0 = (int64_t)(KB1 + 2) * NPART * KBLK + (int64_t)(kb * NPART) * N3 * ROWB;
        const int64_t blk_bytes = (int64_t)Nl * ROWB;
#pragma unroll
        for (int p = 0; p < NPART; ++p)
            *(uint4 *)(base + blk0 + p * blk_bytes + sw128(n, c8)) =
                make_uint4(part[p][0], part[p][1], part[p][2], part[p][3]);
        if (ch == 0) {   // biases (fp32)
            float *bb = bias + (int64_t)net * bias_stride;
            const double *b1 = src + (int64_t)D * H, *b2 = b1 + H + (int64_t)H * H,
                         *b3 = b2 + H + (int64_t)E * H;
            float *nbb = bb + 2 * H + N3 + NSCALE;   // the hidden layers' biases times -log2(e)
            if (layer == 0) { bb[n] = (float)b1[n]; nbb[n] = (float)(b1[n] * -1.4426950408889634); }
            else if (layer == 1) { bb[H + n] = (float)b2[n]; nbb[H + n] = (float)(b2[n] * -1.4426950408889634); }
            else bb[2 * H + n] = n < E ? (float)b3[n] : 0.0f;
        }
    }
}

}  // namespace k3tc

size_t score_tc_net_bytes(int E) {
    const int KB1 = (2 * E + 63) / 64, N3 = (E + 15) / 16 * 16;
    return (size_t)(KB1 + 2) * k3tc::NPART * k3tc::KBLK + (size_t)2 * k3tc::NPART * N3 * k3tc::ROWB;
}
int score_tc_bias_stride(int E) { return 4 * k3tc::H + (E + 15) / 16 * 16 + k3tc::NSCALE; }

bool score_tc_eligible(const DevTrace &tr, int H) {
    return tr.uniform && H == k3tc::H && (tr.E == 8 || tr.E == 16 || tr.E == 32 || tr.E == 64 || tr.E == 128) &&
           tr.K <= 16 && tr.total_events < (1ll << 31);
}

static int g_num_sms = 0;

template <int E, int GROUPS, bool TA = false>
static int set_smem() {
    return cudaFuncSetAttribute(k3tc::k_score_tc<E, GROUPS, TA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                k3tc::Shape<GROUPS, E, TA>::SMEM) == cudaSuccess ? 0 : -1;
}

int preload_score_tc() {
    if (set_smem<8, 3>() || set_smem<16, 3>() || set_smem<32, 3>() || set_smem<64, 3>() || set_smem<8, 2>() ||
        set_smem<16, 2>() || set_smem<32, 2>() || set_smem<64, 2>() || set_smem<128, 2>() ||
        set_smem<8, 2, true>() || set_smem<16, 2, true>() || set_smem<32, 2, true>() || set_smem<64, 2, true>() ||
        set_smem<128, 2, true>())
        return -1;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    return 0;
}

template <int E, int GROUPS, bool TA = false>
static void launch_tc(const k3tc::Params &P, cudaStream_t s) {
    using S = k3tc::Shape<GROUPS, E, TA>;
    const int sms = g_num_sms > 0 ? g_num_sms : 148;
    const unsigned grid = (unsigned)std::min<int64_t>(sms, (P.n_tiles + GROUPS - 1) / GROUPS);
    k3tc::k_score_tc<E, GROUPS, TA><<<grid, S::THREADS, S::SMEM, s>>>(P);
}

template <int E>
static void launch_variant(const k3tc::Params &P, int variant, cudaStream_t s) {
    if (variant == 1) launch_tc<E, 2, true>(P, s);
    else if (variant == 2) launch_tc<E, 2>(P, s);
    else launch_tc<E, 3>(P, s);
}

// Launches: weight scales + images, then the tensor-core scorer over every
// 128-event tile (ranks + flag lists).  snaps: K3 snapshots (launch_score_prep).
// groups (MCB_TUNE_K3_GROUPS): 3 or 2 epilogue groups with the operands in
// shared memory, 1 = two groups with the operands in TMEM; E = 128 always
// runs 2 groups, with the operands in TMEM unless groups == 2.
int launch_score_tc(const DevTrace &tr, const double *params, int num_nets, const int32_t *snaps, uint8_t *wimg,
                    float *bias, uint8_t *ranks, float tau, int32_t *flag_cnt, int32_t *flag_list, int64_t bucket_cap,
                    unsigned long long *stats, float *dbg_scores, int groups, cudaStream_t s, bool prep,
                    int64_t ev_base) {
    using namespace k3tc;
    const int E = tr.E;
    const int KB1 = (2 * E + 63) / 64, N3 = (E + 15) / 16 * 16;
    const int64_t net_bytes = (int64_t)score_tc_net_bytes(E);
    const int bstride = score_tc_bias_stride(E);
    if (prep) {   // weight images + flag lists (once per call; trace pieces reuse them)
        k_wscale<<<num_nets * 3, 256, 0, s>>>(params, E, N3, bias, bstride);
        const int64_t chunks = ((int64_t)H * KB1 * 8 + (int64_t)H * 16 + (int64_t)N3 * 16) * num_nets;
        const unsigned blocks = (unsigned)std::min<int64_t>((chunks + 255) / 256, 4096);
        k_prep_tc<<<blocks, 256, 0, s>>>(params, E, num_nets, KB1, N3, net_bytes, wimg, bias, bstride);
        cudaMemsetAsync(flag_cnt, 0, sizeof(int32_t) * num_nets, s);
    }
    Params P;
    P.tr = tr;
    P.wimg = wimg;
    P.net_bytes = net_bytes;
    P.bias = bias;
    P.bias_stride = bstride;
    P.num_nets = num_nets;
    P.N3 = N3;
    P.KB1 = KB1;
    P.P1 = (KB1 + 1) / 2;
    P.tpc = (tr.T + BM - 1) / BM;
    P.tpc32 = (tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
    P.n_tiles = tr.n_chains * P.tpc;
    P.snaps = snaps;
    P.ranks = ranks;
    P.tau = tau;
    P.flag_cnt = flag_cnt;
    P.flag_list = flag_list;
    P.bucket_cap = bucket_cap;
    P.stats = stats;
    P.dbg_scores = dbg_scores;
    P.ev_base = ev_base;
    if (P.n_tiles == 0) return 3;
    switch (E) {
        case 8: launch_variant<8>(P, groups, s); break;
        case 16: launch_variant<16>(P, groups, s); break;
        case 32: launch_variant<32>(P, groups, s); break;
        case 64: launch_variant<64>(P, groups, s); break;
        default:   // two groups (84 KB of score staging each): operands in TMEM (6 % faster), or smem
            if (groups == 2) launch_tc<128, 2>(P, s);
            else launch_tc<128, 2, true>(P, s);
            break;
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        char b[160];
        snprintf(b, sizeof b, "k_score_tc launch (E = %d, variant %d): %s", E, groups, cudaGetErrorString(e));
        mcb_set_error(MCB_ERR_CUDA, b);
        return -1;
    }
    return 3;
}
