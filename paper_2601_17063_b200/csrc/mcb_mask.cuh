// Expert masks for up to 128 experts held by one thread: uint64_t for
// num_experts <= 64, two words (M128) above.  Shared by the thread-per-
// instance replay (mcb_wide.cu) and the thread speculation of the wide
// segmented replay (mcb_segment_warp.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mm {

struct M128 {
    uint64_t lo, hi;
};
__device__ __forceinline__ M128 operator&(M128 a, M128 b) { return {a.lo & b.lo, a.hi & b.hi}; }
__device__ __forceinline__ M128 operator|(M128 a, M128 b) { return {a.lo | b.lo, a.hi | b.hi}; }
__device__ __forceinline__ M128 operator~(M128 a) { return {~a.lo, ~a.hi}; }
__device__ __forceinline__ bool any(M128 a) { return (a.lo | a.hi) != 0ull; }
__device__ __forceinline__ bool any(uint64_t a) { return a != 0ull; }
__device__ __forceinline__ int popc(M128 a) { return __popcll(a.lo) + __popcll(a.hi); }
__device__ __forceinline__ int popc(uint64_t a) { return __popcll(a); }
template <typename M> __device__ __forceinline__ M zero();
template <> __device__ __forceinline__ uint64_t zero<uint64_t>() { return 0ull; }
template <> __device__ __forceinline__ M128 zero<M128>() { return {0ull, 0ull}; }
template <typename M> __device__ __forceinline__ M bit_of(uint32_t x);
template <> __device__ __forceinline__ uint64_t bit_of<uint64_t>(uint32_t x) { return 1ull << x; }
template <> __device__ __forceinline__ M128 bit_of<M128>(uint32_t x) {
    return x < 64 ? M128{1ull << x, 0ull} : M128{0ull, 1ull << (x - 64)};
}
template <typename M> __device__ __forceinline__ M first_n(int E);   // experts 0 .. E-1
template <> __device__ __forceinline__ uint64_t first_n<uint64_t>(int E) { return E >= 64 ? ~0ull : ((1ull << E) - 1ull); }
template <> __device__ __forceinline__ M128 first_n<M128>(int E) {
    return E >= 128 ? M128{~0ull, ~0ull}
                    : (E >= 64 ? M128{~0ull, E == 64 ? 0ull : ((1ull << (E - 64)) - 1ull)}
                               : M128{(1ull << E) - 1ull, 0ull});
}
__device__ __forceinline__ bool test(uint64_t m, uint32_t x) { return (m >> x) & 1ull; }
__device__ __forceinline__ bool test(M128 m, uint32_t x) { return x < 64 ? ((m.lo >> x) & 1ull) : ((m.hi >> (x - 64)) & 1ull); }
// lowest set bit of a non-empty mask, removed
__device__ __forceinline__ int pop_first(uint64_t &m) {
    const int s = __ffsll((long long)m) - 1;
    m &= m - 1ull;
    return s;
}
__device__ __forceinline__ int pop_first(M128 &m) {
    if (m.lo) {
        const int s = __ffsll((long long)m.lo) - 1;
        m.lo &= m.lo - 1ull;
        return s;
    }
    const int s = __ffsll((long long)m.hi) - 1;
    m.hi &= m.hi - 1ull;
    return 64 + s;
}

// 4 x 32-bit words (bit e % 32 of word e / 32) <-> mask
__device__ __forceinline__ void to_words(uint64_t m, uint32_t *w) {
    w[0] = (uint32_t)m; w[1] = (uint32_t)(m >> 32); w[2] = 0u; w[3] = 0u;
}
__device__ __forceinline__ void to_words(M128 m, uint32_t *w) {
    w[0] = (uint32_t)m.lo; w[1] = (uint32_t)(m.lo >> 32); w[2] = (uint32_t)m.hi; w[3] = (uint32_t)(m.hi >> 32);
}
template <typename M> __device__ __forceinline__ M from_words(const uint32_t *w);
template <> __device__ __forceinline__ uint64_t from_words<uint64_t>(const uint32_t *w) {
    return (uint64_t)w[0] | ((uint64_t)w[1] << 32);
}
template <> __device__ __forceinline__ M128 from_words<M128>(const uint32_t *w) {
    return {(uint64_t)w[0] | ((uint64_t)w[1] << 32), (uint64_t)w[2] | ((uint64_t)w[3] << 32)};
}

// Minimum packed key over the experts of a candidate mask (keys column-major
// per thread, stride BS): 32-bit words,
// highest set bit first (one FLO per candidate), two candidates per trip so
// two key loads are in flight.
template <int BS>
__device__ __forceinline__ uint32_t min_key_word(uint32_t w, uint32_t best, const uint32_t *sk) {
    while (w) {
        const int i = 31 - __clz(w);
        w ^= 1u << i;
        uint32_t k = sk[i * BS];
        if (w) {
            const int i2 = 31 - __clz(w);
            w ^= 1u << i2;
            k = min(k, sk[i2 * BS]);
        }
        best = min(best, k);
    }
    return best;
}
template <int BS>
__device__ __forceinline__ uint32_t min_key(uint64_t cand, const uint32_t *sk) {
    return min_key_word<BS>((uint32_t)(cand >> 32), min_key_word<BS>((uint32_t)cand, ~0u, sk), sk + 32 * BS);
}
template <int BS>
__device__ __forceinline__ uint32_t min_key(M128 cand, const uint32_t *sk) {
    uint32_t b = min_key_word<BS>((uint32_t)cand.lo, ~0u, sk);
    b = min_key_word<BS>((uint32_t)(cand.lo >> 32), b, sk + 32 * BS);
    b = min_key_word<BS>((uint32_t)cand.hi, b, sk + 64 * BS);
    return min_key_word<BS>((uint32_t)(cand.hi >> 32), b, sk + 96 * BS);
}

// The N smallest packed keys over the experts of a candidate mask, ascending
// in low[] (~0u where there are fewer candidates): one insertion network step
// (2N - 1 min / max) per candidate, two key loads in flight.
template <int N>
__device__ __forceinline__ void insert_low(uint32_t k, uint32_t (&low)[N]) {
#pragma unroll
    for (int q = N - 1; q >= 1; --q) low[q] = min(low[q], max(low[q - 1], k));
    low[0] = min(low[0], k);
}
template <int BS, int N>
__device__ __forceinline__ void lowest_keys_word(uint32_t w, const uint32_t *sk, uint32_t (&low)[N]) {
    while (w) {
        const int i = 31 - __clz(w);
        w ^= 1u << i;
        const uint32_t k = sk[i * BS];
        if (w) {
            const int i2 = 31 - __clz(w);
            w ^= 1u << i2;
            insert_low<N>(sk[i2 * BS], low);
        }
        insert_low<N>(k, low);
    }
}
template <int BS, int N, typename M>
__device__ __forceinline__ void lowest_keys(M cand, const uint32_t *sk, uint32_t (&low)[N]) {
    uint32_t w[4];
    to_words(cand, w);
#pragma unroll
    for (int q = 0; q < N; ++q) low[q] = ~0u;
    lowest_keys_word<BS, N>(w[0], sk, low);
    lowest_keys_word<BS, N>(w[1], sk + 32 * BS, low);
    if (sizeof(M) > 8) {
        lowest_keys_word<BS, N>(w[2], sk + 64 * BS, low);
        lowest_keys_word<BS, N>(w[3], sk + 96 * BS, low);
    }
}

// Highest set bit of a non-empty mask.
__device__ __forceinline__ uint32_t top_bit(uint64_t m) { return 63u - (uint32_t)__clzll((long long)m); }
__device__ __forceinline__ uint32_t top_bit(M128 m) {
    return m.hi ? 127u - (uint32_t)__clzll((long long)m.hi) : 63u - (uint32_t)__clzll((long long)m.lo);
}

// A candidate set in RANK space for one event: bit r - 1 for every candidate
// of rank r >= 1 (rank-0 experts are never selectable), and ord[r - 1] = that
// expert.  Ranks of one event are distinct, so the ML victim (arg-max score,
// mlpolicy.py:15-26) of any subset is ord[top_bit(subset)] -- one FLO per
// evicting miss instead of a scan of the candidates' ranks.
template <typename M>
__device__ __forceinline__ void rank_space_word(uint32_t w, int e0, const uint8_t *row, uint8_t *ord, M &out) {
    while (w) {
        const int i = 31 - __clz(w);
        w ^= 1u << i;
        const uint32_t r = row[e0 + i];
        if (w) {
            const int i2 = 31 - __clz(w);
            w ^= 1u << i2;
            const uint32_t r2 = row[e0 + i2];
            if (r2) {
                out = out | bit_of<M>(r2 - 1u);
                ord[r2 - 1u] = (uint8_t)(e0 + i2);
            }
        }
        if (r) {
            out = out | bit_of<M>(r - 1u);
            ord[r - 1u] = (uint8_t)(e0 + i);
        }
    }
}
template <typename M>
__device__ __forceinline__ M rank_space(M cand, const uint8_t *row, uint8_t *ord) {
    uint32_t w[4];
    to_words(cand, w);
    M out = zero<M>();
    rank_space_word(w[0], 0, row, ord, out);
    rank_space_word(w[1], 32, row, ord, out);
    if (sizeof(M) > 8) {
        rank_space_word(w[2], 64, row, ord, out);
        rank_space_word(w[3], 96, row, ord, out);
    }
    return out;
}
template <typename M>
__device__ __forceinline__ M rank_bit(uint32_t r) {   // rank r >= 1 -> its bit, rank 0 -> none
    return r ? bit_of<M>(r - 1u) : zero<M>();
}

// One event's rank row into a thread's shared-memory row (row stride
// mrow_stride(E), 16-byte aligned): four 16-byte copies for E % 16 == 0, bytes otherwise.
__host__ __device__ __forceinline__ int mrow_stride(int E) { return (E + 31) & ~15; }
__device__ __forceinline__ void copy_rank_row(const uint8_t *src, uint8_t *dst, int E) {
    if ((E & 15) == 0) {
#pragma unroll 2
        for (int q = 0; q < E / 16; ++q) *(uint4 *)(dst + 16 * q) = __ldcg((const uint4 *)src + q);
    } else {
        for (int e = 0; e < E; ++e) dst[e] = __ldcg(src + e);
    }
}

// The same copy issued asynchronously (cp.async.cg, 16 bytes per op, no
// registers), so the next event's row is in flight while this one is used;
// E % 16 == 0 only.  rank_row_wait() before reading the row.
__device__ __forceinline__ void rank_row_async(const uint8_t *src, uint8_t *dst, int E) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    for (int q = 0; q < E / 16; ++q)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + 16 * q), "l"(src + 16 * q) : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void rank_row_wait() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ML keys of one event for a thread's column of shared-memory keys
// (keys[e * 128]): key = (256 - rank) << 7 | e, selectable iff rank != 0
// (mlpolicy.py:15-26).  Rows of a multiple of 16 experts are 16-byte aligned
// and read 16 ranks per load, independent loads in flight together.
template <typename M>
__device__ __forceinline__ M ml_row_keys(const uint8_t *row, int E, uint32_t *sk) {
    M valid = zero<M>();
    if ((E & 15) == 0) {
#pragma unroll 2
        for (int s0 = 0; s0 < E; s0 += 16) {
            const uint4 v = __ldcg((const uint4 *)(row + s0));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint32_t r = (w[q >> 2] >> (8 * (q & 3))) & 0xFFu;
                sk[(s0 + q) * 128] = ((256u - r) << 7) | (uint32_t)(s0 + q);
                if (r != 0u) valid = valid | bit_of<M>((uint32_t)(s0 + q));
            }
        }
        return valid;
    }
    for (int s = 0; s < E; ++s) {
        const uint32_t r = __ldcg(row + s);
        sk[s * 128] = ((256u - r) << 7) | (uint32_t)s;
        if (r != 0u) valid = valid | bit_of<M>((uint32_t)s);
    }
    return valid;
}

}  // namespace mm
