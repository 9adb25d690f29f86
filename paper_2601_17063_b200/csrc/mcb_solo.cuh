// Register-resident replay step for caches of num_experts <= 16 (one thread
// per cache instance).  Shared by the whole-chain kernel (k_replay_solo) and
// the segmented speculative replay (mcb_segment.cu) so both execute the
// identical per-access arithmetic.
//
// Semantics: SURVEY.md Appendix A (S7, S9, S11) / policies.py:95-214,
// mlpolicy.py:15-26, engine.py:229-257 (pinning), engine.py:266-297
// (refetch).  Every policy's victim is the argmin over resident \ pinned of
// a packed (key << SH | expert id) word; the keys depend on
// the trace only, so two cache states replaying the same stretch of trace
// share them.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mcb_kernels.cuh"

enum { POL_LRU = 0, POL_LFU = 1, POL_BELADY = 2, POL_ML = 3, POL_FIFO = 4, POL_ARC = 5, POL_LECAR = 6 };

#define SOLO_WMAX 7                       // largest refetch window of the solo kernels
#define FULL_MASK_W 0xFFFFFFFFu
#define MCB_HASH_MUL 0x100000001B3ull     // poly hash: h = h * MUL + code + 1 (mod 2^64)

__device__ __forceinline__ uint64_t poly16(uint64_t h, uint32_t code) {
    return h * MCB_HASH_MUL + (uint64_t)code + 1ull;
}

__device__ __forceinline__ uint64_t pow_mul(uint64_t e) {   // MCB_HASH_MUL^e mod 2^64
    uint64_t r = 1ull, b = MCB_HASH_MUL;
    while (e) {
        if (e & 1ull) r *= b;
        b *= b;
        e >>= 1;
    }
    return r;
}

__device__ __forceinline__ uint32_t sel4(const uint4 &v, uint32_t i) {
    uint32_t r = v.x;
    r = i == 1 ? v.y : r;
    r = i == 2 ? v.z : r;
    r = i == 3 ? v.w : r;
    return r;
}

__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int EM>
struct Solo {
    static constexpr int SH = EM == 8 ? 3 : 4;                 // id bits in a packed key
    static constexpr uint32_t KMAX = (1u << (32 - SH)) - 1u;   // keys must stay below this
};

// Per-instance cache state.  The resident count is popc(res) (a miss that
// does not evict adds one expert, an eviction swaps one for one).  Refetch
// without per-expert bookkeeping: ring[i] holds the experts evicted at decode
// index dec - i (i = 0..W); a victim's first access after its eviction is a
// miss, so at a miss of x, x was evicted within the window iff its bit is in
// some ring slot; its bits are cleared at that miss and the ring shifts when
// the decode index advances (== _refetch_rate's next-access test).
template <int WMAX>
struct SState {
    uint32_t res;
    uint32_t ring_or;
    uint32_t ring[WMAX + 1];
};

template <int WMAX>
__device__ __forceinline__ void sstate_clear(SState<WMAX> &S) {
    S.res = 0u;
    S.ring_or = 0u;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) S.ring[s] = 0u;
}

struct SCount {
    uint32_t misses, nev, refc;
};

// One access of expert x (bit = 1 << x) against state S.  pk[] are the packed
// keys after this access's key update, pin the experts already accessed in
// this decode event, valid the selectable experts (ML: rank != 0).
// Branch-free: the would-be victim is always computed (register min-tree)
// and applied under a predicate.  Returns the outcome code (MCB_OUT_HIT,
// MCB_OUT_MISS or the victim id); *miss is set for the event's miss count.
template <int EM, int WMAX>
__device__ __forceinline__ uint32_t sstep(SState<WMAX> &S, const uint32_t (&pk)[EM], uint32_t bit, uint32_t pin,
                                          uint32_t valid, uint32_t C, SCount &n, bool &stuck, uint32_t &miss_out) {
    const uint32_t cand = S.res & ~pin & valid;
    uint32_t t[EM];
#pragma unroll
    for (int s = 0; s < EM; ++s) t[s] = ((cand >> s) & 1u) ? pk[s] : ~0u;
#pragma unroll
    for (int w = EM / 2; w >= 1; w /= 2)
#pragma unroll
        for (int s = 0; s < w; ++s) t[s] = min(t[s], t[s + w]);
    const bool hit = (S.res & bit) != 0u;
    const bool miss = !hit;
    const bool full = (uint32_t)__popc(S.res) >= C;
    const bool evict = miss && full;
    stuck |= evict && t[0] == ~0u;
    const uint32_t v = t[0] & (uint32_t)(EM - 1);
    const uint32_t vbit = evict ? (1u << v) : 0u;
    S.res = (S.res & ~vbit) | bit;
    n.misses += miss ? 1u : 0u;
    n.nev += evict ? 1u : 0u;
    const uint32_t mbit = miss ? bit : 0u;
    n.refc += (mbit & S.ring_or) ? 1u : 0u;
    S.ring_or = (S.ring_or & ~mbit) | vbit;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) S.ring[s] &= ~mbit;
    S.ring[0] |= vbit;
    miss_out = miss ? 1u : 0u;
    return hit ? MCB_OUT_HIT : (evict ? v : MCB_OUT_MISS);
}

// decode index advances: slot i now holds evictions from dec - i
template <int WMAX>
__device__ __forceinline__ void sstate_next_decode(SState<WMAX> &S, int W) {
#pragma unroll
    for (int s = WMAX; s >= 1; --s) S.ring[s] = S.ring[s - 1];
    S.ring[0] = 0u;
    uint32_t o = 0u;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) o |= (s <= W) ? S.ring[s] : 0u;
    S.ring_or = o;
}

// state equality as far as the future is concerned (ring slots > W are dead)
template <int WMAX>
__device__ __forceinline__ bool sstate_equal(const SState<WMAX> &A, const SState<WMAX> &B, int W) {
    uint32_t d = A.res ^ B.res;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) d |= (s <= W) ? (A.ring[s] ^ B.ring[s]) : 0u;
    return d == 0u;
}

// Lane-cooperative stream reader for a group of G lanes: the group holds a
// chunk of G consecutive 32-bit words (one per lane) and the next chunk in
// flight; get() broadcasts a word by shuffle (whole group, monotone words).
template <int G>
struct U32Stream {
    // 4*G-byte (or G-word) chunks of a stream held one u32 per lane, next
    // chunk prefetched while the current one is consumed.
    const uint32_t *base;
    int64_t limit_words;  // words readable
    int64_t chunk;        // index of the chunk held in `cur`
    uint32_t cur, nxt;
    __device__ __forceinline__ uint32_t load(int64_t ch, int glane) const {
        const int64_t wi = ch * G + glane;
        return wi < limit_words ? __ldg(base + wi) : 0u;
    }
    __device__ __forceinline__ void init(const void *p, int64_t words, int64_t first_word, int glane) {
        base = (const uint32_t *)p;
        limit_words = words;
        chunk = first_word / G;
        cur = load(chunk, glane);
        nxt = load(chunk + 1, glane);
    }
    // word index -> value (must be called by the whole group, monotone words)
    __device__ __forceinline__ uint32_t get(int64_t word, int glane, int gbase, unsigned gmask) {
        const int64_t ch = word / G;
        if (ch != chunk) {
            if (ch == chunk + 1) {
                cur = nxt;
            } else {
                cur = load(ch, glane);
            }
            chunk = ch;
            nxt = load(ch + 1, glane);
        }
        return __shfl_sync(gmask, cur, gbase + (int)(word - ch * G));
    }
};

// Sequential reader of a chain's uint8 id stream, 16 ids per vector load
// with the next vector in flight and an L2 prefetch 512 B ahead.
struct IdReader {
    const uint4 *p;
    int64_t ch;
    int64_t end;   // absolute access index bound (for prefetch)
    uint4 cur, nxt;
    __device__ __forceinline__ void init(const uint8_t *acc, int64_t a, int64_t a_end) {
        p = (const uint4 *)acc;
        ch = a >> 4;
        end = a_end;
        cur = __ldg(p + ch);
        nxt = __ldg(p + ch + 1);
    }
    __device__ __forceinline__ uint32_t get(int64_t a) {
        if ((a >> 4) != ch) {
            ++ch;
            cur = nxt;
            nxt = __ldg(p + ch + 1);
            if ((ch & 7) == 0 && ((ch + 32) << 4) < end) prefetch_l2(p + ch + 32);
        }
        return (sel4(cur, (uint32_t)(a >> 2) & 3u) >> (8u * (uint32_t)(a & 3))) & 0xFFu;
    }
};

// Sequential reader of next_pos (4 per vector load).
struct NextReader {
    const uint4 *p;
    int64_t ch;
    int64_t end;
    uint4 cur, nxt;
    __device__ __forceinline__ void init(const uint32_t *np, int64_t a, int64_t a_end) {
        p = (const uint4 *)np;
        ch = a >> 2;
        end = a_end;
        cur = __ldg(p + ch);
        nxt = __ldg(p + ch + 1);
    }
    __device__ __forceinline__ uint32_t get(int64_t a) {
        if ((a >> 2) != ch) {
            ++ch;
            cur = nxt;
            nxt = __ldg(p + ch + 1);
            if ((ch & 7) == 0 && ((ch + 64) << 2) < end) prefetch_l2(p + ch + 64);
        }
        return sel4(cur, (uint32_t)a & 3u);
    }
};

// The trace-determined key of the accessed expert x at chain position pos
// (absolute access index a), applied to the packed key array.  LFU counts
// are carried in pk itself.
template <int EM, int POL>
__device__ __forceinline__ void solo_key_update(uint32_t (&pk)[EM], uint32_t x, uint32_t bit, uint32_t pos,
                                                uint32_t np) {
    constexpr int SH = Solo<EM>::SH;
    constexpr uint32_t KMAX = Solo<EM>::KMAX;
    uint32_t nk = 0;
    if (POL == POL_LRU) nk = (pos << SH) | x;
    if (POL == POL_LFU) {
        uint32_t cur = 0;
#pragma unroll
        for (int s = 0; s < EM; ++s) cur |= ((bit >> s) & 1u) ? pk[s] : 0u;
        nk = cur + (1u << SH);
    }
    if (POL == POL_BELADY) nk = ((np == MCB_NEXT_INF ? 0u : KMAX - np) << SH) | x;   // farthest next use first
    if (POL == POL_FIFO || POL == POL_ARC || POL == POL_LECAR) return;   // state-dependent (own step functions)
    if (POL != POL_ML) {
#pragma unroll
        for (int s = 0; s < EM; ++s) pk[s] = ((bit >> s) & 1u) ? nk : pk[s];
    }
}

// FIFO (policies.py:152-168): the key is the arrival order, set when x is
// inserted (a miss); positions grow with the arrival clock, so (pos, id)
// orders like the reference's (arrival, id).  State-dependent, so FIFO runs
// in the whole-chain kernels only.
template <int EM>
__device__ __forceinline__ void solo_fifo_insert(uint32_t (&pk)[EM], uint32_t x, uint32_t bit, uint32_t pos,
                                                 uint32_t miss) {
    const uint32_t nk = (pos << Solo<EM>::SH) | x;
#pragma unroll
    for (int s = 0; s < EM; ++s) pk[s] = (miss && ((bit >> s) & 1u)) ? nk : pk[s];
}

// ARC (policies.py:217-302) for num_experts <= 16: the four OrderedDicts as
// expert masks (T1, T2 resident; B1, B2 ghosts) plus each expert's insertion
// clock, so a list's LRU end is its smallest clock; the adaptation target p
// is a float64 updated with the reference's operations.
template <int EM>
struct ArcState {
    uint32_t t1, t2, b1, b2;
    uint32_t ord[EM];
    uint32_t clock;
    double p;
};

template <int EM>
__device__ __forceinline__ void arc_clear(ArcState<EM> &a) {
    a.t1 = a.t2 = a.b1 = a.b2 = 0u;
#pragma unroll
    for (int s = 0; s < EM; ++s) a.ord[s] = 0u;
    a.clock = 0u;
    a.p = 0.0;
}

// LRU end (smallest clock) of the experts in mask; EM if empty
template <int EM>
__device__ __forceinline__ uint32_t arc_lru(const ArcState<EM> &a, uint32_t mask) {
    constexpr int SH = Solo<EM>::SH;
    uint32_t t = ~0u;
#pragma unroll
    for (int s = 0; s < EM; ++s) t = ((mask >> s) & 1u) ? min(t, (a.ord[s] << SH) | (uint32_t)s) : t;
    return t == ~0u ? (uint32_t)EM : (t & (uint32_t)(EM - 1));
}

// move expert v to the MRU end of the list `which` (0 T1, 1 T2, 2 B1, 3 B2); 4 = remove
template <int EM>
__device__ __forceinline__ void arc_put(ArcState<EM> &a, uint32_t v, int which) {
    const uint32_t b = 1u << v;
    a.t1 &= ~b;
    a.t2 &= ~b;
    a.b1 &= ~b;
    a.b2 &= ~b;
    if (which == 0) a.t1 |= b;
    if (which == 1) a.t2 |= b;
    if (which == 2) a.b1 |= b;
    if (which == 3) a.b2 |= b;
    if (which == 4) return;   // removal: no new position
#pragma unroll
    for (int s = 0; s < EM; ++s) a.ord[s] = (s == (int)v) ? a.clock : a.ord[s];
    ++a.clock;
}

// _replace (policies.py:236-254): victim, or EM when every resident is pinned
template <int EM>
__device__ __forceinline__ uint32_t arc_replace(ArcState<EM> &a, bool in_b2, uint32_t pin) {
    const int n1 = __popc(a.t1);
    const bool use_t1 = n1 >= 1 && ((double)n1 > a.p || (in_b2 && (double)n1 == a.p));
    uint32_t v = arc_lru<EM>(a, (use_t1 ? a.t1 : a.t2) & ~pin);
    bool from_t1 = use_t1;
    if (v == (uint32_t)EM) {
        v = arc_lru<EM>(a, (use_t1 ? a.t2 : a.t1) & ~pin);
        from_t1 = !use_t1;
    }
    if (v != (uint32_t)EM) arc_put<EM>(a, v, from_t1 ? 2 : 3);
    return v;
}

// ARCPolicy.access (policies.py:256-302) + the engine's accounting on S
// (resident mask, refetch ring) exactly as sstep: returns the outcome code.
template <int EM, int WMAX>
__device__ __forceinline__ uint32_t sstep_arc(SState<WMAX> &S, ArcState<EM> &a, uint32_t x, uint32_t bit,
                                              uint32_t pin, uint32_t C, SCount &n, bool &stuck, uint32_t &miss_out) {
    const bool hit = ((a.t1 | a.t2) & bit) != 0u;
    miss_out = hit ? 0u : 1u;
    if (hit) {
        arc_put<EM>(a, x, 1);
        return MCB_OUT_HIT;
    }
    uint32_t v = (uint32_t)EM;   // victim (EM: none)
    bool none_left = false;
    const bool full = (uint32_t)__popc(a.t1 | a.t2) >= C;
    if (a.b1 & bit) {
        double q = (double)__popc(a.b2) / (double)__popc(a.b1);
        q = q < 1.0 ? 1.0 : q;
        const double np = a.p + q;
        a.p = (double)C <= np ? (double)C : np;
        if (full) { v = arc_replace<EM>(a, false, pin); none_left = v == (uint32_t)EM; }
        arc_put<EM>(a, x, 1);
    } else if (a.b2 & bit) {
        double q = (double)__popc(a.b1) / (double)__popc(a.b2);
        q = q < 1.0 ? 1.0 : q;
        const double np = a.p - q;
        a.p = 0.0 >= np ? 0.0 : np;
        if (full) { v = arc_replace<EM>(a, true, pin); none_left = v == (uint32_t)EM; }
        arc_put<EM>(a, x, 1);
    } else {
        const uint32_t n1 = (uint32_t)__popc(a.t1);
        const uint32_t l1 = n1 + (uint32_t)__popc(a.b1);
        if (l1 == C) {
            if (n1 < C) {
                arc_put<EM>(a, arc_lru<EM>(a, a.b1), 4);
                if ((uint32_t)__popc(a.t1 | a.t2) >= C) { v = arc_replace<EM>(a, false, pin); none_left = v == (uint32_t)EM; }
            } else {   // B1 empty, T1 full: drop T1's LRU without a ghost entry
                v = arc_lru<EM>(a, a.t1 & ~pin);
                none_left = v == (uint32_t)EM;
                if (!none_left) arc_put<EM>(a, v, 4);
            }
        } else if (l1 < C) {
            const uint32_t total = l1 + (uint32_t)__popc(a.t2) + (uint32_t)__popc(a.b2);
            if (total >= C) {
                if (total == 2 * C) arc_put<EM>(a, arc_lru<EM>(a, a.b2), 4);
                if ((uint32_t)__popc(a.t1 | a.t2) >= C) { v = arc_replace<EM>(a, false, pin); none_left = v == (uint32_t)EM; }
            }
        }
        arc_put<EM>(a, x, 0);
    }
    stuck |= none_left;
    const bool evict = v != (uint32_t)EM;
    const uint32_t vbit = evict ? (1u << v) : 0u;
    S.res = a.t1 | a.t2;
    ++n.misses;
    n.nev += evict ? 1u : 0u;
    n.refc += (bit & S.ring_or) ? 1u : 0u;
    S.ring_or = (S.ring_or & ~bit) | vbit;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) S.ring[s] &= ~bit;
    S.ring[0] |= vbit;
    return evict ? v : MCB_OUT_MISS;
}

// LeCaR (policies.py:305-395) for num_experts <= 16: the LRU stamps and LFU
// counts as packed (key << SH | id) words, the two ghost lists as masks plus
// each ghost's eviction position (positions grow, so a list's oldest entry
// is its smallest position), the weights as float64 and the instance's
// eviction count, which indexes the shared random() stream.
template <int EM>
struct LecarState {
    uint32_t pl[EM];    // (stamp << SH) | id   (_stamp, set at every access)
    uint32_t pf[EM];    // (freq << SH) | id    (_freq, reset at start_sequence)
    uint32_t gpos[EM];  // eviction position of a ghost entry
    uint32_t gl, gf;    // _ghost_lru / _ghost_lfu membership
    uint32_t k;         // evictions so far = random() draws consumed
    double wl, wf;      // weights (w_lru, w_lfu)
};

template <int EM>
__device__ __forceinline__ void lecar_clear(LecarState<EM> &a) {
#pragma unroll
    for (int s = 0; s < EM; ++s) { a.pl[s] = (uint32_t)s; a.pf[s] = (uint32_t)s; a.gpos[s] = 0u; }
    a.gl = a.gf = 0u;
    a.k = 0u;
    a.wl = 0.5;
    a.wf = 0.5;
}

template <int EM>
__device__ __forceinline__ void lecar_new_sequence(LecarState<EM> &a) {   // start_sequence (policies.py:351-352)
#pragma unroll
    for (int s = 0; s < EM; ++s) a.pf[s] = (uint32_t)s;
}

// lecar_update (policies.py:305-327) with the host-made factor
// f = exp(learning_rate * discount**elapsed); no contraction into FMAs.
__device__ __forceinline__ void lecar_reward(double &wl, double &wf, bool ghost_lru, double f) {
    if (ghost_lru) wf = __dmul_rn(wf, f);
    else wl = __dmul_rn(wl, f);
    const double total = __dadd_rn(wl, wf);
    wl = __ddiv_rn(wl, total);
    wf = __ddiv_rn(wf, total);
}

__device__ __forceinline__ double lecar_factor(const ReplayParams &P, int cap_i, uint32_t elapsed) {
    return (int64_t)elapsed < P.lecar_tlen ? __ldg(P.lecar_f + (int64_t)cap_i * P.lecar_tlen + elapsed) : 1.0;
}

// LeCaRPolicy access (CachePolicy.access, policies.py:95-107, with the LeCaR
// hooks) + the engine's accounting on S exactly as sstep: the outcome code.
template <int EM, int WMAX>
__device__ __forceinline__ uint32_t sstep_lecar(SState<WMAX> &S, LecarState<EM> &a, const ReplayParams &P,
                                                int cap_i, uint32_t x, uint32_t bit, uint32_t pos, uint32_t pin,
                                                uint32_t C, SCount &n, bool &stuck, uint32_t &miss_out) {
    constexpr int SH = Solo<EM>::SH;
    const bool hit = (S.res & bit) != 0u;
    // _on_hit / _on_miss: freq += 1; _on_hit / _on_insert: stamp = position
    // (x is never a victim candidate of its own miss, so both apply up front)
#pragma unroll
    for (int s = 0; s < EM; ++s) {
        const bool me = (bit >> s) & 1u;
        a.pf[s] = me ? a.pf[s] + (1u << SH) : a.pf[s];
        a.pl[s] = me ? ((pos << SH) | (uint32_t)s) : a.pl[s];
    }
    miss_out = hit ? 0u : 1u;
    if (hit) return MCB_OUT_HIT;
    if ((a.gl | a.gf) & bit) {   // ghost hit: regret update (policies.py:358-367)
        uint32_t gp = 0u;
#pragma unroll
        for (int s = 0; s < EM; ++s) gp |= ((bit >> s) & 1u) ? a.gpos[s] : 0u;
        lecar_reward(a.wl, a.wf, (a.gl & bit) != 0u, lecar_factor(P, cap_i, pos - gp));
        a.gl &= ~bit;
        a.gf &= ~bit;
    }
    uint32_t v = (uint32_t)EM;
    if ((uint32_t)__popc(S.res) >= C) {
        const uint32_t cand = S.res & ~pin;
        if (!cand) {
            stuck = true;
        } else {
            // _choose_victim (policies.py:379-395)
            const double u = __ldg(P.lecar_u + a.k);
            ++a.k;
            const bool use_lru = u < a.wl;
            uint32_t t = ~0u;
#pragma unroll
            for (int s = 0; s < EM; ++s) t = ((cand >> s) & 1u) ? min(t, use_lru ? a.pl[s] : a.pf[s]) : t;
            v = t & (uint32_t)(EM - 1);
            const uint32_t vb = 1u << v;
#pragma unroll
            for (int s = 0; s < EM; ++s) a.gpos[s] = s == (int)v ? pos : a.gpos[s];
            uint32_t g = (use_lru ? a.gl : a.gf) | vb;
            if ((uint32_t)__popc(g) > C) {   // drop the oldest ghost (popitem(last=False))
                uint32_t o = ~0u;
#pragma unroll
                for (int s = 0; s < EM; ++s) o = ((g >> s) & 1u) ? min(o, (a.gpos[s] << SH) | (uint32_t)s) : o;
                g &= ~(1u << (o & (uint32_t)(EM - 1)));
            }
            if (use_lru) a.gl = g;
            else a.gf = g;
        }
    }
    const bool evict = v != (uint32_t)EM;
    const uint32_t vbit = evict ? (1u << v) : 0u;
    S.res = (S.res & ~vbit) | bit;
    ++n.misses;
    n.nev += evict ? 1u : 0u;
    n.refc += (bit & S.ring_or) ? 1u : 0u;
    S.ring_or = (S.ring_or & ~bit) | vbit;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) S.ring[s] &= ~bit;
    S.ring[0] |= vbit;
    return evict ? v : MCB_OUT_MISS;
}

// ML: packed keys and the selectable mask from one event's rank row
// (argmax score == argmin (256 - rank); rank 0 = NaN / -inf, never selected).
template <int EM>
__device__ __forceinline__ void solo_ml_keys(uint32_t (&pk)[EM], uint32_t &valid, const uint32_t (&rrow)[EM]) {
    constexpr int SH = Solo<EM>::SH;
    valid = 0u;
#pragma unroll
    for (int s = 0; s < EM; ++s) {
        pk[s] = ((256u - rrow[s]) << SH) | (uint32_t)s;
        valid |= (rrow[s] != 0u ? 1u : 0u) << s;
    }
}

// One event's rank row (E bytes).  Full rows (E == EM: rows are 8- / 16-byte
// aligned in the engine's rank buffer) are one vector load.
template <int EM>
__device__ __forceinline__ void load_rank_row(uint32_t (&rrow)[EM], const uint8_t *row, int E) {
    if (E == EM) {
        uint32_t w[EM / 4];
        if constexpr (EM == 8) {
            const uint2 v = __ldcg((const uint2 *)row);
            w[0] = v.x;
            w[1] = v.y;
        } else {
            const uint4 v = __ldcg((const uint4 *)row);
            w[0] = v.x;
            w[1] = v.y;
            w[2] = v.z;
            w[3] = v.w;
        }
#pragma unroll
        for (int s = 0; s < EM; ++s) rrow[s] = (w[s >> 2] >> (8 * (s & 3))) & 0xFFu;
        return;
    }
#pragma unroll
    for (int s = 0; s < EM; ++s) rrow[s] = s < E ? (uint32_t)__ldcg(row + s) : 0u;
}

// Exact fold of cnt[m] additions of lut[m] (any order within the run) onto S
// when the running sum provably stays in S's binade and no addend is a
// rounding tie there; false = use the sequential fold.
__device__ __forceinline__ bool fold_hist_fast(double &S, const uint32_t *cnt, int nb, const double *lut) {
    if (!(S > 0.0)) return false;
    int ex;
    frexp(S, &ex);                                             // S in [2^(ex-1), 2^ex), ulp 2^(ex-53)
    const uint64_t two52 = 1ull << 52, two53 = 1ull << 53;
    const uint64_t s_int = (uint64_t)scalbn(S, 53 - ex);       // in [2^52, 2^53)
    uint64_t tot = 0;
    for (int m = 0; m < nb; ++m) {
        const uint64_t c = cnt[m];
        if (!c) continue;
        const double qf = scalbn(lut[m], 53 - ex);             // exact (power-of-two scaling)
        if (!(qf < (double)two52)) return false;
        const double fl = floor(qf);
        const double fr = qf - fl;
        if (fr == 0.5) return false;                           // tie: depends on the running sum's parity
        const uint64_t q = (uint64_t)fl + (fr > 0.5 ? 1ull : 0ull);
        if (__umul64hi(c, q)) return false;
        const uint64_t p = c * q;
        if (p >= two52) return false;
        tot += p;
        if (tot >= two52) return false;
    }
    if (s_int + tot >= two53) return false;                    // would reach the next binade
    S = scalbn((double)(s_int + tot), ex - 53);
    return true;
}

// sequential float64 fold of events [ev, ev1) from the stored miss counts
__device__ __forceinline__ double fold_codes(double dlat, const uint8_t *codes, int64_t ev, int64_t ev1,
                                             const double *lut) {
    while (ev < ev1 && (ev & 15)) dlat = __dadd_rn(dlat, lut[__ldg(codes + ev++)]);
    const uint4 *v = (const uint4 *)(codes + ev);
    const int64_t nv = (ev1 - ev) >> 4;
    for (int64_t i = 0; i < nv; ++i) {
        const uint4 cur = __ldg(v + i);
        const uint32_t w[4] = {cur.x, cur.y, cur.z, cur.w};
        double a[16];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int b = 0; b < 4; ++b) a[4 * q + b] = lut[(w[q] >> (8 * b)) & 0xFFu];
#pragma unroll
        for (int q = 0; q < 16; ++q) dlat = __dadd_rn(dlat, a[q]);
    }
    ev += nv << 4;
    while (ev < ev1) dlat = __dadd_rn(dlat, lut[__ldg(codes + ev++)]);
    return dlat;
}
