// Segmented speculative replay for 16 < num_experts <= 128 (one warp per
// cache instance), the counterpart of mcb_segment.cu's thread-per-instance
// version.  Same scheme (see mcb_segment.cu): key snapshots every
// MCB_SNAP_EV events, one warp per (instance, segment) replays the segment
// from a guessed state after a warm-up and records start / end state,
// counters, the poly hash and the miss-count histogram; one warp per
// instance then walks the segments carrying the true state, splicing a
// segment whole when the recorded start state equals the true one and
// replaying true and speculative states in lockstep until they coincide
// otherwise.  Results are identical to k_replay's by construction.
//
// Warp state: expert e lives in lane e / EPL, slot e % EPL (as in k_replay);
// per lane the resident bits, refetch ring (evictions of the last W decode
// steps, engine.py:266-297) and the policy keys of its EPL experts.  The
// victim is the lane-local argmin + redux.sync min + ballot for the lowest
// id among equal keys (policies.py:148-214, mlpolicy.py:15-26).
#include <cuda_runtime.h>
#include <stdint.h>

#include "mcb_kernels.cuh"
#include "mcb_mask.cuh"
#include "mcb_solo.cuh"

#define WKEY_SENT 0xFFFFFFFFu
// Warp replay keys are packed (key << WKEY_SH | expert) so that the warp-wide
// minimum names the victim (ties to the smallest id, as before the packing);
// chain-local positions must stay below 2^25 (seg_eligible).
#define WKEY_SH 7
#define WKEY_ID 0x7Fu
#define WKEY_KMAX ((1u << (32 - WKEY_SH)) - 1u)

template <int EPL>
struct WState {
    uint32_t res;                        // this lane's resident slots
    uint32_t ring[SOLO_WMAX + 1];        // this lane's slots evicted at decode index dec - i
    uint32_t ring_or;
    uint32_t count;                      // resident experts (warp-uniform)
};

template <int EPL>
__device__ __forceinline__ void wstate_clear(WState<EPL> &S) {
    S.res = 0u;
    S.ring_or = 0u;
    S.count = 0u;
#pragma unroll
    for (int s = 0; s <= SOLO_WMAX; ++s) S.ring[s] = 0u;
}

// One access of expert x = owner * EPL + slot.  Warp-uniform control flow
// (hit / miss / evict are ballots or uniform counts).  n.misses / n.nev are
// warp-uniform, n.refc counts on the owner lane only.
template <int EPL>
__device__ __forceinline__ uint32_t wstep(WState<EPL> &S, const uint32_t (&key)[EPL], int owner, uint32_t bit,
                                          uint32_t pin, uint32_t valid, uint32_t C, int lane, SCount &n, bool &stuck,
                                          uint32_t &miss_out) {
    const bool mine = lane == owner;
    const bool hit = __ballot_sync(FULL_MASK_W, mine && (S.res & bit)) != 0u;
    miss_out = hit ? 0u : 1u;
    if (hit) return MCB_OUT_HIT;
    uint32_t code = MCB_OUT_MISS, vbit = 0u;
    if (S.count >= C) {
        // keys are packed (key << 7 | expert): the warp minimum is the victim,
        // ties to the smallest id
        const uint32_t cand = S.res & ~pin & valid;
        uint32_t lk = WKEY_SENT;
#pragma unroll
        for (int s = 0; s < EPL; ++s) lk = min(lk, ((cand >> s) & 1u) ? key[s] : WKEY_SENT);
        const uint32_t m = __reduce_min_sync(FULL_MASK_W, lk);
        stuck |= m == WKEY_SENT;
        const uint32_t v = m & WKEY_ID;
        if (lane == (int)(v / EPL)) {
            vbit = 1u << (v % EPL);
            S.res &= ~vbit;
        }
        code = v;
        ++n.nev;
    } else {
        ++S.count;
    }
    ++n.misses;
    if (mine) {
        n.refc += (S.ring_or & bit) ? 1u : 0u;
#pragma unroll
        for (int s = 0; s <= SOLO_WMAX; ++s) S.ring[s] &= ~bit;
        S.ring_or &= ~bit;
        S.res |= bit;
    }
    S.ring[0] |= vbit;
    S.ring_or |= vbit;
    return code;
}

template <int EPL>
__device__ __forceinline__ void wstate_next_decode(WState<EPL> &S, int W) {
#pragma unroll
    for (int s = SOLO_WMAX; s >= 1; --s) S.ring[s] = S.ring[s - 1];
    S.ring[0] = 0u;
    uint32_t o = 0u;
#pragma unroll
    for (int s = 0; s <= SOLO_WMAX; ++s) o |= (s <= W) ? S.ring[s] : 0u;
    S.ring_or = o;
}

template <int EPL>
__device__ __forceinline__ bool wstate_equal(const WState<EPL> &A, const WState<EPL> &B, int W) {
    uint32_t d = A.res ^ B.res;
#pragma unroll
    for (int s = 0; s <= SOLO_WMAX; ++s) d |= (s <= W) ? (A.ring[s] ^ B.ring[s]) : 0u;
    return __all_sync(FULL_MASK_W, d == 0u);
}

// Per (instance, segment) record of the warp version (384 bytes).
struct WSegOut {
    uint32_t misses, nev, refc, comp;
    int32_t stuck_ev;
    uint32_t pad0;
    uint64_t hash;
    uint32_t res_start[4], res_end[4];           // expert masks (bit e % 32 of word e / 32)
    uint32_t ring_start[SOLO_WMAX + 1][4];
    uint32_t ring_end[SOLO_WMAX + 1][4];
    uint16_t hist[MCB_SEG_BINS];
    uint32_t pad1[7];
};
static_assert(sizeof(WSegOut) == 384, "WSegOut layout");

// lane bits (EPL slots) <-> 128-bit expert masks
template <int EPL>
__device__ __forceinline__ uint32_t pack_word(uint32_t bits, int lane, int w) {
    const int e0 = lane * EPL;
    return __reduce_or_sync(FULL_MASK_W, (e0 >> 5) == w ? (bits << (e0 & 31)) : 0u);
}
template <int EPL>
__device__ __forceinline__ uint32_t unpack_bits(const uint32_t *words, int lane) {
    const int e0 = lane * EPL;
    return (words[e0 >> 5] >> (e0 & 31)) & ((1u << EPL) - 1u);
}

template <int EPL>
__device__ __forceinline__ void store_state(const WState<EPL> &S, uint32_t *res4, uint32_t (*ring4)[4], int lane) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const uint32_t v = pack_word<EPL>(S.res, lane, w);
        if (lane == w) res4[w] = v;
    }
#pragma unroll
    for (int s = 0; s <= SOLO_WMAX; ++s)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const uint32_t v = pack_word<EPL>(S.ring[s], lane, w);
            if (lane == w) ring4[s][w] = v;
        }
}

template <int EPL>
__device__ __forceinline__ void load_state(WState<EPL> &S, const uint32_t *res4, const uint32_t (*ring4)[4], int lane,
                                           int W) {
    S.res = unpack_bits<EPL>(res4, lane);
    uint32_t o = 0u;
#pragma unroll
    for (int s = 0; s <= SOLO_WMAX; ++s) {
        S.ring[s] = unpack_bits<EPL>(ring4[s], lane);
        o |= (s <= W) ? S.ring[s] : 0u;
    }
    S.ring_or = o;
    S.count = __reduce_add_sync(FULL_MASK_W, (uint32_t)__popc(S.res));
}

// A segment record held across the warp: lane l owns 32-bit words l, l + 32
// and l + 64 of the 384-byte WSegOut (one coalesced load per word block), so
// the finish walk can prefetch the next segment's record while it splices the
// current one.  Field words: counters 0-4, hash 6-7, res_start 8-11, res_end
// 12-15, ring_start 16 + 4 s, ring_end 48 + 4 s, hist 80-84 (16-bit pairs).
struct WRec {
    uint32_t w[3];
};
static_assert(sizeof(WSegOut) == 3 * 32 * 4, "WRec covers WSegOut");
__device__ __forceinline__ void wrec_load(WRec &r, const WSegOut *o, int lane) {
    const uint32_t *p = (const uint32_t *)o;
#pragma unroll
    for (int i = 0; i < 3; ++i) r.w[i] = __ldg(p + 32 * i + lane);
}
// word I of the record, on every lane (I compile-time)
template <int I>
__device__ __forceinline__ uint32_t wrec_word(const WRec &r) {
    return __shfl_sync(FULL_MASK_W, r.w[I / 32], I % 32);
}
// word BASE + w (w = this lane's word of a 4-word expert mask, 0..3)
template <int BASE>
__device__ __forceinline__ uint32_t wrec_mask_word(const WRec &r, int w) {
    static_assert(BASE % 32 + 3 < 32, "a mask's four words share one block");
    return __shfl_sync(FULL_MASK_W, r.w[BASE / 32], BASE % 32 + w);
}
template <int EPL, int RES, int RING>
__device__ __forceinline__ void load_state_rec(WState<EPL> &S, const WRec &r, int lane, int W) {
    const int e0 = lane * EPL, w = e0 >> 5, sh = e0 & 31;
    const uint32_t m = (1u << EPL) - 1u;
    S.res = (wrec_mask_word<RES>(r, w) >> sh) & m;
    uint32_t o = 0u;
#pragma unroll
    for (int sl = 0; sl <= SOLO_WMAX; ++sl) {
        uint32_t v;
        switch (sl) {   // (compile-time word index per slot)
            case 0: v = wrec_mask_word<RING + 0>(r, w); break;
            case 1: v = wrec_mask_word<RING + 4>(r, w); break;
            case 2: v = wrec_mask_word<RING + 8>(r, w); break;
            case 3: v = wrec_mask_word<RING + 12>(r, w); break;
            case 4: v = wrec_mask_word<RING + 16>(r, w); break;
            case 5: v = wrec_mask_word<RING + 20>(r, w); break;
            case 6: v = wrec_mask_word<RING + 24>(r, w); break;
            default: v = wrec_mask_word<RING + 28>(r, w); break;
        }
        S.ring[sl] = (v >> sh) & m;
        o |= (sl <= W) ? S.ring[sl] : 0u;
    }
    S.ring_or = o;
    S.count = __reduce_add_sync(FULL_MASK_W, (uint32_t)__popc(S.res));
}
static_assert(SOLO_WMAX == 7, "load_state_rec unrolls 8 ring slots");

// ------------------------------------------------------------------ snapshot --
// one warp per (chain, block of MCB_SNAP_EV events), lanes over experts
__global__ void __launch_bounds__(128) k_wseg_summary(const __grid_constant__ ReplayParams P) {
    const DevTrace &tr = P.tr;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int n_snap = P.seg.n_snap, SN = P.seg.snap_e;
    if (wid >= tr.n_chains * n_snap) return;
    const int64_t chain = wid / n_snap;
    const int b = (int)(wid % n_snap);
    int32_t cnt[4] = {0, 0, 0, 0}, last[4] = {-1, -1, -1, -1};
    const int K = tr.K;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t p0 = (int64_t)b * MCB_SNAP_EV * K;
    const int64_t p1 = min((int64_t)(b + 1) * MCB_SNAP_EV, tr.T) * K;
    U32Stream<32> ids;
    ids.init(tr.acc, (tr.total_acc + 3) >> 2, (a0 + p0) >> 2, lane);
    for (int64_t p = p0; p < p1; ++p) {
        const int64_t A = a0 + p;
        const uint32_t word = ids.get(A >> 2, lane, 0, FULL_MASK_W);
        const uint32_t x = (word >> (8 * (uint32_t)(A & 3))) & 0xFFu;
        if ((int)(x & 31) == lane) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if ((int)(x >> 5) == j) { cnt[j] += 1; last[j] = (int32_t)p; }
        }
    }
    int2 *o = P.seg.summ + wid * SN;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e = lane + 32 * j;
        if (e < SN) o[e] = make_int2(last[j], cnt[j]);
    }
}

// ------------------------------------------------------------------- keys --
// Exact keys of this lane's experts at event ev (a snapshot point), their
// seen mask, and (optionally) the guessed resident set: the min(C, #seen)
// seen experts the policy would evict last (largest keys, then largest ids).
template <int EPL, int POL>
__device__ __forceinline__ void wkeys_at(const ReplayParams &P, int64_t chain, int64_t ev, int lane, int ml_variant,
                                         uint32_t (&key)[EPL], uint32_t &seen) {
    const DevTrace &tr = P.tr;
    const int E = tr.E;
    const int2 *sn = P.seg.snap + (chain * P.seg.n_snap + ev / MCB_SNAP_EV) * P.seg.snap_e;
    const int64_t a0 = tr.acc_begin(chain);
    seen = 0u;
#pragma unroll
    for (int s = 0; s < EPL; ++s) {
        const int e = lane * EPL + s;
        const int2 v = e < E ? __ldg(sn + e) : make_int2(-1, 0);
        seen |= (v.x >= 0 ? 1u : 0u) << s;
        uint32_t k = 0u;
        if (POL == POL_LRU) k = v.x >= 0 ? (uint32_t)v.x : 0u;
        if (POL == POL_LFU) k = (uint32_t)v.y;
        if (POL == POL_BELADY) {
            const uint32_t np = v.x >= 0 ? __ldg(P.next_pos + a0 + v.x) : MCB_NEXT_INF;
            k = np == MCB_NEXT_INF ? 0u : WKEY_KMAX - np;
        }
        key[s] = (k << WKEY_SH) | (uint32_t)e;
        if (POL == POL_ML) {
            const uint32_t r = (ev > 0 && e < E) ? (uint32_t)__ldcg(P.rank[ml_variant] + (tr.ev_begin(chain) + ev - 1) * E + e) : 0u;
            key[s] = r ? ((256u - r) << WKEY_SH) | (uint32_t)e : WKEY_SENT;
        }
    }
}

template <int EPL>
__device__ __forceinline__ uint32_t wguess(const uint32_t (&key)[EPL], uint32_t seen, uint32_t C, int lane) {
    const uint32_t n_seen = __reduce_add_sync(FULL_MASK_W, (uint32_t)__popc(seen));
    const uint32_t n_res = min(C, n_seen);
    uint32_t chosen = 0u;
    for (uint32_t r = 0; r < n_res; ++r) {
        // largest key among the unchosen seen experts, ties to the largest id
        // (packed: (key + 1) << 7 | id, a non-selectable ML score as the bare
        // id, below every other key; a lane without candidates offers 0, and
        // a candidate always remains, so a maximum of 0 is expert 0)
        uint32_t lk = 0u;
#pragma unroll
        for (int s = 0; s < EPL; ++s)
            if (((seen & ~chosen) >> s) & 1u)
                lk = max(lk, key[s] == WKEY_SENT ? (uint32_t)(lane * EPL + s) : key[s] + (1u << WKEY_SH));
        const uint32_t m = __reduce_max_sync(FULL_MASK_W, lk);
        const uint32_t v = m & WKEY_ID;
        if (lane == (int)(v / EPL)) chosen |= 1u << (v % EPL);
    }
    return chosen;
}

// ---------------------------------------------------------------- replay --
// Sequential reader of a word stream by the whole warp: 32-word chunks, one
// word per lane, the next chunk in flight; `off` counts items (of 32 / PER
// bits) consumed in the current chunk, so an item costs one shuffle.
template <int PER>   // items per word: 4 (uint8 ids) or 1 (uint32 next-use positions)
struct WCursor {
    const uint32_t *p;     // the next chunk to load (this lane's word)
    const uint32_t *end;   // one past the last readable word
    uint32_t cur, nxt, off;
    __device__ __forceinline__ uint32_t load(const uint32_t *q) const { return q < end ? __ldg(q) : 0u; }
    __device__ __forceinline__ void init(const void *base, int64_t words, int64_t first_item, int lane) {
        const int64_t w0 = (first_item / PER) & ~(int64_t)31;   // the chunk holding the first item
        end = (const uint32_t *)base + words;
        p = (const uint32_t *)base + w0 + lane;
        cur = load(p);
        nxt = load(p + 32);
        p += 64;
        off = (uint32_t)(first_item - w0 * PER);
    }
    __device__ __forceinline__ uint32_t get() {
        if (off == 32u * PER) {
            cur = nxt;
            nxt = load(p);
            p += 32;
            off = 0u;
        }
        const uint32_t w = __shfl_sync(FULL_MASK_W, cur, (int)(off / PER));
        const uint32_t v = PER == 4 ? (w >> (8u * (off & 3u))) & 0xFFu : w;
        ++off;
        return v;
    }
};

template <int EPL, int POL>
struct WReplay {
    // access stream of one chain from access index a, read in order
    WCursor<4> ids;
    WCursor<1> nx;
    __device__ __forceinline__ void init(const ReplayParams &P, int64_t a, int lane) {
        ids.init(P.tr.acc, (P.tr.total_acc + 3) >> 2, a, lane);
        if (POL == POL_BELADY) nx.init(P.next_pos, P.tr.total_acc, a, lane);
    }
    __device__ __forceinline__ uint32_t id() { return ids.get(); }
    __device__ __forceinline__ uint32_t next() { return nx.get(); }
};

template <int EPL, int POL>
__device__ __forceinline__ void wkey_update(uint32_t (&key)[EPL], bool mine, int slot, uint32_t x, uint32_t pos,
                                            uint32_t np) {
    if (!mine) return;
    uint32_t k = 0u;
    if (POL == POL_LRU) k = (pos << WKEY_SH) | x;
    if (POL == POL_BELADY) k = ((np == MCB_NEXT_INF ? 0u : WKEY_KMAX - np) << WKEY_SH) | x;
#pragma unroll
    for (int s = 0; s < EPL; ++s) {
        if (s != slot) continue;
        if (POL == POL_LFU) key[s] += 1u << WKEY_SH;
        else if (POL == POL_LRU || POL == POL_BELADY) key[s] = k;
    }
}

// This lane's EPL bytes of an event's rank row, packed (byte s = expert
// lane * EPL + s); one 32- / 16-bit load when the row splits evenly.
template <int EPL>
__device__ __forceinline__ uint32_t wrow_load(const uint8_t *row, int lane, int E) {
    const int e = lane * EPL;
    if (EPL == 4 && (E & 3) == 0) return e < E ? __ldcg((const uint32_t *)row + lane) : 0u;
    if (EPL == 2 && (E & 1) == 0) return e < E ? (uint32_t)__ldcg((const uint16_t *)row + lane) : 0u;
    uint32_t v = 0u;
#pragma unroll
    for (int s = 0; s < EPL; ++s)
        if (e + s < E) v |= (uint32_t)__ldcg(row + e + s) << (8 * s);
    return v;
}

// The per-event rank rows of a run of events, two events in flight ahead of
// the one being replayed (a row load is an L2 / HBM round trip; one event of
// K accesses is shorter than that on a warp that issues alone).
template <int EPL>
struct WRows {
    const uint8_t *row;   // the next row to load
    int64_t left;         // rows left to load
    int E;
    uint32_t r0, r1;
    __device__ __forceinline__ void init(const uint8_t *first, int64_t n, int E_, int lane) {
        row = first;
        left = n;
        E = E_;
        r0 = left > 0 ? wrow_load<EPL>(row, lane, E) : 0u;
        r1 = left > 1 ? wrow_load<EPL>(row + E, lane, E) : 0u;
        row += 2 * (int64_t)E;
        left -= 2;
    }
    // this event's keys and selectable mask; starts the load two events ahead
    __device__ __forceinline__ void next(uint32_t (&key)[EPL], uint32_t &valid, int lane) {
        const uint32_t e0 = (uint32_t)(lane * EPL);
        const uint32_t r = r0;
        r0 = r1;
        r1 = left > 0 ? wrow_load<EPL>(row, lane, E) : 0u;
        row += E;
        --left;
        valid = 0u;
#pragma unroll
        for (int s = 0; s < EPL; ++s) {
            const uint32_t b = (r >> (8 * s)) & 0xFFu;
            key[s] = b ? ((256u - b) << WKEY_SH) | (e0 + s) : WKEY_SENT;
            valid |= (b ? 1u : 0u) << s;
        }
    }
};

template <int EPL, int POL>
__device__ __forceinline__ void wseg_spec(const ReplayParams &P, int64_t chain, int seg, int pol_i, int cap_i,
                                          int ml_variant, int lane, int pass) {
    const DevTrace &tr = P.tr;
    const int E = tr.E, K = tr.K, W = P.window;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    const int64_t ev0 = (int64_t)seg * P.seg.SE;
    const int64_t ev1 = min(ev0 + P.seg.SE, tr.T);
    // pass 0: warm-up from a guess; pass 1: start at the segment from pass 0's
    // end state of the previous segment (no warm-up)
    const int64_t nw = POL == POL_LRU ? (P.seg.NW < MCB_SNAP_EV ? P.seg.NW : MCB_SNAP_EV) : P.seg.NW;
    const int64_t ws = pass == 0 ? (ev0 > nw ? ev0 - nw : 0) : ev0;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;

    uint32_t key[EPL], seen;
    wkeys_at<EPL, POL>(P, chain, ws, lane, ml_variant, key, seen);
    WState<EPL> S;
    wstate_clear(S);
    if (pass >= 1 && seg > 0) {   // the previous pass's end state of the previous segment
        const WSegOut &q = ((const WSegOut *)P.seg.out[(pass - 1) & 1])[inst * P.seg.n_seg + seg - 1];
        load_state<EPL>(S, q.res_end, q.ring_end, lane, W);
    } else {
        S.res = wguess<EPL>(key, seen, C, lane);
        S.count = __reduce_add_sync(FULL_MASK_W, (uint32_t)__popc(S.res));
    }
    uint32_t valid = 0u;
#pragma unroll
    for (int s = 0; s < EPL; ++s) valid |= (lane * EPL + s < E ? 1u : 0u) << s;
    uint32_t comp = 0, hist = 0;
    SCount n = {0u, 0u, 0u};
    bool stuck = false;
    int32_t stuck_ev = -1;
    uint64_t h = 0;
    const bool track = P.hashes != nullptr;
    WSegOut &o = ((WSegOut *)P.seg.out[pass & 1])[inst * P.seg.n_seg + seg];   // passes alternate buffers
    uint32_t *codes = (uint32_t *)(P.seg.codes + inst * P.seg.Tpad);
    uint32_t word = 0;
    WReplay<EPL, POL> rp;
    rp.init(P, a0 + ws * K, lane);
    WRows<EPL> rows;
    if (POL == POL_ML) rows.init(rank + (e0 + ws) * E, ev1 - ws, E, lane);
    uint32_t pos = (uint32_t)(ws * K);   // chain-local access position

    for (int64_t ev = ws; ev < ev1; ++ev) {
        if (ev == ev0) {
            store_state<EPL>(S, o.res_start, o.ring_start, lane);
            n.misses = n.nev = n.refc = 0u;
            comp = 0u;
            stuck = false;
        }
        if (POL == POL_ML) rows.next(key, valid, lane);
        uint32_t pin = 0, sm = 0;
        for (int j = 0; j < K; ++j, ++pos) {
            const uint32_t x = rp.id();
            const int owner = (int)(x / EPL), slot = (int)(x % EPL);
            const uint32_t bit = 1u << slot;
            const bool mine = lane == owner;
            const uint32_t np = POL == POL_BELADY ? rp.next() : 0u;
            wkey_update<EPL, POL>(key, mine, slot, x, pos, np);
            uint32_t miss;
            const uint32_t code = wstep<EPL>(S, key, owner, bit, pin, valid, C, lane, n, stuck, miss);
            sm += miss;
            if (mine && miss && !(seen & bit)) ++comp;
            if (mine) { seen |= bit; pin |= bit; }
            if (track && ev >= ev0) h = poly16(h, code);
        }
        if (ev >= ev0) {
            if (stuck && stuck_ev < 0) stuck_ev = (int32_t)ev;
            hist += (sm == (uint32_t)lane) ? 1u : 0u;
            word |= sm << (8 * (uint32_t)(ev & 3));
            if ((ev & 3) == 3) {
                if (lane == 0) codes[ev >> 2] = word;
                word = 0;
            }
        }
        wstate_next_decode<EPL>(S, W);
    }
    if ((ev1 & 3) && lane == 0) codes[ev1 >> 2] = word;
    const uint32_t refc = __reduce_add_sync(FULL_MASK_W, n.refc);
    comp = __reduce_add_sync(FULL_MASK_W, comp);
    store_state<EPL>(S, o.res_end, o.ring_end, lane);
    if (lane < MCB_SEG_BINS) o.hist[lane] = lane <= K ? (uint16_t)hist : (uint16_t)0;
    if (lane == 0) {
        o.misses = n.misses;
        o.nev = n.nev;
        o.refc = refc;
        o.comp = comp;
        o.stuck_ev = stuck_ev;
        o.hash = h;
    }
}

template <int EPL>
__global__ void __launch_bounds__(128) k_wseg_spec(const __grid_constant__ ReplayParams P, int pass) {
    const int pol_i = P.pol_map[blockIdx.y];
    if (pass >= 1 && P.pol[pol_i] == MCB_LRU) return;   // LRU's guess is exact
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int n_seg = P.seg.n_seg;
    if (w >= (P.chain_hi - P.chain_lo) * n_seg * P.n_cap) return;
    const int cap_i = (int)(w % P.n_cap);
    const int64_t r = w / P.n_cap;
    const int seg = (int)(r % n_seg);
    const int64_t chain = P.chain_lo + r / n_seg;
    switch (P.pol[pol_i]) {
        case MCB_LRU: wseg_spec<EPL, POL_LRU>(P, chain, seg, pol_i, cap_i, 0, lane, pass); break;
        case MCB_LFU: wseg_spec<EPL, POL_LFU>(P, chain, seg, pol_i, cap_i, 0, lane, pass); break;
        case MCB_BELADY: wseg_spec<EPL, POL_BELADY>(P, chain, seg, pol_i, cap_i, 0, lane, pass); break;
        case MCB_ML: wseg_spec<EPL, POL_ML>(P, chain, seg, pol_i, cap_i, 0, lane, pass); break;
        default: wseg_spec<EPL, POL_ML>(P, chain, seg, pol_i, cap_i, 1, lane, pass); break;
    }
}

// ------------------------------------------------ thread speculation --
// The same speculation with one THREAD per (instance, segment), for long
// chains (many segments, e.g. C3's 1M-token trace): the state is a 64- or
// 128-bit mask (mcb_mask.cuh), the packed keys (key << 7 | id) sit in shared
// memory column-major per thread, and the victim is a minimum over the
// candidate bits (ML: the top bit of the event's rank-space candidate mask,
// mcb_mask.cuh rank_space).  It writes the warp version's WSegOut records, so the warp
// finish walk (which replays any segment whose recorded start state is not
// the true one) is shared.
namespace tspec {

constexpr int BS = 128;
constexpr int SH = 7;
static_assert(SH == 7, "packed keys carry 7 id bits (E <= 128)");
constexpr uint32_t KMAX = (1u << (32 - SH)) - 1u;
constexpr int NLOW = 4;   // smallest keys kept per event (LRU / LFU / Belady) ...
constexpr uint32_t NLOW_MAXC = 32;   // ... for capacities up to this (as K4-wide)

template <int POL, typename M>
__device__ __forceinline__ void tseg_spec(const ReplayParams &P, int64_t chain, int seg, int pol_i, int cap_i,
                                          int ml_variant, uint32_t *sk, uint16_t *hist, int pass) {
    using namespace mm;
    const DevTrace &tr = P.tr;
    const int E = tr.E, K = tr.K, W = P.window;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    const int64_t ev0 = (int64_t)seg * P.seg.SE;
    const int64_t ev1 = min(ev0 + P.seg.SE, tr.T);
    const int64_t nw = POL == POL_LRU ? (P.seg.NW < MCB_SNAP_EV ? P.seg.NW : MCB_SNAP_EV) : P.seg.NW;
    const int64_t ws = pass == 0 ? (ev0 > nw ? ev0 - nw : 0) : ev0;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;
    auto key = [&](int e) -> uint32_t & { return sk[e * BS]; };
    // ML: the event's rank row as bytes, [thread][mrow_stride(E)] inside the key area
    uint8_t *const mrow = (uint8_t *)(sk - threadIdx.x) + threadIdx.x * mrow_stride(E);
    // ML: rank -> expert of the event's candidates (rank_space), [thread][E] after the rank rows
    uint8_t *const mord = (uint8_t *)(sk - threadIdx.x) + BS * mrow_stride(E) + threadIdx.x * E;

    // exact keys and seen set at ws (a snapshot point)
    const int2 *sn = P.seg.snap + (chain * P.seg.n_snap + ws / MCB_SNAP_EV) * P.seg.snap_e;
    M seen = zero<M>();
    int n_seen = 0;
    for (int e = 0; e < E; ++e) {
        const int2 v = __ldg(sn + e);
        uint32_t k = 0u;
        if (POL == POL_LRU) k = v.x >= 0 ? (uint32_t)v.x : 0u;
        if (POL == POL_LFU) k = (uint32_t)v.y;
        if (POL == POL_BELADY) {
            const uint32_t np = v.x >= 0 ? __ldg(P.next_pos + a0 + v.x) : MCB_NEXT_INF;
            k = np == MCB_NEXT_INF ? 0u : KMAX - np;
        }
        if (POL == POL_ML) mrow[e] = ws > 0 ? __ldcg(rank + (e0 + ws - 1) * E + e) : (uint8_t)0;
        else key(e) = (k << SH) | (uint32_t)e;
        if (v.x >= 0) {
            seen = seen | bit_of<M>((uint32_t)e);
            ++n_seen;
        }
    }
    M res = zero<M>(), ring_or = zero<M>();
    M ring[SOLO_WMAX + 1];
#pragma unroll
    for (int i = 0; i <= SOLO_WMAX; ++i) ring[i] = zero<M>();
    if (pass >= 1 && seg > 0) {   // the previous pass's end state of the previous segment
        const WSegOut &q = ((const WSegOut *)P.seg.out[(pass - 1) & 1])[inst * P.seg.n_seg + seg - 1];
        res = from_words<M>(q.res_end);
#pragma unroll
        for (int i = 0; i <= SOLO_WMAX; ++i) {
            ring[i] = from_words<M>(q.ring_end[i]);
            if (i <= W) ring_or = ring_or | ring[i];
        }
    } else {
        // guess: the min(C, #seen) seen experts the policy would evict last
        // (largest packed keys), by a bitwise search for the threshold key
        auto gkey = [&](int e) -> uint32_t {
            return POL == POL_ML ? (((256u - mrow[e]) << SH) | (uint32_t)e) : key(e);
        };
        const int n_res = min((int)C, n_seen);
        if (n_res > 0) {
            uint32_t tau = 0u;
            for (int b = 31; b >= 0; --b) {
                const uint32_t cand = tau | (1u << b);
                int cnt = 0;
                for (int e = 0; e < E; ++e) cnt += (test(seen, (uint32_t)e) && gkey(e) >= cand) ? 1 : 0;
                if (cnt >= n_res) tau = cand;
            }
            for (int e = 0; e < E; ++e)
                if (test(seen, (uint32_t)e) && gkey(e) >= tau) res = res | bit_of<M>((uint32_t)e);
        }
    }
    uint32_t misses = 0, nev = 0, refc = 0, comp = 0;
    int32_t stuck_ev = -1;
    bool stuck = false;
    uint64_t h = 0;
    const bool track = P.hashes != nullptr;
    for (int b = 0; b <= K; ++b) hist[b * BS] = 0;
    WSegOut &o = ((WSegOut *)P.seg.out[pass & 1])[inst * P.seg.n_seg + seg];   // passes alternate buffers
    uint32_t *codes = (uint32_t *)(P.seg.codes + inst * P.seg.Tpad);
    uint32_t word = 0;

    for (int64_t ev = ws; ev < ev1; ++ev) {
        if (ev == ev0) {
            to_words(res, o.res_start);
#pragma unroll
            for (int i = 0; i <= SOLO_WMAX; ++i) to_words(ring[i], o.ring_start[i]);
            misses = nev = refc = comp = 0u;
            stuck = false;
        }
        M cr = zero<M>();   // ML: resident \ pinned in rank space, kept in step with every access
        if (POL == POL_ML) {   // this event's rank row (mlpolicy.py:59-62) as bytes (rank 0 = not selectable)
            copy_rank_row(rank + (e0 + ev) * E, mrow, E);
            cr = rank_space(res, mrow, mord);
        }
        // LRU / LFU / Belady: the event's victims in key order from the NLOW
        // smallest keys of the resident set at its start (see K4-wide, mcb_wide.cu)
        constexpr bool KEYED = POL != POL_ML;
        uint32_t low[NLOW], lp = NLOW;
        if (KEYED && C <= NLOW_MAXC && (uint32_t)popc(res) + (uint32_t)K > C) {
            lowest_keys<BS, NLOW>(res, sk, low);
            lp = 0;
        }
        M pin = zero<M>();
        uint32_t sm = 0;
        for (int j = 0; j < K; ++j) {
            const int64_t A = a0 + ev * K + j;
            const uint32_t x = __ldg(tr.acc + A);
            const uint32_t pos = (uint32_t)(ev * K + j);
            const M bit = bit_of<M>(x);
            if (POL == POL_LRU) key(x) = (pos << SH) | x;
            if (POL == POL_LFU) key(x) += 1u << SH;
            if (POL == POL_BELADY) {
                const uint32_t np = __ldg(P.next_pos + A);
                key(x) = ((np == MCB_NEXT_INF ? 0u : KMAX - np) << SH) | x;
            }
            uint32_t code = MCB_OUT_HIT;
            if (!test(res, x)) {
                M vbit = zero<M>();
                code = MCB_OUT_MISS;
                if ((uint32_t)popc(res) >= C) {
                    const M cand = res & ~pin;
                    // ML: the highest-ranked candidate; none with rank >= 1 (no candidate selectable) = stuck
                    uint32_t lk = ~0u;
                    while (KEYED && lp < NLOW) {
                        uint32_t k = low[0];
#pragma unroll
                        for (int q = 1; q < NLOW; ++q) k = lp == (uint32_t)q ? low[q] : k;
                        ++lp;
                        if (k == ~0u) {   // the start-of-event resident set is used up
                            lp = NLOW;
                        } else if (!test(pin, k & ((1u << SH) - 1u))) {
                            lk = k;
                            break;
                        }
                    }
                    const bool none = POL == POL_ML ? !any(cr) : !any(cand);
                    const uint32_t best = none ? 0u
                                          : (POL == POL_ML ? (uint32_t)mord[top_bit(cr)]
                                                           : (lk != ~0u ? lk : min_key<BS>(cand, sk)));
                    if (none) {
                        stuck = true;
                    } else {
                        if (POL == POL_ML) cr = cr & ~bit_of<M>(top_bit(cr));
                        const uint32_t v = POL == POL_ML ? best : (best & ((1u << SH) - 1u));
                        vbit = bit_of<M>(v);
                        code = v;
                        ++nev;
                    }
                }
                res = (res & ~vbit) | bit;
                ++misses;
                ++sm;
                refc += test(ring_or, x) ? 1u : 0u;
                ring_or = (ring_or & ~bit) | vbit;
#pragma unroll
                for (int i = 0; i <= SOLO_WMAX; ++i) ring[i] = ring[i] & ~bit;
                ring[0] = ring[0] | vbit;
                comp += test(seen, x) ? 0u : 1u;
            }
            if (POL == POL_ML) cr = cr & ~rank_bit<M>(mrow[x]);   // x is pinned for the rest of the event
            seen = seen | bit;
            pin = pin | bit;
            if (track && ev >= ev0) h = poly16(h, code);
        }
        if (ev >= ev0) {
            if (stuck && stuck_ev < 0) stuck_ev = (int32_t)ev;
            hist[sm * BS] += 1;
            word |= sm << (8 * (uint32_t)(ev & 3));
            if ((ev & 3) == 3) {
                codes[ev >> 2] = word;
                word = 0;
            }
        }
#pragma unroll
        for (int i = SOLO_WMAX; i >= 1; --i) ring[i] = ring[i - 1];
        ring[0] = zero<M>();
        M orr = zero<M>();
#pragma unroll
        for (int i = 0; i <= SOLO_WMAX; ++i)
            if (i <= W) orr = orr | ring[i];
        ring_or = orr;
    }
    if (ev1 & 3) codes[ev1 >> 2] = word;   // a segment ends mid-word only at the chain end
    to_words(res, o.res_end);
#pragma unroll
    for (int i = 0; i <= SOLO_WMAX; ++i) to_words(ring[i], o.ring_end[i]);
    for (int b = 0; b < MCB_SEG_BINS; ++b) o.hist[b] = b <= K ? hist[b * BS] : (uint16_t)0;
    o.misses = misses;
    o.nev = nev;
    o.refc = refc;
    o.comp = comp;
    o.stuck_ev = stuck_ev;
    o.hash = h;
}

template <typename M>
__global__ void __launch_bounds__(BS) k_tseg_spec(const __grid_constant__ ReplayParams P, int pass) {
    extern __shared__ uint32_t s_tsk[];   // keys [E][BS], then uint16 histograms [MCB_SEG_BINS][BS]
    const int pol_i = P.pol_map[blockIdx.y];
    if (pass >= 1 && P.pol[pol_i] == MCB_LRU) return;   // LRU's guess is exact
    const int64_t t = (int64_t)blockIdx.x * BS + threadIdx.x;
    const int n_seg = P.seg.n_seg;
    if (t >= (P.chain_hi - P.chain_lo) * n_seg * P.n_cap) return;
    const int cap_i = (int)(t % P.n_cap);
    const int64_t r = t / P.n_cap;
    const int seg = (int)(r % n_seg);
    const int64_t chain = P.chain_lo + r / n_seg;
    uint32_t *sk = s_tsk + threadIdx.x;
    uint16_t *hist = (uint16_t *)(s_tsk + P.tr.E * BS) + threadIdx.x;
    switch (P.pol[pol_i]) {
        case MCB_LRU: tseg_spec<POL_LRU, M>(P, chain, seg, pol_i, cap_i, 0, sk, hist, pass); break;
        case MCB_LFU: tseg_spec<POL_LFU, M>(P, chain, seg, pol_i, cap_i, 0, sk, hist, pass); break;
        case MCB_BELADY: tseg_spec<POL_BELADY, M>(P, chain, seg, pol_i, cap_i, 0, sk, hist, pass); break;
        case MCB_ML: tseg_spec<POL_ML, M>(P, chain, seg, pol_i, cap_i, 0, sk, hist, pass); break;
        default: tseg_spec<POL_ML, M>(P, chain, seg, pol_i, cap_i, 1, sk, hist, pass); break;
    }
}

}  // namespace tspec

// ----------------------------------------------------------------- finish --

template <int EPL, int POL>
__device__ __forceinline__ void wseg_finish(const ReplayParams &P, int64_t chain, int pol_i, int cap_i, int ml_variant,
                                            const double *lut, int lane) {
    const DevTrace &tr = P.tr;
    const int E = tr.E, K = tr.K, W = P.window;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int n_seg = P.seg.n_seg, SE = P.seg.SE;
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;
    const uint8_t *codes = P.seg.codes + inst * P.seg.Tpad;
    const WSegOut *so = (const WSegOut *)P.seg.out[POL == POL_LRU ? 0 : ((P.seg.passes - 1) & 1)] + inst * n_seg;
    const bool track = P.hashes != nullptr;

    WState<EPL> A;                         // the true state, carried across segments
    wstate_clear(A);
    uint32_t misses = 0, nev = 0, refc = 0, comp = 0, fix_events = 0, unconverged = 0, slow = 0;
    bool stuck = false;
    uint64_t h = 0;
    double dlat = 0.0;
    uint32_t valid0 = 0u;
#pragma unroll
    for (int s = 0; s < EPL; ++s) valid0 |= (lane * EPL + s < E ? 1u : 0u) << s;

    WRec rn;                               // the next segment's record, in flight
    if (n_seg > 0) wrec_load(rn, so, lane);
    for (int seg = 0; seg < n_seg; ++seg) {
        const int64_t ev0 = (int64_t)seg * SE;
        const int64_t ev1 = min(ev0 + (int64_t)SE, tr.T);
        const WRec o = rn;
        if (seg + 1 < n_seg) wrec_load(rn, so + seg + 1, lane);
        WState<EPL> B;
        load_state_rec<EPL, 8, 16>(B, o, lane, W);
        bool conv = wstate_equal<EPL>(A, B, W);
        int64_t ev = ev0;
        SCount ca = {0u, 0u, 0u}, cb = {0u, 0u, 0u};
        uint64_t ha = 0, hb = 0;
        bool stuck_a = false, stuck_b = false;
        uint32_t hb_lane = 0;               // B's prefix miss-count histogram (bin = lane)
        if (!conv) {
            uint32_t key[EPL], seen;
            wkeys_at<EPL, POL>(P, chain, ev0, lane, ml_variant, key, seen);
            uint32_t valid = valid0;
            WReplay<EPL, POL> rp;
            rp.init(P, a0 + ev0 * K, lane);
            WRows<EPL> rows;
            if (POL == POL_ML) rows.init(rank + (e0 + ev0) * E, ev1 - ev0, E, lane);
            uint32_t pos = (uint32_t)(ev0 * K);
            while (!conv && ev < ev1) {
                if (POL == POL_ML) rows.next(key, valid, lane);
                uint32_t pin = 0, sma = 0, smb = 0;
                for (int j = 0; j < K; ++j, ++pos) {
                    const uint32_t x = rp.id();
                    const int owner = (int)(x / EPL), slot = (int)(x % EPL);
                    const uint32_t bit = 1u << slot;
                    const bool mine = lane == owner;
                    const uint32_t np = POL == POL_BELADY ? rp.next() : 0u;
                    wkey_update<EPL, POL>(key, mine, slot, x, pos, np);
                    uint32_t ma, mb;
                    const uint32_t codea = wstep<EPL>(A, key, owner, bit, pin, valid, C, lane, ca, stuck_a, ma);
                    const uint32_t codeb = wstep<EPL>(B, key, owner, bit, pin, valid, C, lane, cb, stuck_b, mb);
                    sma += ma;
                    smb += mb;
                    if (mine) pin |= bit;
                    if (track) { ha = poly16(ha, codea); hb = poly16(hb, codeb); }
                }
                dlat = __dadd_rn(dlat, lut[sma]);
                hb_lane += (smb == (uint32_t)lane) ? 1u : 0u;
                wstate_next_decode<EPL>(A, W);
                wstate_next_decode<EPL>(B, W);
                ++ev;
                conv = wstate_equal<EPL>(A, B, W);
            }
            fix_events += (uint32_t)(ev - ev0);
        }
        const uint32_t refa = __reduce_add_sync(FULL_MASK_W, ca.refc);
        const uint32_t refb = __reduce_add_sync(FULL_MASK_W, cb.refc);
        uint64_t hseg;
        if (conv) {
            const int32_t o_stuck = (int32_t)wrec_word<4>(o);
            misses += ca.misses + wrec_word<0>(o) - cb.misses;
            nev += ca.nev + wrec_word<1>(o) - cb.nev;
            refc += refa + wrec_word<2>(o) - refb;
            stuck = stuck || stuck_a || (o_stuck >= 0 && o_stuck >= ev);
            const uint64_t o_hash = (uint64_t)wrec_word<6>(o) | ((uint64_t)wrec_word<7>(o) << 32);
            hseg = track ? o_hash + (ha - hb) * pow_mul((uint64_t)(ev1 - ev) * K) : 0ull;
            load_state_rec<EPL, 12, 48>(A, o, lane, W);
            // hist[b] = 16-bit half (b & 1) of word 80 + b / 2: lane 16 + b / 2 of block 2
            const uint32_t hw = __shfl_sync(FULL_MASK_W, o.w[2], 16 + ((lane >> 1) & 15));
            const uint32_t h_lane = (lane & 1) ? (hw >> 16) : (hw & 0xFFFFu);   // lane b holds hist[b]
            uint32_t cnt[MCB_SEG_BINS];
#pragma unroll
            for (int b = 0; b < MCB_SEG_BINS; ++b) {
                const uint32_t hbv = __shfl_sync(FULL_MASK_W, hb_lane, b);
                const uint32_t hv = __shfl_sync(FULL_MASK_W, h_lane, b);
                cnt[b] = b <= K ? hv - hbv : 0u;
            }
            if (!fold_hist_fast(dlat, cnt, K + 1, lut)) {
                dlat = fold_codes(dlat, codes, ev, ev1, lut);
                ++slow;
            }
        } else {
            misses += ca.misses;
            nev += ca.nev;
            refc += refa;
            stuck = stuck || stuck_a;
            hseg = ha;
            ++unconverged;
        }
        comp += wrec_word<3>(o);
        if (track) h = h * pow_mul((uint64_t)(ev1 - ev0) * K) + hseg;
    }
    if (lane != 0) return;
    if (P.stats) {
        atomicAdd(P.stats + 1, (unsigned long long)fix_events);
        atomicAdd(P.stats + 2, (unsigned long long)unconverged);
        atomicAdd(P.stats + 3, (unsigned long long)n_seg);
        atomicAdd(P.stats + 4, (unsigned long long)slow);
    }
    const uint32_t total = (uint32_t)(tr.T * K);
    int64_t *out = P.inst_out + inst * MCB_R_N;
    out[MCB_R_PREFILL_HITS] = 0;
    out[MCB_R_PREFILL_MISSES] = 0;
    out[MCB_R_DECODE_HITS] = total - misses;
    out[MCB_R_DECODE_MISSES] = misses;
    out[MCB_R_COMPULSORY] = comp;
    out[MCB_R_EVICTIONS] = nev;
    out[MCB_R_REFETCHED] = refc;
    out[MCB_R_STATUS] = stuck ? MCB_ERR_NO_EVICTABLE : MCB_OK;
    P.inst_lat[inst * 2 + 0] = dlat;
    P.inst_lat[inst * 2 + 1] = 0.0;
    if (track) P.hashes[inst] = h;
}

template <int EPL>
__global__ void __launch_bounds__(32) k_wseg_finish(const __grid_constant__ ReplayParams P) {
    __shared__ double lut[MCB_SEG_BINS];
    const int pol_i = P.pol_map[blockIdx.y];
    const int pol = P.pol[pol_i];
    const int K = P.tr.K;
    const int lane = threadIdx.x & 31;
    if (lane <= K) {
        // step_latency_s (engine.py:58-62) per miss count, + ml_score_cost_s for ML decode steps
        const uint32_t m = lane;
        const double lat = m > 0 ? __dmul_rn((double)(P.loads_serial ? m : 1u), P.t_load)
                                 : __dmul_rn((double)K, P.t_compute);
        lut[m] = __dadd_rn(lat, (pol == MCB_ML || pol == MCB_ML_NO_PREFILL) ? P.ml_cost : 0.0);
    }
    __syncwarp();
    const int64_t t = blockIdx.x;
    if (t >= (P.chain_hi - P.chain_lo) * P.n_cap) return;
    const int cap_i = (int)(t % P.n_cap);
    const int64_t chain = P.chain_lo + t / P.n_cap;
    switch (pol) {
        case MCB_LRU: wseg_finish<EPL, POL_LRU>(P, chain, pol_i, cap_i, 0, lut, lane); break;
        case MCB_LFU: wseg_finish<EPL, POL_LFU>(P, chain, pol_i, cap_i, 0, lut, lane); break;
        case MCB_BELADY: wseg_finish<EPL, POL_BELADY>(P, chain, pol_i, cap_i, 0, lut, lane); break;
        case MCB_ML: wseg_finish<EPL, POL_ML>(P, chain, pol_i, cap_i, 0, lut, lane); break;
        default: wseg_finish<EPL, POL_ML>(P, chain, pol_i, cap_i, 1, lut, lane); break;
    }
}

template <int EPL>
static int launch_wseg_t(const ReplayParams &p, cudaStream_t s, int phase) {
    int n = 0;
    if (phase != SEG_FINISH && p.seg.thread_spec) {
        const int64_t n_spec = (p.chain_hi - p.chain_lo) * p.seg.n_seg * p.n_cap;   // threads
        const dim3 g((unsigned)((n_spec + tspec::BS - 1) / tspec::BS), (unsigned)p.n_pol_launch);
        const size_t smem = (size_t)p.tr.E * tspec::BS * 4 + (size_t)MCB_SEG_BINS * tspec::BS * 2;
        for (int pass = 0; pass < p.seg.passes; ++pass) {
            if (p.tr.E <= 64) tspec::k_tseg_spec<uint64_t><<<g, tspec::BS, smem, s>>>(p, pass);
            else tspec::k_tseg_spec<mm::M128><<<g, tspec::BS, smem, s>>>(p, pass);
            ++n;
        }
    } else if (phase != SEG_FINISH) {
        const int64_t n_spec = (p.chain_hi - p.chain_lo) * p.seg.n_seg * p.n_cap;   // warps
        const dim3 g((unsigned)((n_spec + 3) / 4), (unsigned)p.n_pol_launch);
        k_wseg_spec<EPL><<<g, 128, 0, s>>>(p, 0);
        ++n;
        if (p.seg.passes > 1) {
            k_wseg_spec<EPL><<<g, 128, 0, s>>>(p, 1);
            ++n;
        }
    }
    if (phase != SEG_SPEC) {
        const int64_t n_fin = (p.chain_hi - p.chain_lo) * p.n_cap;
        k_wseg_finish<EPL><<<dim3((unsigned)n_fin, (unsigned)p.n_pol_launch), 32, 0, s>>>(p);
        ++n;
    }
    return n;
}

int launch_replay_segmented_warp(const ReplayParams &p, cudaStream_t s, int phase) {
    if ((p.chain_hi - p.chain_lo) * p.n_pol_launch * p.n_cap == 0) return 0;
    if (p.tr.E <= 32) return launch_wseg_t<1>(p, s, phase);
    if (p.tr.E <= 64) return launch_wseg_t<2>(p, s, phase);
    return launch_wseg_t<4>(p, s, phase);
}

int launch_seg_snapshot_warp(const ReplayParams &p, cudaStream_t s) {
    const int64_t n = p.tr.n_chains * p.seg.n_snap;   // warps
    k_wseg_summary<<<(unsigned)((n + 3) / 4), 128, 0, s>>>(p);
    return 1;
}

size_t wseg_out_bytes(int64_t n_inst, int n_seg) { return (size_t)n_inst * n_seg * sizeof(WSegOut); }

int preload_segment_warp_kernels() {
    cudaFuncAttributes a;
    const void *fns[] = {(const void *)k_wseg_summary, (const void *)k_wseg_spec<1>, (const void *)k_wseg_spec<2>,
                         (const void *)k_wseg_spec<4>, (const void *)k_wseg_finish<1>,
                         (const void *)k_wseg_finish<2>, (const void *)k_wseg_finish<4>,
                         (const void *)tspec::k_tseg_spec<uint64_t>, (const void *)tspec::k_tseg_spec<mm::M128>};
    for (const void *f : fns)
        if (cudaFuncGetAttributes(&a, f) != cudaSuccess) return -1;
    const int max_smem = 128 * tspec::BS * 4 + MCB_SEG_BINS * tspec::BS * 2;
    if (cudaFuncSetAttribute((const void *)tspec::k_tseg_spec<mm::M128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_smem) != cudaSuccess)
        return -1;
    return 0;
}
