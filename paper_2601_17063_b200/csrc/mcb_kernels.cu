// sm_100a kernels of the expert-cache replay engine.
//
//   K2  k_next_use      reverse segmented next-use scan (Belady oracle)
//   K3  k_feat_snap     per-chain recency/frequency scan, tile snapshots
//       k_score_tile    feature rebuild + float64 scorer MLP + per-event ranks
//   K4  k_replay        lane-group-per-instance cache replay (LRU/LFU/Belady/ML)
//   K5  k_fold          per-(trace, policy, capacity) layer-order fold
//
// Reference semantics: pkg/src/moecache/engine.py:205-263 (_replay_layer),
// policies.py:95-214, mlpolicy.py:15-62, features.py:34-52, net.py:43-105,
// replay.py:44-89; normative restatement in SURVEY.md Appendix A.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <math.h>
#include <stdint.h>

#include "mcb_kernels.cuh"
#include "mcb_solo.cuh"

#define FULL_MASK 0xFFFFFFFFu

// ===========================================================================
// K2: next-use positions.  One warp per chain walks its stream backwards in
// windows of 32 positions.  Inside a window __match_any_sync groups equal
// experts: a lane's next use is the next higher lane of its group, or, for
// the last occurrence in the window, the first occurrence after the window
// (per-expert table in shared memory, E <= 128 entries per warp).  The lowest
// lane of each group then publishes its position as the new first occurrence.
// Integer only, so bit-exact with OracleIndex.next_use (policies.py:65-76):
// next_use(e, p) = next_pos[p] - p, inf when next_pos == 0xFFFFFFFF.
// ===========================================================================
//
// Long chains (few of them, e.g. one Mixtral trace: 32 chains of 131K
// accesses) are cut into blocks so every SM has warps: pass 1 scans each
// block backwards from an empty table and records the block's per-expert
// first occurrence; a reverse scan over blocks turns those into "first
// occurrence after block b"; pass 2 re-scans each block from that table and
// writes the positions.  Same integer results as the single-block walk.
// ===========================================================================
template <bool WRITE>
__global__ void __launch_bounds__(128) k_next_use(DevTrace tr, int64_t blk_acc, int64_t n_blk,
                                                  const uint32_t *__restrict__ tab_in, uint32_t *__restrict__ tab_out,
                                                  uint32_t *__restrict__ next_pos) {
    __shared__ uint32_t table[4][MCB_MAX_EXPERTS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t id = (int64_t)blockIdx.x * 4 + w;
    const int64_t c = id / n_blk, blk = id % n_blk;
    if (c >= tr.n_chains) return;
    const int E = tr.E;
    uint32_t *tbl = table[w];
    const uint32_t *tin = tab_in ? tab_in + id * E : nullptr;
    for (int e = lane; e < MCB_MAX_EXPERTS; e += 32) tbl[e] = (tin && e < E) ? tin[e] : MCB_NEXT_INF;
    __syncwarp();
    const int64_t a0 = tr.acc_begin(c);
    const int64_t n_chain = tr.acc_end(c) - a0;
    const int64_t p0 = blk * blk_acc;                       // multiple of 32
    const int64_t n = min(n_chain, p0 + blk_acc);           // block = [p0, n)
    const uint8_t *acc = tr.acc + a0;
    uint32_t *out = next_pos + a0;
    const int64_t w0 = p0 >> 5;
    const int64_t nwin = (n + 31) >> 5;
    // software pipeline: the load of window w-1 is in flight while w is processed
    uint32_t x_next = 0;
    if (nwin > w0) {
        const int64_t p = ((nwin - 1) << 5) + lane;
        x_next = p < n ? (uint32_t)__ldg(acc + p) : 256u + lane;
    }
    for (int64_t win = nwin - 1; win >= w0; --win) {
        const int64_t p = (win << 5) + lane;
        const bool valid = p < n;
        const uint32_t x = x_next;
        if (win > w0) x_next = (uint32_t)__ldg(acc + p - 32);
        const uint32_t m = __match_any_sync(FULL_MASK, x);
        const uint32_t higher = m & ~((2u << lane) - 1u);
        uint32_t r;
        if (higher) r = (uint32_t)((win << 5) + __ffs(higher) - 1);
        else r = valid ? tbl[x] : 0u;
        __syncwarp();
        if (valid && (m & ((1u << lane) - 1u)) == 0u) tbl[x] = (uint32_t)p;
        __syncwarp();
        if (WRITE && valid) out[p] = r;
    }
    if (tab_out)
        for (int e = lane; e < E; e += 32) tab_out[id * E + e] = tbl[e];
}

// Many chains (C4, C5, their per-rank shares): one THREAD per chain walks it
// backwards with its own table [E][thread] in shared memory (last position
// seen per expert) -- no warp MATCH (the warp walk is MIO-throttled), 16 ids
// per vector load with the next one in flight, 16 results per four 16-byte
// stores.  Uniform traces with T*K a multiple of 16.
__global__ void __launch_bounds__(128) k_next_use_thread(DevTrace tr, uint32_t *__restrict__ next_pos) {
    extern __shared__ uint32_t s_nu[];   // [E][128]
    const int64_t c = (int64_t)blockIdx.x * 128 + threadIdx.x;
    if (c >= tr.n_chains) return;
    const int E = tr.E;
    uint32_t *tab = s_nu + threadIdx.x;
    for (int e = 0; e < E; ++e) tab[e * 128] = MCB_NEXT_INF;
    const int64_t len = tr.T * tr.K;
    const uint4 *src = (const uint4 *)(tr.acc + c * len);
    uint4 *dst = (uint4 *)(next_pos + c * len);
    const int64_t nb = len / 16;
    uint4 nxt = nb > 0 ? __ldg(src + nb - 1) : make_uint4(0, 0, 0, 0);
    for (int64_t b = nb - 1; b >= 0; --b) {
        const uint4 v = nxt;
        if (b > 0) nxt = __ldg(src + b - 1);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        uint32_t r[16];
#pragma unroll
        for (int i = 15; i >= 0; --i) {
            const uint32_t x = (w[i >> 2] >> (8 * (i & 3))) & 0xFFu;
            r[i] = tab[x * 128];
            tab[x * 128] = (uint32_t)(b * 16 + i);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[b * 4 + q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
    }
}

// firsts[c][b][e] (first occurrence in block b) -> after[c][b][e] (first
// occurrence in any later block), one thread per (chain, expert)
__global__ void k_next_use_blocks(int64_t n_chains, int E, int64_t n_blk, const uint32_t *__restrict__ firsts,
                                  uint32_t *__restrict__ after) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_chains * E) return;
    const int64_t c = t / E;
    const int e = (int)(t % E);
    uint32_t nf = MCB_NEXT_INF;
    for (int64_t b = n_blk - 1; b >= 0; --b) {
        const int64_t i = (c * n_blk + b) * E + e;
        after[i] = nf;
        const uint32_t f = firsts[i];
        if (f != MCB_NEXT_INF) nf = f;
    }
}

// blocks per chain for the blocked walk (1 = single walk per chain)
int64_t next_use_blocks(const DevTrace &tr) {
    if (!tr.uniform || tr.n_chains == 0) return 1;
    const int64_t len = tr.T * tr.K;
    const int64_t target_warps = 148ll * 16;
    int64_t nb = (target_warps + tr.n_chains - 1) / tr.n_chains;
    const int64_t cap = len / 2048;                        // blocks of at least 2048 accesses
    if (nb > cap) nb = cap;
    return nb > 1 ? nb : 1;
}

size_t next_use_scratch_words(const DevTrace &tr) {
    const int64_t nb = next_use_blocks(tr);
    return nb > 1 ? (size_t)(2 * tr.n_chains * nb * tr.E) : 0;
}

int launch_next_use(const DevTrace &tr, uint32_t *next_pos, uint32_t *scratch, cudaStream_t s) {
    if (tr.n_chains == 0) return 0;
    if (tr.uniform && tr.n_chains >= 8192 && (tr.T * tr.K) % 16 == 0 && tr.E <= MCB_MAX_EXPERTS) {
        k_next_use_thread<<<(unsigned)((tr.n_chains + 127) / 128), 128, (size_t)tr.E * 128 * sizeof(uint32_t), s>>>(
            tr, next_pos);
        return 1;
    }
    const int64_t nb = scratch ? next_use_blocks(tr) : 1;
    if (nb <= 1) {
        const int64_t blocks = (tr.n_chains + 3) / 4;
        k_next_use<true><<<(unsigned)blocks, 128, 0, s>>>(tr, (int64_t)1 << 40, 1, nullptr, nullptr, next_pos);
        return 1;
    }
    const int64_t len = tr.T * tr.K;
    const int64_t blk_acc = ((len + nb - 1) / nb + 31) / 32 * 32;
    const int64_t n_blk = (len + blk_acc - 1) / blk_acc;
    uint32_t *firsts = scratch, *after = scratch + tr.n_chains * n_blk * tr.E;
    const unsigned g = (unsigned)((tr.n_chains * n_blk + 3) / 4);
    k_next_use<false><<<g, 128, 0, s>>>(tr, blk_acc, n_blk, nullptr, firsts, next_pos);
    k_next_use_blocks<<<(unsigned)((tr.n_chains * tr.E + 127) / 128), 128, 0, s>>>(tr.n_chains, tr.E, n_blk, firsts,
                                                                                     after);
    k_next_use<true><<<g, 128, 0, s>>>(tr, blk_acc, n_blk, after, nullptr, next_pos);
    return 3;
}

// ===========================================================================
// K4: replay.  One lane group of G lanes replays one cache instance
// (chain, policy, capacity).  Expert e lives in lane e / EPL, slot e % EPL.
// Per lane: resident / pinned / seen bits, the policy key of each of its
// experts for ALL experts (LRU last position, LFU in-sequence count, Belady
// bitwise-not of the next-use position, ML 256 - score rank), and the
// pending-refetch decode index of experts it evicted.  Every policy's victim
// is the argmin of (key, expert id) over resident \ pinned:
// a lane-local scan in slot order, a redux.sync min over the group, and a
// ballot that picks the lowest lane among equal keys, i.e. the lowest id.
// ===========================================================================
#define KEY_SENT 0xFFFFFFFFu

template <int EPL>
__device__ __forceinline__ void set_slot(uint32_t (&a)[EPL], int slot, uint32_t v) {
#pragma unroll
    for (int s = 0; s < EPL; ++s)
        if (s == slot) a[s] = v;
}
template <int EPL>
__device__ __forceinline__ uint32_t get_slot(const uint32_t (&a)[EPL], int slot) {
    uint32_t v = a[0];
#pragma unroll
    for (int s = 1; s < EPL; ++s)
        if (s == slot) v = a[s];
    return v;
}

// ARC (policies.py:217-302) for the lane-group replay: per lane the T1 / T2 /
// B1 / B2 membership of its EPL experts and their insertion clocks; list
// sizes, the clock and the adaptation target p are group-uniform.  A list's
// LRU end is the smallest clock (redux.sync min + ballot; clocks are unique).
template <int EPL>
struct WArc {
    uint32_t t1, t2, b1, b2;
    uint32_t ord[EPL];
    uint32_t clock;
    int n1, n2, nb1, nb2;
    double p;
};

template <int EPL>
__device__ __forceinline__ void warc_lru(const WArc<EPL> &a, uint32_t mask, unsigned gmask, int gbase, int &vlane,
                                         int &vs) {
    uint32_t lk = KEY_SENT;
    int ls = 0;
#pragma unroll
    for (int s = 0; s < EPL; ++s)
        if (((mask >> s) & 1u) && a.ord[s] < lk) { lk = a.ord[s]; ls = s; }
    const uint32_t m = __reduce_min_sync(gmask, lk);
    if (m == KEY_SENT) { vlane = -1; vs = 0; return; }
    const unsigned b = __ballot_sync(gmask, lk == m) & gmask;
    const int wl = __ffs(b) - 1;
    vs = __shfl_sync(gmask, ls, wl);
    vlane = wl - gbase;
}

// move expert (vlane, vs) to list which (0 T1, 1 T2, 2 B1, 3 B2, 4 remove)
template <int EPL>
__device__ __forceinline__ void warc_put(WArc<EPL> &a, int vlane, int vs, int which, unsigned gmask, int gbase,
                                         int glane) {
    int old = 0;
    if (glane == vlane) {
        const uint32_t b = 1u << vs;
        old = (a.t1 & b) ? 1 : (a.t2 & b) ? 2 : (a.b1 & b) ? 3 : (a.b2 & b) ? 4 : 0;
        a.t1 &= ~b;
        a.t2 &= ~b;
        a.b1 &= ~b;
        a.b2 &= ~b;
        if (which == 0) a.t1 |= b;
        if (which == 1) a.t2 |= b;
        if (which == 2) a.b1 |= b;
        if (which == 3) a.b2 |= b;
        if (which != 4) set_slot<EPL>(a.ord, vs, a.clock);
    }
    old = __shfl_sync(gmask, old, gbase + vlane);
    a.n1 -= old == 1; a.n2 -= old == 2; a.nb1 -= old == 3; a.nb2 -= old == 4;
    a.n1 += which == 0; a.n2 += which == 1; a.nb1 += which == 2; a.nb2 += which == 3;
    if (which != 4) ++a.clock;
}

template <int EPL>
__device__ __forceinline__ void warc_replace(WArc<EPL> &a, bool in_b2, uint32_t pin, unsigned gmask, int gbase,
                                             int glane, int &vl, int &vs) {
    const bool use_t1 = a.n1 >= 1 && ((double)a.n1 > a.p || (in_b2 && (double)a.n1 == a.p));
    warc_lru<EPL>(a, (use_t1 ? a.t1 : a.t2) & ~pin, gmask, gbase, vl, vs);
    bool from_t1 = use_t1;
    if (vl < 0) {
        warc_lru<EPL>(a, (use_t1 ? a.t2 : a.t1) & ~pin, gmask, gbase, vl, vs);
        from_t1 = !use_t1;
    }
    if (vl >= 0) warc_put<EPL>(a, vl, vs, from_t1 ? 2 : 3, gmask, gbase, glane);
}

// miss path of ARCPolicy.access (policies.py:264-302): victim (vl, vs) or
// vl = -1; none_left when every candidate is pinned
template <int EPL>
__device__ __forceinline__ void warc_miss(WArc<EPL> &a, int owner, int slot, uint32_t pin, uint32_t C,
                                          unsigned gmask, int gbase, int glane, int &vl, int &vs, bool &none_left) {
    const uint32_t bit = 1u << slot;
    const bool mine = glane == owner;
    const bool in_b1 = (__ballot_sync(gmask, mine && (a.b1 & bit)) & gmask) != 0u;
    const bool in_b2 = (__ballot_sync(gmask, mine && (a.b2 & bit)) & gmask) != 0u;
    const int c = (int)C;
    const bool full = a.n1 + a.n2 >= c;
    vl = -1;
    vs = 0;
    none_left = false;
    if (in_b1 || in_b2) {
        if (in_b1) {
            double q = (double)a.nb2 / (double)a.nb1;
            q = q < 1.0 ? 1.0 : q;
            const double np = a.p + q;
            a.p = (double)c <= np ? (double)c : np;
        } else {
            double q = (double)a.nb1 / (double)a.nb2;
            q = q < 1.0 ? 1.0 : q;
            const double np = a.p - q;
            a.p = 0.0 >= np ? 0.0 : np;
        }
        if (full) {
            warc_replace<EPL>(a, in_b2, pin, gmask, gbase, glane, vl, vs);
            none_left = vl < 0;
        }
        warc_put<EPL>(a, owner, slot, 1, gmask, gbase, glane);
        return;
    }
    const int l1 = a.n1 + a.nb1;
    if (l1 == c) {
        if (a.n1 < c) {
            int bl, bs;
            warc_lru<EPL>(a, a.b1, gmask, gbase, bl, bs);
            warc_put<EPL>(a, bl, bs, 4, gmask, gbase, glane);
            if (a.n1 + a.n2 >= c) {
                warc_replace<EPL>(a, false, pin, gmask, gbase, glane, vl, vs);
                none_left = vl < 0;
            }
        } else {   // B1 empty, T1 full: drop T1's LRU without a ghost entry
            warc_lru<EPL>(a, a.t1 & ~pin, gmask, gbase, vl, vs);
            none_left = vl < 0;
            if (vl >= 0) warc_put<EPL>(a, vl, vs, 4, gmask, gbase, glane);
        }
    } else if (l1 < c) {
        const int total = l1 + a.n2 + a.nb2;
        if (total >= c) {
            if (total == 2 * c) {
                int bl, bs;
                warc_lru<EPL>(a, a.b2, gmask, gbase, bl, bs);
                warc_put<EPL>(a, bl, bs, 4, gmask, gbase, glane);
            }
            if (a.n1 + a.n2 >= c) {
                warc_replace<EPL>(a, false, pin, gmask, gbase, glane, vl, vs);
                none_left = vl < 0;
            }
        }
    }
    warc_put<EPL>(a, owner, slot, 0, gmask, gbase, glane);
}

template <int G, int EPL, int POL, bool UNIFORM>
__device__ __forceinline__ void replay_instance(const ReplayParams &P, int64_t chain, int pol_i, int cap_i,
                                                int64_t inst, int ml_variant) {
    const DevTrace &tr = P.tr;
    const int lane = threadIdx.x & 31;
    const int glane = lane % G;
    const int gbase = lane - glane;
    const unsigned gmask = (G == 32) ? FULL_MASK : (((1u << G) - 1u) << gbase);
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int E = tr.E;

    uint32_t res = 0, pin = 0, seen = 0;
    uint32_t key[EPL], pend[EPL];
    WArc<EPL> arc;
    if (POL == POL_ARC) {
        arc.t1 = arc.t2 = arc.b1 = arc.b2 = 0u;
#pragma unroll
        for (int s = 0; s < EPL; ++s) arc.ord[s] = 0u;
        arc.clock = 0u;
        arc.n1 = arc.n2 = arc.nb1 = arc.nb2 = 0;
        arc.p = 0.0;
    }
    // LeCaR (policies.py:330-395): key[] holds the stamps, kf[] the counts;
    // per lane the ghost-list membership of its experts and their eviction
    // positions; list sizes, weights and the draw counter are group-uniform.
    uint32_t kf[EPL], gpos[EPL], gl = 0u, gf = 0u, n_draw = 0u;
    int ngl = 0, ngf = 0;
    double wl = 0.5, wf = 0.5;
#pragma unroll
    for (int s = 0; s < EPL; ++s) { key[s] = 0; pend[s] = 0; kf[s] = 0; gpos[s] = 0; }
    uint32_t count = 0, ph = 0, pm = 0, dh = 0, dm = 0, nev = 0, comp = 0, refc = 0;
    double dlat = 0.0, plat = 0.0;
    uint64_t h = 0;
    int status = MCB_OK;

    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const int64_t n_ev = tr.ev_end(chain) - e0;
    const int64_t acc_words = (tr.total_acc + 3) >> 2;

    U32Stream<G> ids;   // access ids, 4 per word
    ids.init(tr.acc, acc_words, a0 >> 2, glane);
    U32Stream<G> nx;    // Belady next-use positions, 1 per word
    if (POL == POL_BELADY) nx.init(P.next_pos, tr.total_acc, a0, glane);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;
    uint16_t *outc = P.outcomes ? P.outcomes + ((int64_t)pol_i * P.n_cap + cap_i) * tr.total_acc : nullptr;

    uint32_t nrow[EPL];
#pragma unroll
    for (int s = 0; s < EPL; ++s) {
        const int e = glane * EPL + s;
        nrow[s] = (POL == POL_ML && n_ev > 0 && e < E) ? (uint32_t)__ldcg(rank + e0 * E + e) : 0u;
    }
    uint32_t pos = 0, dec = 0;
    for (int64_t ev = 0; ev < n_ev; ++ev) {
        const uint32_t info = UNIFORM ? mcb_ev_pack((uint32_t)tr.K, (uint32_t)tr.K, true, ev == 0)
                                      : __ldg(tr.ev_info + e0 + ev);
        const uint32_t nacc = mcb_ev_nacc(info);
        const bool decode = mcb_ev_decode(info);
        if (P.res_masks) {   // resident set before the event (dataset.py:61-63)
            uint8_t *m = P.res_masks + (e0 + ev) * E;
#pragma unroll
            for (int s = 0; s < EPL; ++s) {
                const int e = glane * EPL + s;
                if (e < E) m[e] = (uint8_t)((res >> s) & 1u);
            }
        }
        if (POL == POL_LFU && mcb_ev_newseq(info)) {
            // start_sequence: LFU counts reset (policies.py:184-185)
#pragma unroll
            for (int s = 0; s < EPL; ++s) key[s] = 0;
        }
        if (POL == POL_LECAR && mcb_ev_newseq(info)) {
#pragma unroll
            for (int s = 0; s < EPL; ++s) kf[s] = 0;   // start_sequence (policies.py:351-352)
        }
        if (POL == POL_ML) {
            // per-event score ranks (mlpolicy.py:59-62): argmax score == argmin (256 - rank);
            // the next event's row is already in flight (prefetched one event ahead)
#pragma unroll
            for (int s = 0; s < EPL; ++s) {
                key[s] = nrow[s] ? 256u - nrow[s] : KEY_SENT;
                const int e = glane * EPL + s;
                nrow[s] = (ev + 1 < n_ev && e < E) ? (uint32_t)__ldcg(rank + (e0 + ev + 1) * E + e) : 0u;
            }
        }
        pin = 0;
        uint32_t step_miss = 0;
        for (uint32_t j = 0; j < nacc; ++j, ++pos) {
            const int64_t A = a0 + pos;
            const uint32_t word = ids.get(A >> 2, glane, gbase, gmask);
            const uint32_t x = (word >> (8 * (uint32_t)(A & 3))) & 0xFFu;
            const int owner = (int)(x / EPL);
            const int slot = (int)(x % EPL);
            const bool mine = glane == owner;
            const uint32_t bit = 1u << slot;
            const bool hit = (__ballot_sync(gmask, mine && (res & bit)) & gmask) != 0u;
            if (POL == POL_BELADY) {
                const uint32_t np = nx.get(A, glane, gbase, gmask);
                if (mine) set_slot<EPL>(key, slot, ~np);
            }
            if ((POL == POL_LRU || POL == POL_LECAR) && mine) set_slot<EPL>(key, slot, pos);
            if (POL == POL_LECAR && mine) set_slot<EPL>(kf, slot, get_slot<EPL>(kf, slot) + 1u);
            if (POL == POL_LFU && mine) set_slot<EPL>(key, slot, get_slot<EPL>(key, slot) + 1u);
            uint32_t code = MCB_OUT_HIT;
            if (hit) {
                if (decode) ++dh; else ++ph;
                if (POL == POL_ARC) warc_put<EPL>(arc, owner, slot, 1, gmask, gbase, glane);   // to T2's MRU end
            } else {
                if (decode) ++dm; else ++pm;
                ++step_miss;
                if (POL == POL_LECAR) {   // _on_miss ghost hit: regret update (policies.py:358-367)
                    const bool in_gl = (__ballot_sync(gmask, mine && (gl & bit)) & gmask) != 0u;
                    const bool in_gf = (__ballot_sync(gmask, mine && (gf & bit)) & gmask) != 0u;
                    if (in_gl || in_gf) {
                        const uint32_t gp = __shfl_sync(gmask, get_slot<EPL>(gpos, slot), gbase + owner);
                        lecar_reward(wl, wf, in_gl, lecar_factor(P, cap_i, pos - gp));
                        if (mine) { gl &= ~bit; gf &= ~bit; }
                        if (in_gl) --ngl;
                        else --ngf;
                    }
                }
                if (POL == POL_ARC) {
                    int vl, vs;
                    bool none_left;
                    warc_miss<EPL>(arc, owner, slot, pin, C, gmask, gbase, glane, vl, vs, none_left);
                    if (none_left) { status = MCB_ERR_NO_EVICTABLE; break; }
                    res = arc.t1 | arc.t2;
                    count = (uint32_t)(arc.n1 + arc.n2);
                    if (vl >= 0) {
                        if (glane == vl) set_slot<EPL>(pend, vs, dec + 1u);
                        code = (uint32_t)(vl * EPL + vs);
                        ++nev;
                    } else {
                        code = MCB_OUT_MISS;
                    }
                } else if (count >= C) {
                    const uint32_t cand = res & ~pin;
                    bool use_lru = true;
                    if (POL == POL_LECAR) {   // _choose_victim (policies.py:379-395)
                        use_lru = __ldg(P.lecar_u + n_draw) < wl;
                        ++n_draw;
                    }
                    uint32_t lk = KEY_SENT;
                    int ls = 0;
#pragma unroll
                    for (int s = 0; s < EPL; ++s) {
                        const uint32_t ks = (POL == POL_LECAR && !use_lru) ? kf[s] : key[s];
                        if (((cand >> s) & 1u) && ks < lk) { lk = ks; ls = s; }
                    }
                    const uint32_t m = __reduce_min_sync(gmask, lk);
                    if (m == KEY_SENT) { status = MCB_ERR_NO_EVICTABLE; break; }
                    const unsigned b = __ballot_sync(gmask, lk == m) & gmask;
                    const int wl = __ffs(b) - 1;
                    const int vs = __shfl_sync(gmask, ls, wl);
                    const int vlane = wl - gbase;
                    if (glane == vlane) {
                        res &= ~(1u << vs);
                        set_slot<EPL>(pend, vs, dec + 1u);
                    }
                    code = (uint32_t)(vlane * EPL + vs);
                    ++nev;
                    if (POL == POL_LECAR) {   // ghost[victim] = position; trim to capacity
                        if (glane == vlane) {
                            set_slot<EPL>(gpos, vs, pos);
                            if (use_lru) gl |= 1u << vs;
                            else gf |= 1u << vs;
                        }
                        int &ng = use_lru ? ngl : ngf;
                        if (++ng > (int)C) {
                            const uint32_t g = use_lru ? gl : gf;
                            uint32_t ok = KEY_SENT;
                            int os = 0;
#pragma unroll
                            for (int s = 0; s < EPL; ++s)
                                if (((g >> s) & 1u) && gpos[s] < ok) { ok = gpos[s]; os = s; }
                            const uint32_t om = __reduce_min_sync(gmask, ok);
                            const int ol = __ffs(__ballot_sync(gmask, ok == om) & gmask) - 1;
                            if (lane == ol) {
                                gl &= ~(1u << os);
                                gf &= ~(1u << os);
                            }
                            --ng;
                        }
                    }
                } else {
                    ++count;
                    code = MCB_OUT_MISS;
                }
                if (mine) {
                    // compulsory (engine.py:248-250) and refetch of an earlier
                    // victim (engine.py:289-296): its first access after the
                    // eviction is necessarily this miss
                    if (!(seen & bit)) {
                        ++comp;
                    } else {
                        const uint32_t pe = get_slot<EPL>(pend, slot);
                        if (pe && (int64_t)dec - (int64_t)(pe - 1u) <= (int64_t)P.window) ++refc;
                    }
                    set_slot<EPL>(pend, slot, 0u);
                    seen |= bit;
                    res |= bit;
                    if (POL == POL_FIFO) set_slot<EPL>(key, slot, pos);   // arrival (policies.py:159-161)
                }
            }
            if (decode && mine) pin |= bit;
            if (outc) {
                h = poly16(h, code);
                if (glane == 0) outc[A] = (uint16_t)code;
            } else if (P.hashes) {
                h = poly16(h, code);
            }
        }
        if (status != MCB_OK) break;
        // step_latency_s (engine.py:58-62) accumulated in event order (engine.py:258-262)
        double lat;
        if (step_miss > 0)
            lat = __dmul_rn((double)(P.loads_serial ? step_miss : 1u), P.t_load);
        else
            lat = __dmul_rn((double)nacc, P.t_compute);
        if (decode) dlat = __dadd_rn(dlat, __dadd_rn(lat, POL == POL_ML ? P.ml_cost : 0.0));
        else plat = __dadd_rn(plat, lat);
        if (decode) ++dec;
    }
    comp = __reduce_add_sync(gmask, comp);
    refc = __reduce_add_sync(gmask, refc);
    if (glane == 0) {
        int64_t *o = P.inst_out + inst * MCB_R_N;
        o[MCB_R_PREFILL_HITS] = ph;
        o[MCB_R_PREFILL_MISSES] = pm;
        o[MCB_R_DECODE_HITS] = dh;
        o[MCB_R_DECODE_MISSES] = dm;
        o[MCB_R_COMPULSORY] = comp;
        o[MCB_R_EVICTIONS] = nev;
        o[MCB_R_REFETCHED] = refc;
        o[MCB_R_STATUS] = status;
        P.inst_lat[inst * 2 + 0] = dlat;
        P.inst_lat[inst * 2 + 1] = plat;
        if (P.hashes) P.hashes[inst] = h;
    }
}

template <int G, int EPL, bool UNIFORM>
__global__ void __launch_bounds__(128) k_replay(const __grid_constant__ ReplayParams P) {
    const int64_t li = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;   // instance of this launch
    const int64_t n_inst = (P.chain_hi - P.chain_lo) * P.n_pol_launch * P.n_cap;
    if (li >= n_inst) return;
    const int cap_i = (int)(li % P.n_cap);
    const int pol_i = P.pol_map[(li / P.n_cap) % P.n_pol_launch];
    const int64_t chain = P.chain_lo + li / ((int64_t)P.n_cap * P.n_pol_launch);
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    switch (P.pol[pol_i]) {
        case MCB_LRU: replay_instance<G, EPL, POL_LRU, UNIFORM>(P, chain, pol_i, cap_i, inst, 0); break;
        case MCB_LFU: replay_instance<G, EPL, POL_LFU, UNIFORM>(P, chain, pol_i, cap_i, inst, 0); break;
        case MCB_BELADY: replay_instance<G, EPL, POL_BELADY, UNIFORM>(P, chain, pol_i, cap_i, inst, 0); break;
        case MCB_ML: replay_instance<G, EPL, POL_ML, UNIFORM>(P, chain, pol_i, cap_i, inst, 0); break;
        case MCB_FIFO: replay_instance<G, EPL, POL_FIFO, UNIFORM>(P, chain, pol_i, cap_i, inst, 0); break;
        case MCB_ARC: replay_instance<G, EPL, POL_ARC, UNIFORM>(P, chain, pol_i, cap_i, inst, 0); break;
        case MCB_LECAR: replay_instance<G, EPL, POL_LECAR, UNIFORM>(P, chain, pol_i, cap_i, inst, 0); break;
        default: replay_instance<G, EPL, POL_ML, UNIFORM>(P, chain, pol_i, cap_i, inst, 1); break;
    }
}

// ---------------------------------------------------------------------------
// K4-solo: one THREAD per cache instance, for num_experts <= 16.  All state
// (resident mask, refetch ring, the packed per-expert keys, counters) lives
// in registers, so an access costs no cross-lane traffic; the per-access step
// is sstep() (mcb_solo.cuh), shared with the segmented replay.  blockIdx.y
// selects the policy, so a warp never diverges on policy; the threads of a
// warp share chains (consecutive capacities of one chain), so their id /
// next-use / rank loads coalesce into broadcasts.
// ---------------------------------------------------------------------------
template <int EM, int POL, bool UNIFORM, int WMAX>
__device__ __forceinline__ void solo_instance(const ReplayParams &P, int64_t chain, int pol_i, int cap_i, int ml_variant) {
    constexpr int SH = Solo<EM>::SH;
    const DevTrace &tr = P.tr;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int E = tr.E;
    const int W = P.window;          // 0 <= W <= WMAX (checked at launch)
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;

    uint32_t pk[EM];                 // packed keys (key << SH | id), all experts
#pragma unroll
    for (int s = 0; s < EM; ++s) pk[s] = (uint32_t)s;
    SState<WMAX> S;
    sstate_clear(S);
    ArcState<EM> arc;
    if (POL == POL_ARC) arc_clear<EM>(arc);
    LecarState<EM> lec;
    if (POL == POL_LECAR) lecar_clear<EM>(lec);
    uint32_t pin = 0, seen = 0, valid = (1u << E) - 1u;
    uint32_t ph = 0, pm = 0, dh = 0, dm = 0, comp = 0;
    SCount n = {0u, 0u, 0u};
    double dlat = 0.0, plat = 0.0;
    uint64_t h = 0;
    bool stuck = false;

    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const int64_t n_ev = tr.ev_end(chain) - e0;
    const int64_t a_end = tr.acc_end(chain);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;
    uint16_t *outc = P.outcomes ? P.outcomes + ((int64_t)pol_i * P.n_cap + cap_i) * tr.total_acc : nullptr;
    const bool track = outc != nullptr || P.hashes != nullptr;

    IdReader ids;
    ids.init(tr.acc, a0, a_end);
    NextReader nx;
    if (POL == POL_BELADY) nx.init(P.next_pos, a0, a_end);
    uint32_t rrow[EM];
    if (POL == POL_ML && n_ev > 0) load_rank_row<EM>(rrow, rank + e0 * E, E);
    uint32_t info_next = (!UNIFORM && n_ev > 0) ? __ldg(tr.ev_info + e0) : 0u;

    int64_t A = a0;
    uint32_t pos = 0;
    for (int64_t ev = 0; ev < n_ev; ++ev) {
        uint32_t info;
        if (UNIFORM) {
            info = mcb_ev_pack((uint32_t)tr.K, (uint32_t)tr.K, true, ev == 0);
        } else {
            info = info_next;
            info_next = ev + 1 < n_ev ? __ldg(tr.ev_info + e0 + ev + 1) : 0u;
        }
        const uint32_t nacc = mcb_ev_nacc(info);
        const bool decode = UNIFORM ? true : mcb_ev_decode(info);
        if (POL == POL_LFU && !UNIFORM && mcb_ev_newseq(info)) {
#pragma unroll
            for (int s = 0; s < EM; ++s) pk[s] = (uint32_t)s;   // start_sequence (policies.py:184-185)
        }
        if (POL == POL_LECAR && !UNIFORM && mcb_ev_newseq(info)) lecar_new_sequence<EM>(lec);
        if (P.res_masks) {   // resident set before the event (dataset.py:61-63)
            uint8_t *m = P.res_masks + (e0 + ev) * E;
            for (int e = 0; e < E; ++e) m[e] = (uint8_t)((S.res >> e) & 1u);
        }
        if (POL == POL_ML) {
            solo_ml_keys<EM>(pk, valid, rrow);   // this event's rank row (mlpolicy.py:59-62)
            if (ev + 1 < n_ev) load_rank_row<EM>(rrow, rank + (e0 + ev + 1) * E, E);
        }
        pin = 0;
        uint32_t step_miss = 0;
        for (uint32_t j = 0; j < nacc; ++j, ++pos, ++A) {
            const uint32_t x = ids.get(A);
            const uint32_t bit = 1u << x;
            const uint32_t np = (POL == POL_BELADY) ? nx.get(A) : 0u;
            solo_key_update<EM, POL>(pk, x, bit, pos, np);
            uint32_t miss;
            uint32_t code;
            if (POL == POL_ARC) {
                code = sstep_arc<EM, WMAX>(S, arc, x, bit, decode ? pin : 0u, C, n, stuck, miss);
            } else if (POL == POL_LECAR) {
                code = sstep_lecar<EM, WMAX>(S, lec, P, cap_i, x, bit, pos, pin, C, n, stuck, miss);
            } else {
                code = sstep<EM, WMAX>(S, pk, bit, pin, valid, C, n, stuck, miss);
                if (POL == POL_FIFO) solo_fifo_insert<EM>(pk, x, bit, pos, miss);
            }
            step_miss += miss;
            if (decode) { dh += 1u - miss; dm += miss; }
            else { ph += 1u - miss; pm += miss; }
            comp += (miss && !(seen & bit)) ? 1u : 0u;   // compulsory (engine.py:248-250)
            seen |= bit;
            pin |= decode ? bit : 0u;
            if (track) {
                h = poly16(h, code);
                if (outc) outc[A] = (uint16_t)code;
            }
        }
        double lat;
        if (step_miss > 0)
            lat = __dmul_rn((double)(P.loads_serial ? step_miss : 1u), P.t_load);
        else
            lat = __dmul_rn((double)nacc, P.t_compute);
        if (decode) {
            dlat = __dadd_rn(dlat, __dadd_rn(lat, POL == POL_ML ? P.ml_cost : 0.0));
            sstate_next_decode<WMAX>(S, W);
        } else {
            plat = __dadd_rn(plat, lat);
        }
    }
    (void)SH;
    int64_t *o = P.inst_out + inst * MCB_R_N;
    o[MCB_R_PREFILL_HITS] = ph;
    o[MCB_R_PREFILL_MISSES] = pm;
    o[MCB_R_DECODE_HITS] = dh;
    o[MCB_R_DECODE_MISSES] = dm;
    o[MCB_R_COMPULSORY] = comp;
    o[MCB_R_EVICTIONS] = n.nev;
    o[MCB_R_REFETCHED] = n.refc;
    o[MCB_R_STATUS] = stuck ? MCB_ERR_NO_EVICTABLE : MCB_OK;
    P.inst_lat[inst * 2 + 0] = dlat;
    P.inst_lat[inst * 2 + 1] = plat;
    if (P.hashes) P.hashes[inst] = h;
}

template <int EM, bool UNIFORM>
__global__ void __launch_bounds__(128) k_replay_solo(const __grid_constant__ ReplayParams P) {
    const int pol_i = P.pol_map[blockIdx.y];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (P.chain_hi - P.chain_lo) * P.n_cap) return;
    const int cap_i = (int)(t % P.n_cap);
    const int64_t chain = P.chain_lo + t / P.n_cap;
    switch (P.pol[pol_i]) {
        case MCB_LRU: solo_instance<EM, POL_LRU, UNIFORM, SOLO_WMAX>(P, chain, pol_i, cap_i, 0); break;
        case MCB_LFU: solo_instance<EM, POL_LFU, UNIFORM, SOLO_WMAX>(P, chain, pol_i, cap_i, 0); break;
        case MCB_BELADY: solo_instance<EM, POL_BELADY, UNIFORM, SOLO_WMAX>(P, chain, pol_i, cap_i, 0); break;
        case MCB_ML: solo_instance<EM, POL_ML, UNIFORM, SOLO_WMAX>(P, chain, pol_i, cap_i, 0); break;
        case MCB_FIFO: solo_instance<EM, POL_FIFO, UNIFORM, SOLO_WMAX>(P, chain, pol_i, cap_i, 0); break;
        case MCB_ARC: solo_instance<EM, POL_ARC, UNIFORM, SOLO_WMAX>(P, chain, pol_i, cap_i, 0); break;
        case MCB_LECAR: solo_instance<EM, POL_LECAR, UNIFORM, SOLO_WMAX>(P, chain, pol_i, cap_i, 0); break;
        default: solo_instance<EM, POL_ML, UNIFORM, SOLO_WMAX>(P, chain, pol_i, cap_i, 1); break;
    }
}

template <int EM>
static void launch_solo_t(const ReplayParams &p, cudaStream_t s) {
    const int64_t n = (p.chain_hi - p.chain_lo) * p.n_cap;
    // Few instances (latency-bound chains, e.g. one Mixtral trace): one warp
    // per block, with a shared-memory reservation that keeps other kernels'
    // blocks (the concurrently running K3) off its SM, so each replay warp
    // issues alone.  Many instances: ordinary 128-thread blocks.
    const int64_t warps = (n + 31) / 32 * p.n_pol_launch;
    const bool exclusive = warps <= 64;
    const int bs = exclusive ? 32 : 128;
    const size_t smem = exclusive ? (size_t)160 * 1024 : 0;
    const dim3 grid((unsigned)((n + bs - 1) / bs), (unsigned)p.n_pol_launch);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_replay_solo<EM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(k_replay_solo<EM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr_set = true;
    }
    if (p.tr.uniform) k_replay_solo<EM, true><<<grid, bs, smem, s>>>(p);
    else k_replay_solo<EM, false><<<grid, bs, smem, s>>>(p);
}

template <int G, int EPL>
static void launch_replay_t(const ReplayParams &p, cudaStream_t s) {
    const int64_t n_inst = (p.chain_hi - p.chain_lo) * p.n_pol_launch * p.n_cap;
    const int per_block = 128 / G;
    const unsigned blocks = (unsigned)((n_inst + per_block - 1) / per_block);
    if (p.tr.uniform) k_replay<G, EPL, true><<<blocks, 128, 0, s>>>(p);
    else k_replay<G, EPL, false><<<blocks, 128, 0, s>>>(p);
}

int launch_replay(const ReplayParams &p, cudaStream_t s) {
    if ((p.chain_hi - p.chain_lo) * p.n_pol_launch * p.n_cap == 0) return 0;
    const int E = p.tr.E;
    // solo kernels pack (key << 3|4 | id) into 32 bits: chains must stay below 2^28 accesses.
    // Thread-per-instance only pays off when there are enough instances to
    // fill the machine; few long chains (e.g. one Mixtral trace) are
    // latency-bound, and a whole warp per instance has the shorter per-access
    // critical path (lane-parallel victim search, no divergence).
    const int64_t n_inst = (p.chain_hi - p.chain_lo) * p.n_pol_launch * p.n_cap;
    const int64_t chain_bound = p.tr.uniform ? p.tr.T * p.tr.K : p.tr.total_acc;   // longest chain (upper bound)
    const bool solo_ok = chain_bound < (1ll << 27) && n_inst >= p.solo_min_instances && p.window >= 0 &&
                         p.window <= SOLO_WMAX;
    if (E <= 8 && solo_ok) { launch_solo_t<8>(p, s); return 1; }
    if (E <= 16 && solo_ok) { launch_solo_t<16>(p, s); return 1; }
    // many instances of 16 < E <= 128 (e.g. C4's 4,096 traces): one thread per instance
    if (n_inst >= p.wide_min_instances)
        if (const int n_wide = launch_replay_wide(p, s)) return n_wide;   // one launch per policy
    // Lane-group size: one whole warp per instance by default.  Groups of 8 /
    // 16 lanes (4 / 2 instances per warp) are available through
    // MCB_TUNE_GROUP_LANES but measured slower even with many instances
    // (c4-shaped, 20K instances: 32 lanes 11.8e9, 16 lanes 8.5e9, 8 lanes
    // 7.8e9 accesses/s): the groups of a warp diverge on hit / miss.
    int G = p.group_lanes > 0 ? p.group_lanes : 32;
    const int gmin = E <= 64 ? 8 : 16;   // at most 8 experts per lane
    if (G < gmin) G = gmin;
    if (E <= 32) {
        if (G == 8) launch_replay_t<8, 4>(p, s);
        else if (G == 16) launch_replay_t<16, 2>(p, s);
        else launch_replay_t<32, 1>(p, s);
    } else if (E <= 64) {
        if (G == 8) launch_replay_t<8, 8>(p, s);
        else if (G == 16) launch_replay_t<16, 4>(p, s);
        else launch_replay_t<32, 2>(p, s);
    } else {
        if (G == 16) launch_replay_t<16, 8>(p, s);
        else launch_replay_t<32, 4>(p, s);
    }
    return 1;
}

// ===========================================================================
// K5: fold chains -> (trace, policy, capacity) in layer order (engine.py:330-343)
// ===========================================================================
__global__ void k_fold(const __grid_constant__ ReplayParams P, int num_traces, int64_t *__restrict__ reports,
                       double *__restrict__ latency) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)num_traces * P.n_pol * P.n_cap;
    if (i >= n) return;
    const int cap_i = (int)(i % P.n_cap);
    const int pol_i = (int)((i / P.n_cap) % P.n_pol);
    const int64_t trace = i / ((int64_t)P.n_cap * P.n_pol);
    int64_t acc[MCB_R_N] = {0, 0, 0, 0, 0, 0, 0, 0};
    double dl = 0.0, pl = 0.0;
    for (int l = 0; l < P.tr.L; ++l) {
        const int64_t chain = trace * P.tr.L + l;
        const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
        const int64_t *o = P.inst_out + inst * MCB_R_N;
#pragma unroll
        for (int k = 0; k < MCB_R_STATUS; ++k) acc[k] += o[k];
        if (acc[MCB_R_STATUS] == 0 && o[MCB_R_STATUS] != 0) acc[MCB_R_STATUS] = o[MCB_R_STATUS];
        dl = __dadd_rn(dl, P.inst_lat[inst * 2 + 0]);
        pl = __dadd_rn(pl, P.inst_lat[inst * 2 + 1]);
    }
#pragma unroll
    for (int k = 0; k < MCB_R_N; ++k) reports[i * MCB_R_N + k] = acc[k];
    latency[i * 2 + 0] = dl;
    latency[i * 2 + 1] = pl;
}

int launch_fold(const ReplayParams &p, int num_traces, int64_t *reports, double *latency, cudaStream_t s) {
    const int64_t n = (int64_t)num_traces * p.n_pol * p.n_cap;
    if (n == 0) return 0;
    k_fold<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(p, num_traces, reports, latency);
    return 1;
}

// ===========================================================================
// K3: ML scorer.
// ===========================================================================
// Prepared weights per net for the fp64 tensor-core MLP (all K-major
// "[K][N]" so a B fragment is 4 rows x 8 contiguous columns), zero-padded to
// the tile granularity: Hp = round_up(H, 8) hidden units, Kp1 = round_up(2E, 4)
// input features, Ep = round_up(E, 8) outputs.  Padded units / features carry
// zero weights and biases, so they contribute exact zeros.
//   Wt1[Kp1][Hp] b1[Hp] Wt2[Hp][Hp] b2[Hp] Wt3[Hp][Ep] b3[Ep]
__host__ __device__ int mlp_hp(int H) { return (H + 7) / 8 * 8; }
__host__ __device__ int mlp_kp1(int E) { return (2 * E + 3) / 4 * 4; }
__host__ __device__ int mlp_ep(int E) { return (E + 7) / 8 * 8; }
__host__ __device__ size_t prepared_net_doubles(int E, int H) {
    const size_t Hp = mlp_hp(H), Kp1 = mlp_kp1(E), Ep = mlp_ep(E);
    return Kp1 * Hp + Hp + Hp * Hp + Hp + Hp * Ep + Ep;
}
// .evnet parameter count per net (net.py:282-305): w1[H][2E] b1 w2[H][H] b2 w3[E][H] b3
__host__ __device__ size_t net_param_doubles(int E, int H) {
    const size_t D = 2 * (size_t)E;
    return D * H + H + (size_t)H * H + H + (size_t)H * E + E;
}

__global__ void k_prepare_nets(const double *__restrict__ params, int E, int H, int num_nets,
                               double *__restrict__ wt) {
    const int D = 2 * E, Hp = mlp_hp(H), Kp1 = mlp_kp1(E), Ep = mlp_ep(E);
    const int64_t per = (int64_t)prepared_net_doubles(E, H), src_per = (int64_t)net_param_doubles(E, H);
    const int64_t total = per * num_nets;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t net = i / per;
        int64_t r = i % per;
        const double *src = params + net * src_per;
        // source offsets (.evnet): w1[H][D] b1 w2[H][H] b2 w3[E][H] b3
        const int64_t s_w1 = 0, s_b1 = (int64_t)H * D, s_w2 = s_b1 + H, s_b2 = s_w2 + (int64_t)H * H,
                      s_w3 = s_b2 + H, s_b3 = s_w3 + (int64_t)E * H;
        double v = 0.0;
        if (r < (int64_t)Kp1 * Hp) {                      // Wt1[k][h] = w1[h][k]
            const int64_t k = r / Hp, hh = r % Hp;
            if (k < D && hh < H) v = src[s_w1 + hh * D + k];
        } else if ((r -= (int64_t)Kp1 * Hp) < Hp) {
            if (r < H) v = src[s_b1 + r];
        } else if ((r -= Hp) < (int64_t)Hp * Hp) {        // Wt2[k][h] = w2[h][k]
            const int64_t k = r / Hp, hh = r % Hp;
            if (k < H && hh < H) v = src[s_w2 + hh * H + k];
        } else if ((r -= (int64_t)Hp * Hp) < Hp) {
            if (r < H) v = src[s_b2 + r];
        } else if ((r -= Hp) < (int64_t)Hp * Ep) {        // Wt3[k][e] = w3[e][k]
            const int64_t k = r / Ep, e = r % Ep;
            if (k < H && e < E) v = src[s_w3 + e * H + k];
        } else {
            r -= (int64_t)Hp * Ep;
            if (r < E) v = src[s_b3 + r];
        }
        wt[i] = v;
    }
}

int launch_prepare_nets(const double *params, int E, int H, int num_nets, double *wt, cudaStream_t s) {
    const int64_t total = (int64_t)prepared_net_doubles(E, H) * num_nets;
    const unsigned blocks = (unsigned)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    k_prepare_nets<<<blocks, 256, 0, s>>>(params, E, H, num_nets, wt);
    return 1;
}

// Snapshot record per tile: last[E] (update index of the last routing, -1 =
// never), freq[E], u (updates since the sequence start), rt_lo, rt_hi
// (routed-list offset of the tile's first event within the chain).
__host__ __device__ __forceinline__ int snap_stride(int E) { return 2 * E + 4; }

__global__ void k_tile_offsets(DevTrace tr, int64_t *__restrict__ tile_off) {
    // single block exclusive scan of ceil(n_ev / TILE) over chains
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < tr.n_chains; base += blockDim.x) {
        const int64_t c = base + threadIdx.x;
        int64_t v = 0;
        if (c < tr.n_chains) v = (tr.ev_end(c) - tr.ev_begin(c) + MCB_TILE_EV - 1) / MCB_TILE_EV;
        // block inclusive scan (Hillis-Steele in shared memory)
        __shared__ int64_t buf[1024];
        buf[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < (int)blockDim.x; o <<= 1) {
            const int64_t add = threadIdx.x >= (unsigned)o ? buf[threadIdx.x - o] : 0;
            __syncthreads();
            buf[threadIdx.x] += add;
            __syncthreads();
        }
        if (c < tr.n_chains) tile_off[c] = carry + buf[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += buf[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0) tile_off[tr.n_chains] = carry;
}

__device__ __forceinline__ int64_t chain_tile_begin(const DevTrace &tr, const int64_t *tile_off, int64_t c) {
    if (tr.uniform) return c * ((tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV);
    return tile_off[c];
}

// One warp per chain: sequential FeatureTracker scan (features.py:34-39),
// reset at sequence boundaries (mlpolicy.py:56-57), updates only for decode
// events unless include_prefill (mlpolicy.py:59-61).
__global__ void __launch_bounds__(128) k_feat_snap(DevTrace tr, int include_prefill, const int64_t *tile_off,
                                                   int32_t *__restrict__ snaps) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (c >= tr.n_chains) return;
    const int E = tr.E;
    const int SN = snap_stride(E);
    int32_t last[4], f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) { last[j] = -1; f[j] = 0; }
    int32_t u = 0;
    const int64_t e0 = tr.ev_begin(c), n_ev = tr.ev_end(c) - e0;
    const uint8_t *routed = tr.routed_ptr() + tr.rt_begin(c);
    int64_t rt = 0;
    int64_t tile = chain_tile_begin(tr, tile_off, c);
    for (int64_t ev = 0; ev < n_ev; ++ev) {
        const uint32_t info = tr.info(c, e0 + ev);
        if (ev % MCB_TILE_EV == 0) {
            int32_t *sp = snaps + tile * SN;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int e = lane + 32 * j;
                if (e < E) { sp[e] = last[j]; sp[E + e] = f[j]; }
            }
            if (lane == 0) { sp[2 * E] = u; sp[2 * E + 1] = (int32_t)(rt & 0xFFFFFFFF); sp[2 * E + 2] = (int32_t)(rt >> 32); }
            ++tile;
        }
        if (mcb_ev_newseq(info)) {
#pragma unroll
            for (int j = 0; j < 4; ++j) { last[j] = -1; f[j] = 0; }
            u = 0;
        }
        const uint32_t nrt = mcb_ev_nrt(info);
        if (mcb_ev_decode(info) || include_prefill) {
            ++u;
            for (uint32_t r = 0; r < nrt; ++r) {
                const int x = __ldg(routed + rt + r);
                if ((x & 31) == lane) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        { const bool hit_j = (x >> 5) == j; last[j] = hit_j ? u : last[j]; f[j] += hit_j ? 1 : 0; }
                }
            }
        }
        rt += nrt;
    }
}

// exp(x) for x <= 0 in float64, branch-free, table-driven: k = rint(64 x /
// ln2), x = k ln2/64 + r with |r| <= ln2/128, exp(x) = 2^(k>>6) * T[k&63] *
// exp(r) with T[j] = 2^(j/64) (shared-memory table, correctly rounded) and
// exp(r) by its degree-5 Taylor polynomial (truncation < 2^-54).  Within a
// few ulp of the correctly rounded exp for x >= -708.
__device__ double g_exp2_64[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284, 1.0442737824274138, 1.0556451783605572,
    1.0671404006768237, 1.0787607977571199, 1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
    1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812, 1.189207115002721, 1.202156731452703,
    1.215247359980469, 1.22848053610687, 1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
    1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303, 1.3542555469368927, 1.3690024229745905,
    1.383909881963832, 1.3989796725383112, 1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
    1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384, 1.5422108254079407, 1.559004400237837,
    1.5759808451078865, 1.593142151342267, 1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
    1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062, 1.7562521603732995, 1.7753764925265212,
    1.7947090750031072, 1.8142521755003989, 1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
    1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951};
__device__ __forceinline__ double exp_nonpos(double x, const double *tab) {
    // literal coefficients: they become constant-bank operands of the DFMAs
    // (no separate uniform loads); x < -708 is clamped (its logistic is below
    // 1e-307, so the SiLU output differs from the reference's by < 1e-304
    // absolute, far below the ulp of any score)
    x = fmax(x, -708.0);
    const double kd = rint(x * 92.33248261689366);                 // 64 / ln2
    double r = fma(kd, -0.010830424696249145, x);                  // -(ln2/64) hi
    r = fma(kd, -3.623510646634843e-19, r);                        // -(ln2/64) lo
    double p = fma(1.0 / 120.0, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const int k = (int)kd;
    const double m = __dmul_rn(tab[k & 63], p);
    const int hi = __double2hiint(m) + ((k >> 6) << 20);
    return __hiloint2double(hi, __double2loint(m));
}

// 1/d for d in [1, 2]: hardware float64 reciprocal approximation (MUFU.RCP64H)
// and two Newton steps (error below one ulp of the double result).
__device__ __forceinline__ double rcp_1_2(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}

// logistic(z) of net.py:43-49 (sign-split: 1/(1+e^-z) for z >= 0,
// e^z/(1+e^z) otherwise), evaluated branch-free from e = exp(-|z|) so lanes
// of both signs share one exp and one reciprocal; agrees with the reference
// to a few ulp (ranks are checked for near-ties at 1e-12, see k_score_tile).
__device__ __forceinline__ double sigmoid_ref(double z, const double *tab) {
    const double e = exp_nonpos(-fabs(z), tab);
    const double r = rcp_1_2(1.0 + e);
    return z >= 0.0 ? r : __dmul_rn(e, r);
}

// Uniform traces (decode-only, one sequence per chain): the tracker state at
// a tile start is a prefix over earlier tiles, computed in two parallel
// passes instead of one sequential walk per chain:
//   k_tile_summary  one warp per tile: per-expert routing count in the tile
//                   and the 1-based index of its last routing in the tile
//   k_snap_scan     one warp per (chain, 32 experts): walk over its tiles ->
//                   snapshot (last update index, count, u) at every tile start
__global__ void __launch_bounds__(128) k_tile_summary(DevTrace tr, int32_t *__restrict__ summ) {
    // one warp per 32-event tile: lane i marks bit i of occ[e] for each
    // expert e its event routes to; then per expert count = popc(occ),
    // last routing (1-based) = 32 - clz(occ)
    static_assert(MCB_TILE_EV == 32, "one lane per event of a tile");
    __shared__ uint32_t occ_s[4][MCB_MAX_EXPERTS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t tile = (int64_t)blockIdx.x * 4 + w;
    const int64_t tpc = (tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
    if (tile >= tr.n_chains * tpc) return;
    const int64_t c = tile / tpc, ev0 = (tile % tpc) * MCB_TILE_EV;
    const int nev = (int)min((int64_t)MCB_TILE_EV, tr.T - ev0);
    const int E = tr.E, K = tr.K;
    uint32_t *occ = occ_s[w];
    for (int e = lane; e < E; e += 32) occ[e] = 0u;
    __syncwarp();
    if (lane < nev) {
        const uint8_t *ids = tr.acc + (c * tr.T + ev0 + lane) * K;
        for (int k = 0; k < K; ++k) atomicOr(&occ[__ldg(ids + k)], 1u << lane);
    }
    __syncwarp();
    int32_t *o = summ + tile * 2 * E;
    for (int e = lane; e < E; e += 32) {
        const uint32_t m = occ[e];
        o[e] = __popc(m);
        o[E + e] = m ? 32 - __clz(m) : 0;
    }
}

// Few long chains (C3: 16 chains of 32K tiles): one warp per (chain, expert),
// 32 tiles at a time, lane j = tile t0 + j,
// warp-wide exclusive prefix sum of the routing counts and prefix max of the
// last-routing update index (u at a tile start is t * TILE for decode-only
// single-sequence chains), carried across chunks.
__global__ void __launch_bounds__(128) k_snap_scan_tiles(DevTrace tr, const int32_t *__restrict__ summ,
                                                   int32_t *__restrict__ snaps) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int E = tr.E, SN = 2 * E + 4;
    const int64_t c = wid / E;
    const int e = (int)(wid % E);
    if (c >= tr.n_chains) return;
    const int64_t tpc = (tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
    int32_t carry_f = 0, carry_last = -1;
    for (int64_t t0 = 0; t0 < tpc; t0 += 32) {
        const int64_t t = t0 + lane;
        const bool ok = t < tpc;
        const int32_t *sm = summ + (c * tpc + (ok ? t : 0)) * 2 * E;
        const int32_t cnt = ok ? __ldg(sm + e) : 0;
        const int32_t l = ok ? __ldg(sm + E + e) : 0;
        const int32_t la = l > 0 ? (int32_t)(t * MCB_TILE_EV) + l : -1;
        int32_t incl_f = cnt, incl_l = la;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t vf = __shfl_up_sync(FULL_MASK, incl_f, o);
            const int32_t vl = __shfl_up_sync(FULL_MASK, incl_l, o);
            if (lane >= o) { incl_f += vf; incl_l = max(incl_l, vl); }
        }
        const int32_t ex_f = __shfl_up_sync(FULL_MASK, incl_f, 1), ex_l = __shfl_up_sync(FULL_MASK, incl_l, 1);
        const int32_t f_before = carry_f + (lane ? ex_f : 0);
        const int32_t l_before = max(carry_last, lane ? ex_l : -1);
        if (ok) {
            int32_t *sp = snaps + (c * tpc + t) * SN;
            sp[e] = l_before;
            sp[E + e] = f_before;
            if (e == 0) {
                const int64_t rt = t * MCB_TILE_EV * (int64_t)tr.K;
                sp[2 * E] = (int32_t)(t * MCB_TILE_EV);
                sp[2 * E + 1] = (int32_t)(rt & 0xFFFFFFFF);
                sp[2 * E + 2] = (int32_t)(rt >> 32);
            }
        }
        carry_f += __shfl_sync(FULL_MASK, incl_f, 31);
        carry_last = max(carry_last, __shfl_sync(FULL_MASK, incl_l, 31));
    }
}

// One warp per (chain, 32 experts), lane = expert: a sequential walk over
// the chain's tiles carrying (count, last routing) -- every load and store is
// one coalesced row segment (the tile-per-lane scan read and wrote one 4-byte
// word per 512-byte row).  u at a tile start is t * TILE for decode-only
// single-sequence chains; later tiles have later update indices, so the last
// routing before tile t is the latest non-empty tile's.
__global__ void __launch_bounds__(128) k_snap_scan(DevTrace tr, const int32_t *__restrict__ summ,
                                                   int32_t *__restrict__ snaps) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int E = tr.E, SN = 2 * E + 4, EB = (E + 31) / 32;
    const int64_t c = wid / EB;
    const int e = (int)(wid % EB) * 32 + lane;
    if (c >= tr.n_chains) return;
    const int64_t tpc = (tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
    const bool on = e < E;
    const int32_t *sm = summ + c * tpc * 2 * E;
    int32_t *sp = snaps + c * tpc * SN;
    int32_t carry_f = 0, carry_last = -1;
#pragma unroll 4
    for (int64_t t = 0; t < tpc; ++t) {
        const int32_t cnt = on ? __ldg(sm + t * 2 * E + e) : 0;
        const int32_t l = on ? __ldg(sm + t * 2 * E + E + e) : 0;
        if (on) {
            sp[t * SN + e] = carry_last;
            sp[t * SN + E + e] = carry_f;
        }
        if (e == 0) {
            const int64_t rt = t * MCB_TILE_EV * (int64_t)tr.K;
            sp[t * SN + 2 * E] = (int32_t)(t * MCB_TILE_EV);
            sp[t * SN + 2 * E + 1] = (int32_t)(rt & 0xFFFFFFFF);
            sp[t * SN + 2 * E + 2] = (int32_t)(rt >> 32);
        }
        carry_f += cnt;
        carry_last = l > 0 ? (int32_t)(t * MCB_TILE_EV) + l : carry_last;
    }
}

// fp64 tensor-core MLP layer (DMMA.8x8x4 via mma.sync m8n8k4 f64):
//   O[i][n] = act(sum_k A[i][k] * Wt[k][n] + b[n]),  i < 32 events of the tile
// A and O row-major in shared memory (leading dims = 4 mod 16 doubles, which
// makes the 8x4 A-fragment loads bank-conflict free; O may alias A: all warps
// finish reading A before the epilogue writes); Wt streamed from
// L1/L2.  Warp w owns n-tiles w, w+8, ... (NTW of them) x all four 8-row
// m-tiles: per k-step 4 A + NTW B fragments feed 4*NTW DMMAs.  Fragments:
// A(row=lane/4, k=lane%4), B(k=lane%4, col=lane/4), C(row=lane/4,
// col=2*(lane%4)+{0,1}).  float64 throughout (net.py:98-105 is float64).
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NTW, int KC = 0>
__device__ __forceinline__ void mma_layer(const double *A, int lda, int K_rt, const double *__restrict__ Wt,
                                          const double *__restrict__ bias, int N, double *O, int ldo, bool act,
                                          const double *tab) {
    const int K = KC ? KC : K_rt;   // compile-time depth: the k-loop unrolls fully, addresses fold
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int NT = N >> 3;
    const bool idle = warp >= NT;
    double acc[4][NTW][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int j = 0; j < NTW; ++j) acc[mt][j][0] = acc[mt][j][1] = 0.0;
    bool have[NTW];
    int col[NTW];
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
        have[j] = warp + 8 * j < NT;
        col[j] = (warp + 8 * j) * 8;
    }
    if (!idle) {
    const double *arow = A + g * lda + q;
    const double *wcol = Wt + (int64_t)q * N + g;
    // fragments of k-step k0 + 4 are in flight while k-step k0 multiplies
    double a[4], b[NTW];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) a[mt] = arow[mt * 8 * lda];
#pragma unroll
    for (int j = 0; j < NTW; ++j) b[j] = have[j] ? __ldg(wcol + col[j]) : 0.0;
#pragma unroll (KC ? 16 : 8)
    for (int k0 = 0; k0 < K; k0 += 4) {
        double an[4], bn[NTW];
        const int kn = k0 + 4 < K ? k0 + 4 : k0;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) an[mt] = arow[mt * 8 * lda + kn];
#pragma unroll
        for (int j = 0; j < NTW; ++j) bn[j] = have[j] ? __ldg(wcol + (int64_t)kn * N + col[j]) : 0.0;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int j = 0; j < NTW; ++j) dmma884(acc[mt][j][0], acc[mt][j][1], a[mt], b[j]);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a[mt] = an[mt];
#pragma unroll
        for (int j = 0; j < NTW; ++j) b[j] = bn[j];
    }
    }
    // every warp has consumed A before anyone overwrites it (O may alias A)
    __syncthreads();
    if (idle) return;
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
        if (!have[j]) continue;
        const int c0 = col[j] + 2 * q;
        const double b0 = __ldg(bias + c0), b1 = __ldg(bias + c0 + 1);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const double z0 = __dadd_rn(acc[mt][j][0], b0), z1 = __dadd_rn(acc[mt][j][1], b1);
            double2 v;
            v.x = act ? __dmul_rn(z0, sigmoid_ref(z0, tab)) : z0;
            v.y = act ? __dmul_rn(z1, sigmoid_ref(z1, tab)) : z1;
            *(double2 *)(O + (mt * 8 + g) * ldo + c0) = v;
        }
    }
}

// Narrow layer (N <= 16: the score layer for E <= 16): one 8x8 output tile
// per warp (up to 8 tiles = 4 m-tiles x N/8), two accumulators over
// alternating k-steps so consecutive DMMAs are independent.
template <int KC = 0>
__device__ __forceinline__ void mma_layer_narrow(const double *A, int lda, int K_rt, const double *__restrict__ Wt,
                                                 const double *__restrict__ bias, int N, double *O, int ldo,
                                                 bool act, const double *tab) {
    const int K = KC ? KC : K_rt;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int NT = N >> 3;
    const bool idle = warp >= 4 * NT;
    const int mt = idle ? 0 : warp / NT, nt = idle ? 0 : warp % NT;
    const double *arow = A + (mt * 8 + g) * lda + q;
    const double *wcol = Wt + (int64_t)q * N + nt * 8 + g;
    double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
    if (!idle) {
#pragma unroll (KC ? 32 : 8)
        for (int k0 = 0; k0 < K; k0 += 8) {
            const double a0 = arow[k0], b0 = __ldg(wcol + (int64_t)k0 * N);
            const bool two = k0 + 4 < K;
            const double a1 = two ? arow[k0 + 4] : 0.0, b1 = two ? __ldg(wcol + (int64_t)(k0 + 4) * N) : 0.0;
            dmma884(c0, c1, a0, b0);
            dmma884(d0, d1, a1, b1);
        }
    }
    // every warp has consumed A before anyone overwrites it (O may alias A:
    // the in-place hidden layer of a net with hidden <= 16)
    __syncthreads();
    if (idle) return;
    const int cc = nt * 8 + 2 * q;
    const double z0 = __dadd_rn(__dadd_rn(c0, d0), __ldg(bias + cc));
    const double z1 = __dadd_rn(__dadd_rn(c1, d1), __ldg(bias + cc + 1));
    double2 v;
    v.x = act ? __dmul_rn(z0, sigmoid_ref(z0, tab)) : z0;
    v.y = act ? __dmul_rn(z1, sigmoid_ref(z1, tab)) : z1;
    *(double2 *)(O + (mt * 8 + g) * ldo + cc) = v;
}

__device__ __forceinline__ void mma_layer_any(const double *A, int lda, int K, const double *Wt, const double *bias,
                                              int N, double *O, int ldo, bool act, const double *tab) {
    const int NT = N >> 3;
    if (NT <= 2) mma_layer_narrow(A, lda, K, Wt, bias, N, O, ldo, act, tab);
    else if (NT <= 8) mma_layer<1>(A, lda, K, Wt, bias, N, O, ldo, act, tab);
    else if (NT <= 16) mma_layer<2>(A, lda, K, Wt, bias, N, O, ldo, act, tab);
    else mma_layer<4>(A, lda, K, Wt, bias, N, O, ldo, act, tab);
}

// the same with the layer shape known at compile time (specialised scorers)
template <int N, int KC>
__device__ __forceinline__ void mma_layer_fixed(const double *A, int lda, const double *Wt, const double *bias,
                                                double *O, int ldo, bool act, const double *tab) {
    constexpr int NT = N >> 3;
    if constexpr (NT <= 2) mma_layer_narrow<KC>(A, lda, KC, Wt, bias, N, O, ldo, act, tab);
    else if constexpr (NT <= 8) mma_layer<1, KC>(A, lda, KC, Wt, bias, N, O, ldo, act, tab);
    else if constexpr (NT <= 16) mma_layer<2, KC>(A, lda, KC, Wt, bias, N, O, ldo, act, tab);
    else mma_layer<4, KC>(A, lda, KC, Wt, bias, N, O, ldo, act, tab);
}

__host__ __device__ __forceinline__ int mlp_ld(int cols) { return (cols + 15) / 16 * 16 + 4; }

// One block (256 threads) per (chain, tile of 64 events): warp 0 rebuilds
// the features of each event from the tile snapshot (features.py:34-52:
// [1/r || f / max_f]), the block runs the float64 MLP (EvictionNet.forward,
// net.py:88-105) in the transposed layout above, and ranks every expert's
// score within its event: rank = 1 + #{selectable j : s_j < s_e} for
// selectable e (s > -inf), 0 otherwise (NaN / -inf are never evicted,
// mlpolicy.py:15-26).  argmax score with lowest-id ties == argmax rank with
// lowest-id ties.
// Feature vectors [1/r || f / max_f] (features.py:44-52, float64) of the
// events [ev0, ev0 + nev) of chain c (one 32-event tile of a decode-only
// single-sequence trace) from the tile's tracker snapshot: thread i sets bit
// i of occ[e] for each expert its event routes to (features.py:34-39), so
// recency and counts at event i are the snapshot plus in-tile prefix bits.
// Rows go to out[i * ld + ...]; all_rows also zero-fills rows i >= nev.
// Shared scratch: occ[E] (u64), pmax[32].  Every thread of the block calls it.
__device__ __forceinline__ void tile_features_uniform(const DevTrace &tr, const int32_t *__restrict__ snaps,
                                                      int64_t tile, int64_t c, int64_t ev0, int nev, int E,
                                                      unsigned long long *occ, int32_t *pmax, double *out, int ld,
                                                      bool all_rows) {
    const int tid = threadIdx.x;
    const int32_t *sp = snaps + tile * (2 * E + 4);
    const int32_t u0 = sp[2 * E];
    for (int e = tid; e < E; e += blockDim.x) occ[e] = 0ull;
    __syncthreads();
    const uint8_t *ids = tr.acc + (c * tr.T + ev0) * tr.K;
    if (tid < nev)
        for (int k = 0; k < tr.K; ++k) atomicOr(&occ[__ldg(ids + tid * tr.K + k)], 1ull << tid);
    __syncthreads();
    if (tid < MCB_TILE_EV) {
        int32_t m = 0;
        if (tid < nev) {
            const unsigned long long upto = tid == 63 ? ~0ull : ((2ull << tid) - 1ull);
            for (int k = 0; k < tr.K; ++k) {
                const int x = __ldg(ids + tid * tr.K + k);
                m = max(m, sp[E + x] + __popcll(occ[x] & upto));
            }
        }
        pmax[tid] = m;
    }
    __syncthreads();
    if (tid < 32) {   // inclusive prefix max over the tile's events, then max with the snapshot max_f
        int32_t a = 2 * tid < MCB_TILE_EV ? pmax[2 * tid] : 0;
        int32_t b = max(a, 2 * tid + 1 < MCB_TILE_EV ? pmax[2 * tid + 1] : 0);
        int32_t m0 = 0;
        for (int e = 0; e < E; ++e) m0 = max(m0, sp[E + e]);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(FULL_MASK, b, o);
            if (tid >= o) { a = max(a, t); b = max(b, t); }
        }
        if (2 * tid < MCB_TILE_EV) pmax[2 * tid] = max(a, m0);
        if (2 * tid + 1 < MCB_TILE_EV) pmax[2 * tid + 1] = max(b, m0);
    }
    __syncthreads();
    for (int q = tid; q < MCB_TILE_EV * E; q += blockDim.x) {
        const int i = q % MCB_TILE_EV, e = q / MCB_TILE_EV;
        double rv = 0.0, fv = 0.0;
        if (i < nev) {
            const unsigned long long seen = occ[e] & (i == 63 ? ~0ull : ((2ull << i) - 1ull));
            const int32_t f = sp[E + e] + __popcll(seen);
            const int32_t lastu = seen ? u0 + (63 - __clzll(seen)) + 1 : sp[e];
            const int32_t u = u0 + i + 1;
            rv = lastu < 0 ? 0.0 : 1.0 / (double)(u - lastu + 1);
            const int32_t mf = pmax[i];
            fv = mf > 0 ? (double)f / (double)mf : 0.0;
        }
        if (i < nev || all_rows) {
            out[i * ld + e] = rv;
            out[i * ld + E + e] = fv;
        }
    }
}

// ---------------------------------------------------------------------------
// Feature rows of the events [ev0, ev0 + nev) of chain c (general traces:
// prefill, several sequences) from the tile's tracker snapshot, by one warp
// walking the tile's events in order (features.py:34-52: reset at a new
// sequence, update on decode events or on every event with include_prefill).
// Rows go to bufA[i * ldA + ...]; all_rows also zero-fills rows i >= nev.
__device__ __forceinline__ void tile_features_general(const DevTrace &tr, const int32_t *__restrict__ snaps,
                                                      int64_t tile, int64_t c, int64_t e0, int64_t ev0, int nev,
                                                      int E, int include_prefill, double *bufA, int ldA, int lane,
                                                      bool all_rows) {
    const int32_t *sp = snaps + tile * (2 * E + 4);
    int32_t last[4], f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e = lane + 32 * j;
        last[j] = e < E ? sp[e] : -1;
        f[j] = e < E ? sp[E + e] : 0;
    }
    int32_t u = sp[2 * E];
    int64_t rt = (int64_t)(uint32_t)sp[2 * E + 1] | ((int64_t)sp[2 * E + 2] << 32);
    int32_t maxf = __reduce_max_sync(FULL_MASK, max(max(f[0], f[1]), max(f[2], f[3])));
    const uint8_t *routed = tr.routed_ptr() + tr.rt_begin(c);
    for (int i = 0; i < MCB_TILE_EV; ++i) {
        if (i < nev) {
            const uint32_t info = tr.info(c, e0 + ev0 + i);
            const uint32_t nrt = mcb_ev_nrt(info);
            if (mcb_ev_newseq(info)) {
#pragma unroll
                for (int j = 0; j < 4; ++j) { last[j] = -1; f[j] = 0; }
                u = 0;
                maxf = 0;
            }
            if (mcb_ev_decode(info) || include_prefill) {
                ++u;
                for (uint32_t r = 0; r < nrt; ++r) {
                    const int x = __ldg(routed + rt + r);
                    if ((x & 31) == lane) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            { const bool hit_j = (x >> 5) == j; last[j] = hit_j ? u : last[j]; f[j] += hit_j ? 1 : 0; }
                    }
                }
                maxf = __reduce_max_sync(FULL_MASK, max(max(f[0], f[1]), max(f[2], f[3])));
            }
            rt += nrt;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int e = lane + 32 * j;
            if (e < E) {
                double rv = 0.0, fv = 0.0;
                if (i < nev) {
                    rv = last[j] < 0 ? 0.0 : 1.0 / (double)(u - last[j] + 1);
                    fv = maxf > 0 ? (double)f[j] / (double)maxf : 0.0;
                }
                if (i < nev || all_rows) {
                    bufA[i * ldA + e] = rv;
                    bufA[i * ldA + E + e] = fv;
                }
            }
        }
    }
}

// Training data (dataset.py:35-96, decode-only single-sequence traces):
// features of every decode step (the K3 feature rows) and capped next-use
// distance targets; the Belady residency masks come from the replay kernels
// (ReplayParams::res_masks).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_train_features(DevTrace tr, const int32_t *__restrict__ snaps,
                                                        double *__restrict__ features) {
    __shared__ unsigned long long occ[MCB_MAX_EXPERTS];
    __shared__ int32_t pmax[MCB_TILE_EV];
    const int64_t tile = blockIdx.x;
    const int64_t tpc = (tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
    if (tile >= tr.n_chains * tpc) return;
    const int64_t c = tile / tpc, ev0 = (tile % tpc) * MCB_TILE_EV;
    const int nev = (int)min((int64_t)MCB_TILE_EV, tr.T - ev0);
    const int E = tr.E;
    tile_features_uniform(tr, snaps, tile, c, ev0, nev, E, occ, pmax, features + (c * tr.T + ev0) * 2 * E, 2 * E,
                          false);
}

// targets[c][t][e] = min(d, cap) / cap with d the events until e is next
// routed strictly after t (StepNextUse.distance, replay.py:92-109; never
// again -> 1.0).  One warp per chain walks its events backwards, lanes over
// experts.
__global__ void __launch_bounds__(128) k_train_targets(DevTrace tr, int cap, double *__restrict__ targets) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (c >= tr.n_chains) return;
    const int E = tr.E, K = tr.K;
    int64_t next[4] = {-1, -1, -1, -1};
    const double dcap = (double)cap;
    const uint8_t *ids = tr.acc + c * tr.T * K;
    for (int64_t t = tr.T - 1; t >= 0; --t) {
        double *row = targets + (c * tr.T + t) * E;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int e = lane + 32 * j;
            if (e < E) {
                const int64_t d = next[j] < 0 ? (int64_t)cap : min(next[j] - t, (int64_t)cap);
                row[e] = __ddiv_rn((double)d, dcap);
            }
        }
        for (int k = 0; k < K; ++k) {
            const int x = __ldg(ids + t * K + k);
            if ((x & 31) == lane)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if ((x >> 5) == j) next[j] = t;
        }
    }
}

// General traces (prefill, several sequences): one warp per scorer tile
// writes the feature rows of the tile's events (every event; the caller keeps
// the decode rows, dataset.py:61-70).
__global__ void __launch_bounds__(32) k_train_features_general(DevTrace tr, const int32_t *__restrict__ snaps,
                                                               const int64_t *__restrict__ tile_off,
                                                               int include_prefill, double *__restrict__ features) {
    const int64_t tile = blockIdx.x;
    if (tile >= tile_off[tr.n_chains]) return;
    int64_t lo = 0, hi = tr.n_chains;   // largest c with tile_off[c] <= tile
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (tile_off[mid] <= tile) lo = mid; else hi = mid;
    }
    const int64_t c = lo, e0 = tr.ev_begin(c);
    const int64_t ev0 = (tile - tile_off[c]) * MCB_TILE_EV;
    const int nev = (int)min((int64_t)MCB_TILE_EV, tr.ev_end(c) - e0 - ev0);
    tile_features_general(tr, snaps, tile, c, e0, ev0, nev, tr.E, include_prefill,
                          features + (e0 + ev0) * 2 * tr.E, 2 * tr.E, threadIdx.x & 31, false);
}

// Targets of general traces: StepNextUse (replay.py:92-109) counts event
// ticks to the next event whose ROUTED list (not its accesses) holds e.
__global__ void __launch_bounds__(128) k_train_targets_general(DevTrace tr, int cap, double *__restrict__ targets) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (c >= tr.n_chains) return;
    const int E = tr.E;
    int64_t next[4] = {-1, -1, -1, -1};
    const double dcap = (double)cap;
    const uint8_t *routed = tr.routed_ptr();
    const int64_t e0 = tr.ev_begin(c);
    int64_t rt = tr.rt_begin(c + 1);
    for (int64_t t = tr.ev_end(c) - e0 - 1; t >= 0; --t) {
        double *row = targets + (e0 + t) * E;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int e = lane + 32 * j;
            if (e < E) {
                const int64_t d = next[j] < 0 ? (int64_t)cap : min(next[j] - t, (int64_t)cap);
                row[e] = __ddiv_rn((double)d, dcap);
            }
        }
        const uint32_t nrt = mcb_ev_nrt(tr.info(c, e0 + t));
        rt -= nrt;
        for (uint32_t k = 0; k < nrt; ++k) {
            const int x = __ldg(routed + rt + k);
            if ((x & 31) == lane)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if ((x >> 5) == j) next[j] = t;
        }
    }
}

int launch_train_features(const DevTrace &tr, const int32_t *snaps, const int64_t *tile_off, int64_t max_tiles,
                          int include_prefill, double *features, cudaStream_t s) {
    if (max_tiles <= 0) return 0;
    if (tr.uniform) k_train_features<<<(unsigned)max_tiles, 128, 0, s>>>(tr, snaps, features);
    else k_train_features_general<<<(unsigned)max_tiles, 32, 0, s>>>(tr, snaps, tile_off, include_prefill, features);
    return 1;
}

int launch_train_targets(const DevTrace &tr, int distance_cap, double *targets, cudaStream_t s) {
    if (tr.n_chains == 0) return 0;
    if (tr.uniform) k_train_targets<<<(unsigned)((tr.n_chains + 3) / 4), 128, 0, s>>>(tr, distance_cap, targets);
    else k_train_targets_general<<<(unsigned)((tr.n_chains + 3) / 4), 128, 0, s>>>(tr, distance_cap, targets);
    return 1;
}

// Order-preserving map of float64 to uint64 (-0.0 canonicalised to +0.0, so
// equal doubles map to equal keys) and its inverse.
__device__ __forceinline__ unsigned long long ordered_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x + 0.0);
    return b ^ ((unsigned long long)((long long)b >> 63) | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k ^ 0x8000000000000000ull) : ~k));
}

// max_e |s_e| over the finite scores of one event row (warp-wide): the scale
// of the float64 near-tie test, which is normwise so that two small scores
// produced by cancellation of large terms are flagged too.
__device__ __forceinline__ double row_scale(const double *srow, int E, int lane) {
    double m = 0.0;
    for (int e = lane; e < E; e += 32) {
        const double x = fabs(srow[e]);
        if (x < INFINITY) m = fmax(m, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL_MASK, m, o));
    return m;
}

// Ranks of one event's E scores by a warp-wide bitonic sort of the scores'
// order-preserving integer keys (P elements per lane, N = 32 P >= E; padding
// sorts last as +inf; equal scores need no tie-break because equal values get
// equal ranks): rank = 1 + #{selectable j : s_j < s_e} = 1 + (first sorted
// position of s_e's value) - #non-selectable, 0 for NaN / -inf (never
// evicted, mlpolicy.py:15-26).  A near-tie (two distinct scores within 1e-12 * max|s|
// relative) is always an adjacent sorted pair, which sets *flag.
template <int P>
__device__ __forceinline__ void rank_event_sorted(const double *srow, int E, uint8_t *rrow, int32_t *flag, int lane) {
    constexpr int N = 32 * P;
    const double scale = row_scale(srow, E, lane);
    const unsigned long long KNEG = ordered_key(-INFINITY), KPOS = ordered_key(INFINITY);
    unsigned long long v[P];
    int id[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int n = lane * P + p;
        id[p] = n;
        if (n < E) {
            const double x = srow[n];
            v[p] = x > -INFINITY ? ordered_key(x) : KNEG;   // NaN -> -inf: never selectable
        } else {
            v[p] = KPOS;
        }
    }
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= P) {   // partner in lane ^ (j / P)
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const unsigned long long ov = __shfl_xor_sync(FULL_MASK, v[p], j / P);
                    const int oid = __shfl_xor_sync(FULL_MASK, id[p], j / P);
                    const int n = lane * P + p;
                    const bool up = (n & k) == 0, lower = (n & j) == 0;
                    // keep the smaller key in the lower slot of an ascending pair
                    const bool take = lower == up ? ov < v[p] : ov > v[p];
                    if (take) { v[p] = ov; id[p] = oid; }
                }
            } else {        // partner in the same lane: p ^ j
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    if (p & j) continue;
                    const int q = p | j, n = lane * P + p;
                    const bool up = (n & k) == 0;
                    if (up ? v[q] < v[p] : v[q] > v[p]) {
                        const unsigned long long tv = v[p]; v[p] = v[q]; v[q] = tv;
                        const int ti = id[p]; id[p] = id[q]; id[q] = ti;
                    }
                }
            }
        }
    }
    // first sorted position of each value (inclusive max-scan of run starts)
    const unsigned long long prev_last = __shfl_up_sync(FULL_MASK, v[P - 1], 1);
    int start[P];
    int nsel_local = 0, loc = -1;
    bool near = false;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int n = lane * P + p;
        const unsigned long long pk = p > 0 ? v[p - 1] : prev_last;
        const bool first = n == 0 || v[p] != pk;
        loc = max(loc, first ? n : -1);
        start[p] = loc;
        nsel_local += (v[p] == KNEG) ? 1 : 0;
        if (n > 0 && v[p] != pk && pk != KNEG && v[p] != KPOS) {
            const double a = key_value(v[p]), b = key_value(pk);
            if (fabs(a - b) <= 1e-12 * scale) near = true;
        }
    }
    int carry = loc;   // warp inclusive max-scan of the lanes' last run start
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL_MASK, carry, o);
        if (lane >= o) carry = max(carry, t);
    }
    const int before = __shfl_up_sync(FULL_MASK, carry, 1);
    const int nsel = __reduce_add_sync(FULL_MASK, nsel_local);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int st = (lane > 0 && start[p] < 0) ? before : max(start[p], lane > 0 ? before : -1);
        if (id[p] < E) rrow[id[p]] = v[p] != KNEG ? (uint8_t)(st - nsel + 1) : (uint8_t)0;
    }
    if (__any_sync(FULL_MASK, near) && lane == 0) *flag = 1;
}

// Faster variant (E <= 128): the sort moves one word per element -- the
// order-preserving key with its low 7 bits replaced by the expert id -- so
// there is no separate id to shuffle and no tie-break.  Two different
// scores that agree in all but the low 7 key bits (or an exact tie) would
// compare by id; such an event (adjacent equal truncated keys after the
// sort, rare) is re-ranked exactly by rank_event_sorted.
template <int P>
__device__ __forceinline__ void rank_event_packed(const double *srow, int E, uint8_t *rrow, int32_t *flag, int lane) {
    constexpr int N = 32 * P;
    const double scale = row_scale(srow, E, lane);
    const unsigned long long KNEG = ordered_key(-INFINITY) & ~0x7Full, KPOS = ~0ull;
    unsigned long long v[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int n = lane * P + p;
        if (n < E) {
            const double x = srow[n];
            v[p] = (x > -INFINITY ? (ordered_key(x) & ~0x7Full) : KNEG) | (unsigned long long)n;
        } else {
            v[p] = KPOS;
        }
    }
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= P) {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const unsigned long long ov = __shfl_xor_sync(FULL_MASK, v[p], j / P);
                    const int n = lane * P + p;
                    const bool up = (n & k) == 0, lower = (n & j) == 0;
                    v[p] = (lower == up) ? min(v[p], ov) : max(v[p], ov);
                }
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    if (p & j) continue;
                    const int q = p | j, n = lane * P + p;
                    const bool up = (n & k) == 0;
                    const unsigned long long lo = min(v[p], v[q]), hi = max(v[p], v[q]);
                    v[p] = up ? lo : hi;
                    v[q] = up ? hi : lo;
                }
            }
        }
    }
    // adjacent equal truncated keys: the order between them is unknown
    const unsigned long long prev_last = __shfl_up_sync(FULL_MASK, v[P - 1], 1);
    bool collide = false;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int n = lane * P + p;
        const unsigned long long pk = p > 0 ? v[p - 1] : prev_last;
        if (n > 0 && v[p] != KPOS && (v[p] >> 7) == (pk >> 7) && (v[p] >> 7) != (KNEG >> 7)) collide = true;
    }
    if (__any_sync(FULL_MASK, collide)) {
        rank_event_sorted<P>(srow, E, rrow, flag, lane);
        return;
    }
    // all selectable keys are distinct: rank = sorted position - #non-selectable + 1
    int nsel_local = 0;
    bool near = false;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int n = lane * P + p;
        const unsigned long long pk = p > 0 ? v[p - 1] : prev_last;
        nsel_local += ((v[p] >> 7) == (KNEG >> 7) && v[p] != KPOS) ? 1 : 0;
        if (n > 0 && v[p] != KPOS && (pk >> 7) != (KNEG >> 7)) {
            const double a = srow[(int)(v[p] & 0x7Full)], b = srow[(int)(pk & 0x7Full)];
            if (fabs(a - b) <= 1e-12 * scale) near = true;
        }
    }
    const int nsel = __reduce_add_sync(FULL_MASK, nsel_local);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int n = lane * P + p;
        if (v[p] == KPOS) continue;
        const int id = (int)(v[p] & 0x7Full);
        rrow[id] = (v[p] >> 7) != (KNEG >> 7) ? (uint8_t)(n - nsel + 1) : (uint8_t)0;
    }
    if (__any_sync(FULL_MASK, near) && lane == 0) *flag = 1;
}

// Integer ranks of the fp64 scores of rows [0, nev) of bufA (row stride ldA)
// into s_rank[row][E], near-tie flags into s_flag[row] (rank = 1 + #{selectable
// j : s_j < s_e}, 0 for NaN / -inf; near tie = two distinct scores within
// 1e-12 * max_e |s_e|, normwise).  Every thread of the block calls it; ends with a barrier.
__device__ __forceinline__ void rank_tile_rows(const double *bufA, int ldA, int E, int nev, uint8_t *s_rank,
                                               int32_t *s_flag) {
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < MCB_TILE_EV; i += blockDim.x) s_flag[i] = 0;
    __syncthreads();
    if (E <= 16) {
        // few experts: each (event, expert) thread counts the smaller scores
        for (int q = tid; q < MCB_TILE_EV * E; q += blockDim.x) {
            const int i = q % MCB_TILE_EV, e = q / MCB_TILE_EV;
            if (i >= nev) continue;
            const double s = bufA[i * ldA + e];
            uint32_t r = 0;
            bool near = false;
            if (s > -INFINITY) {
                // rank = 1 + #{selectable j : s_j < s}; the near-tie test only needs the
                // nearest smaller score (every adjacent pair of the sorted order is
                // tested by its larger member)
                r = 1;
                double below = -INFINITY, scale = 0.0;
#pragma unroll 8
                for (int j = 0; j < E; ++j) {
                    const double sj = bufA[i * ldA + j];
                    if (fabs(sj) < INFINITY) scale = fmax(scale, fabs(sj));
                    if (sj > -INFINITY && sj < s) {
                        ++r;
                        below = fmax(below, sj);
                    }
                }
                near = below > -INFINITY && fabs(s - below) <= 1e-12 * scale;
            }
            s_rank[i * E + e] = (uint8_t)r;
            if (near) s_flag[i] = 1;
        }
    } else {
        // many experts: one warp sorts each event's scores (bitonic, in
        // registers) -- O(E log^2 E) instead of O(E^2) per event
        const int warp = tid >> 5;
        for (int i = warp; i < nev; i += (int)(blockDim.x >> 5)) {
            if (E <= 32) rank_event_packed<1>(bufA + i * ldA, E, s_rank + i * E, s_flag + i, lane);
            else if (E <= 64) rank_event_packed<2>(bufA + i * ldA, E, s_rank + i * E, s_flag + i, lane);
            else rank_event_packed<4>(bufA + i * ldA, E, s_rank + i * E, s_flag + i, lane);
        }
    }
    __syncthreads();
}

template <int TE, int TH>   // (num_experts, hidden) specialisation, 0 = runtime
__global__ void __launch_bounds__(256, TE ? 4 : 1) k_score_tile(DevTrace tr, const double *__restrict__ wt_all, int H_rt,
                                                     int num_nets, int include_prefill,
                                                     const int64_t *__restrict__ tile_off,
                                                     const int32_t *__restrict__ snaps, int64_t tile_lo,
                                                     int64_t tile_hi,
                                                     uint8_t *__restrict__ ranks, double *__restrict__ scores,
                                                     unsigned long long *uncertain) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int E = TE ? TE : tr.E, D = 2 * E, H = TH ? TH : H_rt;
    const int Hp = mlp_hp(H), Kp1 = mlp_kp1(E), Ep = mlp_ep(E);
    const int ldA = mlp_ld(Kp1 > Ep ? Kp1 : Ep), ldB = mlp_ld(Hp);
    double *bufA = (double *)smem_raw;                    // [TILE][ldA]: features, then scores
    double *bufB = bufA + ldA * MCB_TILE_EV;              // [TILE][ldB]: h1, then h2 (in place)
    uint8_t *s_rank = (uint8_t *)(bufB + ldB * MCB_TILE_EV);  // [TILE][E]
    int32_t *s_flag = (int32_t *)(s_rank + MCB_TILE_EV * MCB_MAX_EXPERTS);  // [TILE]

    __shared__ double s_exp2[64];
    if (threadIdx.x < 64) s_exp2[threadIdx.x] = g_exp2_64[threadIdx.x];   // visible after the first barrier
    // persistent: each CTA walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...
    for (int64_t tile_it = tile_lo + blockIdx.x; tile_it < tile_hi; tile_it += gridDim.x) {
    int64_t tile = tile_it;
    int64_t c, tile_in_chain;
    if (tr.uniform) {
        // chain-major: the CTAs in flight (a window of consecutive tiles) work
        // on the same chain, i.e. the same layer net, so its weights stay hot
        // in L1 / L2 instead of every SM streaming several nets
        const int64_t tpc = (tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
        c = tile / tpc;
        tile_in_chain = tile % tpc;
    } else {
        if (tile >= tile_off[tr.n_chains]) break;   // n_tiles is an upper bound in general mode
        int64_t lo = 0, hi = tr.n_chains;          // largest c with tile_off[c] <= tile
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) / 2;
            if (tile_off[mid] <= tile) lo = mid; else hi = mid;
        }
        c = lo;
        tile_in_chain = tile - tile_off[c];
    }
    const int64_t e0 = tr.ev_begin(c);
    const int64_t ev0 = tile_in_chain * MCB_TILE_EV;
    const int nev = (int)min((int64_t)MCB_TILE_EV, tr.ev_end(c) - e0 - ev0);
    const int tid = threadIdx.x, lane = tid & 31;

    if (tr.uniform) {
        // decode-only single sequence: every event updates, no resets, so the
        // tracker state at event i is the snapshot plus in-tile prefix counts
        // (features.py:34-39): thread i sets bit i of occ[e] for its routed e.
        tile_features_uniform(tr, snaps, tile, c, ev0, nev, E, (unsigned long long *)s_rank, s_flag, bufA, ldA,
                              true);
    } else if (tid < 32) {
        tile_features_general(tr, snaps, tile, c, e0, ev0, nev, E, include_prefill, bufA, ldA, lane, true);
    }
    for (int q = tid; q < MCB_TILE_EV * (Kp1 - D); q += blockDim.x)   // zero feature padding
        bufA[(q / (Kp1 - D)) * ldA + D + q % (Kp1 - D)] = 0.0;
    __syncthreads();
    const int64_t layer = c % tr.L;
    const double *wt = wt_all + (num_nets == 1 ? 0 : layer) * (int64_t)prepared_net_doubles(E, H);
    const double *Wt1 = wt, *b1 = Wt1 + (int64_t)Kp1 * Hp, *Wt2 = b1 + Hp, *b2 = Wt2 + (int64_t)Hp * Hp,
                 *Wt3 = b2 + Hp, *b3 = Wt3 + (int64_t)Hp * Ep;
    if constexpr (TE > 0 && TH > 0) {
        constexpr int cHp = (TH + 7) / 8 * 8, cKp1 = (2 * TE + 3) / 4 * 4, cEp = (TE + 7) / 8 * 8;
        mma_layer_fixed<cHp, cKp1>(bufA, ldA, Wt1, b1, bufB, ldB, true, s_exp2);    // h1 -> B
        __syncthreads();
        mma_layer_fixed<cHp, cHp>(bufB, ldB, Wt2, b2, bufB, ldB, true, s_exp2);     // h2 -> B (in place)
        __syncthreads();
        mma_layer_fixed<cEp, cHp>(bufB, ldB, Wt3, b3, bufA, ldA, false, s_exp2);    // scores -> A
        __syncthreads();
    } else {
        mma_layer_any(bufA, ldA, Kp1, Wt1, b1, Hp, bufB, ldB, true, s_exp2);    // h1 -> B
        __syncthreads();
        mma_layer_any(bufB, ldB, Hp, Wt2, b2, Hp, bufB, ldB, true, s_exp2);     // h2 -> B (in place)
        __syncthreads();
        mma_layer_any(bufB, ldB, Hp, Wt3, b3, Ep, bufA, ldA, false, s_exp2);    // scores -> A
        __syncthreads();
    }
    rank_tile_rows(bufA, ldA, E, nev, s_rank, s_flag);
    if (scores)
        for (int q = tid; q < nev * E; q += blockDim.x) scores[(e0 + ev0) * E + q] = bufA[(q / E) * ldA + q % E];
    __syncthreads();
    uint8_t *dst = ranks + (e0 + ev0) * E;
    for (int q = tid; q < nev * E; q += blockDim.x) dst[q] = s_rank[q];
    if (tid == 0 && uncertain) {
        unsigned long long cnt = 0;
        for (int i = 0; i < nev; ++i) cnt += s_flag[i];
        if (cnt) atomicAdd(uncertain, cnt);
    }
    __syncthreads();   // shared buffers are reused by the next tile
    }
}

// float64 re-score of the events the tensor-core scorer could not certify
// (mcb_score_tc.cu): flag_list holds, per net (bucket), the chain-major event
// indices of a uniform trace.  Each CTA takes 32 listed events of one net at a
// time, rebuilds their float64 features from the K3 snapshot of their 32-event
// tile plus the tile's earlier events (features.py:34-52), runs the same
// float64 MLP and ranking as k_score_tile and overwrites their rank rows.
template <int TE, int TH>
__global__ void __launch_bounds__(256, 3) k_rescore(DevTrace tr, const double *__restrict__ wt_all, int H_rt,
                                                   int num_nets, const int32_t *__restrict__ snaps,
                                                   const int32_t *__restrict__ flag_cnt,
                                                   const int32_t *__restrict__ flag_list, int64_t bucket_cap,
                                                   uint8_t *__restrict__ ranks, unsigned long long *uncertain) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int E = TE ? TE : tr.E, D = 2 * E, H = TH ? TH : H_rt;
    const int Hp = mlp_hp(H), Kp1 = mlp_kp1(E), Ep = mlp_ep(E);
    const int ldA = mlp_ld(Kp1 > Ep ? Kp1 : Ep), ldB = mlp_ld(Hp);
    double *bufA = (double *)smem_raw;
    double *bufB = bufA + ldA * MCB_TILE_EV;
    uint8_t *s_rank = (uint8_t *)(bufB + ldB * MCB_TILE_EV);
    int32_t *s_flag = (int32_t *)(s_rank + MCB_TILE_EV * MCB_MAX_EXPERTS);
    __shared__ double s_exp2[64];
    __shared__ int64_t s_pref[MCB_MAX_EXPERTS + 1];
    __shared__ int32_t s_ev[MCB_TILE_EV];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 64) s_exp2[tid] = g_exp2_64[tid];
    if (tid == 0) {
        int64_t a = 0;
        s_pref[0] = 0;
        for (int bk = 0; bk < num_nets; ++bk) {
            a += (flag_cnt[bk] + MCB_TILE_EV - 1) / MCB_TILE_EV;
            s_pref[bk + 1] = a;
        }
    }
    __syncthreads();
    const int64_t total = s_pref[num_nets];
    const int64_t tpc32 = (tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
    const int SN = 2 * E + 4;
    for (int64_t vt = blockIdx.x; vt < total; vt += gridDim.x) {
        int bk = 0;
        while (s_pref[bk + 1] <= vt) ++bk;
        const int64_t i0 = (vt - s_pref[bk]) * MCB_TILE_EV;
        const int nev = (int)min((int64_t)MCB_TILE_EV, (int64_t)flag_cnt[bk] - i0);
        if (tid < MCB_TILE_EV) s_ev[tid] = tid < nev ? flag_list[bk * bucket_cap + i0 + tid] : -1;
        __syncthreads();
        for (int r = warp; r < MCB_TILE_EV; r += (int)(blockDim.x >> 5)) {
            const int32_t ev = s_ev[r];
            int32_t last[4], f[4];
            int32_t u = 0, maxf = 0;
            if (ev >= 0) {
                const int64_t c = ev / tr.T, i = ev % tr.T, s32 = i / MCB_TILE_EV;
                const int32_t *sp = snaps + (c * tpc32 + s32) * SN;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int e = lane + 32 * j;
                    last[j] = e < E ? sp[e] : -1;
                    f[j] = e < E ? sp[E + e] : 0;
                }
                // the tile's events up to and including this one (features.py:34-39):
                // lane l ORs bit l into the occurrence word of each expert event
                // j0 + l routes (shared-memory atomics into this warp's 128 words of
                // the rank staging, free until the ranking), then lane l reads the
                // occurrence masks of experts l + 32 w
                const int64_t j0 = s32 * MCB_TILE_EV;
                const int nprefix = (int)(i - j0) + 1;
                uint32_t *so = (uint32_t *)s_rank + warp * MCB_MAX_EXPERTS;
#pragma unroll
                for (int w = 0; w < 4; ++w) so[lane + 32 * w] = 0u;
                __syncwarp();
                if (lane < nprefix) {
                    const uint8_t *ids = tr.acc + (c * tr.T + j0 + lane) * tr.K;
                    for (int k = 0; k < tr.K; ++k) atomicOr(so + __ldg(ids + k), 1u << lane);
                }
                __syncwarp();
                uint32_t occ[4];   // lane l: occurrence masks of experts l + 32 w
#pragma unroll
                for (int w = 0; w < 4; ++w) occ[w] = so[lane + 32 * w];
                __syncwarp();   // read before the warp's next event clears the words
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (occ[j]) {
                        last[j] = (int32_t)j0 + (31 - __clz(occ[j])) + 1;
                        f[j] += __popc(occ[j]);
                    }
                u = (int32_t)i + 1;
                maxf = __reduce_max_sync(FULL_MASK, max(max(f[0], f[1]), max(f[2], f[3])));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int e = lane + 32 * j;
                if (e < E) {
                    double rv = 0.0, fv = 0.0;
                    if (ev >= 0) {
                        rv = last[j] < 0 ? 0.0 : 1.0 / (double)(u - last[j] + 1);
                        fv = maxf > 0 ? (double)f[j] / (double)maxf : 0.0;
                    }
                    bufA[r * ldA + e] = rv;
                    bufA[r * ldA + E + e] = fv;
                }
            }
        }
        for (int q = tid; q < MCB_TILE_EV * (Kp1 - D); q += blockDim.x)   // zero feature padding
            bufA[(q / (Kp1 - D)) * ldA + D + q % (Kp1 - D)] = 0.0;
        __syncthreads();
        const double *wt = wt_all + (num_nets == 1 ? 0 : bk) * (int64_t)prepared_net_doubles(E, H);
        const double *Wt1 = wt, *b1 = Wt1 + (int64_t)Kp1 * Hp, *Wt2 = b1 + Hp, *b2 = Wt2 + (int64_t)Hp * Hp,
                     *Wt3 = b2 + Hp, *b3 = Wt3 + (int64_t)Hp * Ep;
        if constexpr (TE > 0 && TH > 0) {
            constexpr int cHp = (TH + 7) / 8 * 8, cKp1 = (2 * TE + 3) / 4 * 4, cEp = (TE + 7) / 8 * 8;
            mma_layer_fixed<cHp, cKp1>(bufA, ldA, Wt1, b1, bufB, ldB, true, s_exp2);
            __syncthreads();
            mma_layer_fixed<cHp, cHp>(bufB, ldB, Wt2, b2, bufB, ldB, true, s_exp2);
            __syncthreads();
            mma_layer_fixed<cEp, cHp>(bufB, ldB, Wt3, b3, bufA, ldA, false, s_exp2);
            __syncthreads();
        } else {
            mma_layer_any(bufA, ldA, Kp1, Wt1, b1, Hp, bufB, ldB, true, s_exp2);
            __syncthreads();
            mma_layer_any(bufB, ldB, Hp, Wt2, b2, Hp, bufB, ldB, true, s_exp2);
            __syncthreads();
            mma_layer_any(bufB, ldB, Hp, Wt3, b3, Ep, bufA, ldA, false, s_exp2);
            __syncthreads();
        }
        rank_tile_rows(bufA, ldA, E, nev, s_rank, s_flag);
        for (int q = tid; q < nev * E; q += blockDim.x) ranks[(int64_t)s_ev[q / E] * E + q % E] = s_rank[q];
        if (tid == 0 && uncertain) {
            unsigned long long cnt = 0;
            for (int i = 0; i < nev; ++i) cnt += s_flag[i];
            if (cnt) atomicAdd(uncertain, cnt);
        }
        __syncthreads();
    }
}

typedef void (*rescore_fn)(DevTrace, const double *, int, int, const int32_t *, const int32_t *, const int32_t *,
                           int64_t, uint8_t *, unsigned long long *);
static rescore_fn rescore_kernel(int E, int H) {
    if (H == 128) {
        if (E == 8) return k_rescore<8, 128>;
        if (E == 16) return k_rescore<16, 128>;
        if (E == 64) return k_rescore<64, 128>;
        if (E == 128) return k_rescore<128, 128>;
    }
    return k_rescore<0, 0>;
}

static size_t score_smem(int E, int H) {
    const int Hp = mlp_hp(H), Kp1 = mlp_kp1(E), Ep = mlp_ep(E);
    const int ldA = mlp_ld(Kp1 > Ep ? Kp1 : Ep), ldB = mlp_ld(Hp);
    return (size_t)MCB_TILE_EV * (ldA + ldB) * sizeof(double) + MCB_TILE_EV * MCB_MAX_EXPERTS +
           MCB_TILE_EV * sizeof(int32_t);
}

// Specialisations of the scorer for the shapes of the BASELINE configs
// (Mixtral E=8, Qwen3 E=128, OLMoE / DSV2-Lite E=64, E=16; hidden 128 as
// EvictionNet's default, net.py:64); anything else runs the runtime-shape
// instantiation <0, 0>.
typedef void (*score_fn)(DevTrace, const double *, int, int, int, const int64_t *, const int32_t *, int64_t,
                         int64_t, uint8_t *, double *, unsigned long long *);
static score_fn score_kernel(int E, int H) {
    if (H == 128) {
        if (E == 8) return k_score_tile<8, 128>;
        if (E == 16) return k_score_tile<16, 128>;
        if (E == 64) return k_score_tile<64, 128>;
        if (E == 128) return k_score_tile<128, 128>;
    }
    return k_score_tile<0, 0>;
}

// Function attributes are set once per shape (all instantiations at once).
void prepare_launch_attributes(const DevTrace &tr, int H) {
    (void)tr;
    (void)H;
}

// K3 part 1: tile snapshots of the feature tracker (all chains)
int launch_score_prep(const DevTrace &tr, int include_prefill, int32_t *snaps, int64_t *tile_off, int64_t max_tiles,
                      cudaStream_t s) {
    if (tr.n_chains == 0) return 0;
    if (tr.uniform) {
        // snaps scratch holds [summaries | snapshots]
        int32_t *summ = snaps + max_tiles * (2 * tr.E + 4);
        k_tile_summary<<<(unsigned)((max_tiles + 3) / 4), 128, 0, s>>>(tr, summ);
        // many chains: lane = expert, coalesced walk over the tiles; few long
        // chains (not enough warps to fill the GPU): lane = tile, warp scans
        const int64_t tpc = (tr.T + MCB_TILE_EV - 1) / MCB_TILE_EV;
        const int64_t walkers = tr.n_chains * ((tr.E + 31) / 32);
        if (walkers >= 4096 || tpc <= 64)
            k_snap_scan<<<(unsigned)((walkers + 3) / 4), 128, 0, s>>>(tr, summ, snaps);
        else
            k_snap_scan_tiles<<<(unsigned)((tr.n_chains * tr.E + 3) / 4), 128, 0, s>>>(tr, summ, snaps);
    } else {
        k_tile_offsets<<<1, 1024, 0, s>>>(tr, tile_off);
        k_feat_snap<<<(unsigned)((tr.n_chains + 3) / 4), 128, 0, s>>>(tr, include_prefill, tile_off, snaps);
    }
    return 2;
}

// K3 part 2: score tiles [tile_lo, tile_hi) (persistent CTAs).  Uniform
// traces number tiles chain-major, so a chain range maps to a tile range.
// K3 grid (k3_ctas): < 0 (default) = one CTA per 32-event tile; 0 =
// persistent, as many CTAs as fit (4 per SM for the specialised shapes);
// k > 0 = persistent with at most k CTAs per SM.  Measured on C2
// (tools/k3_sweep.sh): one CTA per tile is faster alone (4.12 vs 4.51 ms:
// better tail balance) and lets the concurrent non-ML replay's blocks in as
// CTAs retire (persistent CTAs hold the whole register file, so the replay
// waited for K3): 6.09 vs 6.55 ms per step.
int launch_score_tiles(const DevTrace &tr, const double *wt, int H, int num_nets, int include_prefill,
                       uint8_t *ranks, double *scores, const int32_t *snaps, const int64_t *tile_off,
                       int64_t tile_lo, int64_t tile_hi, unsigned long long *uncertain, int k3_ctas,
                       cudaStream_t s) {
    if (tile_hi <= tile_lo) return 0;
    const size_t smem = score_smem(tr.E, H);
    const score_fn fn = score_kernel(tr.E, H);
    int dev = 0, n_sm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)fn, 256, smem);
    if (k3_ctas > 0 && k3_ctas < per_sm) per_sm = k3_ctas;
    const int64_t grid = k3_ctas < 0 ? tile_hi - tile_lo
                                       : std::min<int64_t>(tile_hi - tile_lo, (int64_t)n_sm * (per_sm > 0 ? per_sm : 1));
    fn<<<(unsigned)grid, 256, smem, s>>>(tr, wt, H, num_nets, include_prefill, tile_off, snaps, tile_lo, tile_hi,
                                         ranks, scores, uncertain);
    return 1;
}

int launch_score(const DevTrace &tr, const double *wt, int H, int num_nets, int include_prefill, uint8_t *ranks,
                 double *scores, int32_t *snaps, int64_t *tile_off, int64_t max_tiles,
                 unsigned long long *uncertain, int k3_ctas, cudaStream_t s) {
    if (tr.n_chains == 0) return 0;
    int launched = launch_score_prep(tr, include_prefill, snaps, tile_off, max_tiles, s);
    launched += launch_score_tiles(tr, wt, H, num_nets, include_prefill, ranks, scores, snaps, tile_off, 0,
                                   max_tiles, uncertain, k3_ctas, s);
    return launched;
}

// float64 re-score of the tensor-core scorer's flagged events (persistent
// grid; the per-net counts are read on the device).
int launch_rescore(const DevTrace &tr, const double *wt, int H, int num_nets, const int32_t *snaps,
                   const int32_t *flag_cnt, const int32_t *flag_list, int64_t bucket_cap, uint8_t *ranks,
                   unsigned long long *uncertain, cudaStream_t s) {
    if (tr.n_chains == 0) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = score_smem(tr.E, H);
    const rescore_fn fn = rescore_kernel(tr.E, H);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fn<<<(unsigned)(8 * sms), 256, smem, s>>>(tr, wt, H, num_nets, snaps, flag_cnt, flag_list, bucket_cap, ranks,
                                             uncertain);
    return 1;
}

// Force-load every kernel of the library at context creation (CUDA 12 lazy
// module loading would otherwise load them inside the first timed call) and
// set their shared-memory limits once.
int preload_kernels() {
    cudaFuncAttributes a;
    const void *fns[] = {
        (const void *)k_next_use<true>, (const void *)k_next_use<false>, (const void *)k_next_use_blocks,
        (const void *)k_next_use_thread, (const void *)k_fold, (const void *)k_train_features, (const void *)k_train_targets, (const void *)k_prepare_nets, (const void *)k_tile_offsets,
        (const void *)k_feat_snap, (const void *)k_tile_summary, (const void *)k_snap_scan,
        (const void *)k_snap_scan_tiles,
        (const void *)k_score_tile<0, 0>, (const void *)k_score_tile<8, 128>, (const void *)k_score_tile<16, 128>,
        (const void *)k_score_tile<64, 128>, (const void *)k_score_tile<128, 128>,
        (const void *)k_replay<32, 1, true>, (const void *)k_replay<32, 1, false>,
        (const void *)k_replay<32, 2, true>, (const void *)k_replay<32, 2, false>,
        (const void *)k_replay<32, 4, true>, (const void *)k_replay<32, 4, false>,
        (const void *)k_replay<8, 4, true>, (const void *)k_replay<8, 4, false>,
        (const void *)k_replay<16, 2, true>, (const void *)k_replay<16, 2, false>,
        (const void *)k_replay<8, 8, true>, (const void *)k_replay<8, 8, false>,
        (const void *)k_replay<16, 4, true>, (const void *)k_replay<16, 4, false>,
        (const void *)k_replay<16, 8, true>, (const void *)k_replay<16, 8, false>,
        (const void *)k_replay_solo<8, true>, (const void *)k_replay_solo<8, false>,
        (const void *)k_replay_solo<16, true>, (const void *)k_replay_solo<16, false>,
    };
    if (cudaFuncSetAttribute(k_next_use_thread, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             MCB_MAX_EXPERTS * 128 * (int)sizeof(uint32_t)) != cudaSuccess)
        return -1;
    for (const void *f : fns)
        if (cudaFuncGetAttributes(&a, f) != cudaSuccess) return -1;
    cudaFuncSetAttribute(k_replay_solo<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_replay_solo<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_replay_solo<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_replay_solo<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const void *scorers[] = {(const void *)k_score_tile<0, 0>, (const void *)k_score_tile<8, 128>,
                             (const void *)k_score_tile<16, 128>, (const void *)k_score_tile<64, 128>,
                             (const void *)k_score_tile<128, 128>};
    for (const void *f : scorers) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return 0;
}
