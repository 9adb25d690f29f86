// K4-wide: one THREAD per cache instance for 16 < num_experts <= 128 (whole
// chains; LRU, LFU, Belady, ML, FIFO).  The warp-per-instance replay
// (k_replay) spends a warp's issue slot on every access; here one thread
// carries the instance:
//   * resident / pinned / seen / selectable sets and the refetch ring are
//     64-bit (E <= 64) or 128-bit (two words) masks in registers;
//   * the per-expert packed keys (key << 7 | id) live in
//     shared memory, column-major per thread (keys[s][thread]), so the
//     per-access key write is one conflict-free store whatever the expert;
//   * the victim is the minimum key over the candidate bits only (at most C
//     loads), and only on an evicting miss;
//   * LRU keeps no keys: a doubly linked recency list of the resident
//     experts (byte links in shared memory) gives the victim in O(1) -- the
//     tail is the minimum last-access position, and it is never pinned
//     unless every resident expert is (pinned experts were accessed in the
//     current event, after every other resident one);
//   * ML keeps the event's rank row as bytes (one row per thread, four
//     16-byte copies per event), turns resident \ pinned into a rank-space
//     mask once per event (rank_space: bit r - 1 per candidate of rank r,
//     plus rank -> expert bytes) and keeps it in step with every access, so
//     each evicting miss takes the highest-ranked candidate with one FLO
//     (rank 0 = NaN / -inf score, never selectable).  The per-miss rank scan
//     it replaces ran once per miss under SIMT divergence (70 % of the ML
//     launch's instructions on C4).
// Semantics are sstep()'s (mcb_solo.cuh) on wide masks: policies.py:95-214,
// mlpolicy.py:15-26, engine.py:229-257 (pinning), engine.py:266-297 (refetch).
// Used when there are enough instances to fill the GPU (many traces, e.g. C4).
#include <cuda_runtime.h>
#include <stdint.h>

#include "mcb_internal.h"
#include "mcb_kernels.cuh"
#include "mcb_mask.cuh"
#include "mcb_solo.cuh"

namespace wide {

using namespace mm;

constexpr int BS = 128;     // threads per block
constexpr int SH = 7;       // id bits of a packed key (E <= 128)
static_assert(SH == 7, "packed keys carry 7 id bits (E <= 128)");
constexpr uint32_t KMAX = (1u << (32 - SH)) - 1u;

constexpr uint32_t NIL = 0xFFu;   // end of the LRU list
constexpr int NLOW = 4;           // smallest keys kept per event (LFU / Belady / FIFO)
constexpr uint32_t NLOW_MAXC = 32;   // ... for capacities up to this (a larger resident set costs more to
                                     // select from per event than the few evicting misses it serves: C5)

template <int POL, bool UNIFORM, int WMAX, typename M>
__device__ __forceinline__ void wide_instance(const ReplayParams &P, int64_t chain, int pol_i, int cap_i,
                                              int ml_variant, uint32_t *sk) {
    const DevTrace &tr = P.tr;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int E = tr.E;
    const int W = P.window;
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    auto key = [&](int s) -> uint32_t & { return sk[s * BS]; };
    if (POL != POL_LRU && POL != POL_ML)
        for (int s = 0; s < E; ++s) key(s) = (uint32_t)s;
    // LRU: next / prev links [2][E][BS] bytes; ML: this thread's rank row
    uint8_t *const lb = (uint8_t *)(sk - threadIdx.x) + threadIdx.x;
    auto nxt = [&](uint32_t e) -> uint8_t & { return lb[e * BS]; };
    auto prv = [&](uint32_t e) -> uint8_t & { return lb[(E + e) * BS]; };
    uint32_t head = NIL, tail = NIL;
    uint8_t *const mrow0 = (uint8_t *)(sk - threadIdx.x) + threadIdx.x * mrow_stride(E);
    // ML: rank -> expert of the event's candidates, [thread][E] after the rank rows
    uint8_t *const mord = (uint8_t *)(sk - threadIdx.x) + BS * mrow_stride(E) + threadIdx.x * E;
    // ML with E % 16 == 0 (and E >= 32, so it fits the key area): two rank-row
    // buffers after the rank -> expert bytes, the next event's row copied
    // asynchronously while this one is used (its load latency is otherwise
    // exposed once per event when few instances share an SM)
    const bool ml_async = POL == POL_ML && (E & 15) == 0 && E >= 32;
    uint8_t *const mrow1 = (uint8_t *)(sk - threadIdx.x) + BS * (mrow_stride(E) + E) + threadIdx.x * mrow_stride(E);

    M res = zero<M>(), seen = zero<M>(), ring_or = zero<M>();
    M ring[WMAX + 1];
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) ring[s] = zero<M>();
    M valid = first_n<M>(E);
    uint32_t ph = 0, pm = 0, dh = 0, dm = 0, comp = 0, nev = 0, refc = 0;
    double dlat = 0.0, plat = 0.0;
    uint64_t h = 0;
    bool stuck = false;

    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const int64_t n_ev = tr.ev_end(chain) - e0;
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;
    uint16_t *outc = P.outcomes ? P.outcomes + ((int64_t)pol_i * P.n_cap + cap_i) * tr.total_acc : nullptr;
    const bool track = outc != nullptr || P.hashes != nullptr;

    const int64_t a_end = tr.acc_end(chain);
    IdReader ids;   // 16 ids per vector load, the next vector in flight
    ids.init(tr.acc, a0, a_end);
    NextReader nx;
    if (POL == POL_BELADY) nx.init(P.next_pos, a0, a_end);
    int64_t A = a0;
    uint32_t pos = 0;
    if (ml_async && n_ev > 0) rank_row_async(rank + e0 * E, mrow0, E);
    for (int64_t ev = 0; ev < n_ev; ++ev) {
        const uint32_t info = UNIFORM ? mcb_ev_pack((uint32_t)tr.K, (uint32_t)tr.K, true, ev == 0)
                                      : __ldg(tr.ev_info + e0 + ev);
        const uint32_t nacc = mcb_ev_nacc(info);
        const bool decode = UNIFORM ? true : mcb_ev_decode(info);
        if (POL == POL_LFU && !UNIFORM && mcb_ev_newseq(info))
            for (int s = 0; s < E; ++s) key(s) = (uint32_t)s;   // start_sequence (policies.py:184-185)
        if (P.res_masks) {   // resident set before the event (dataset.py:61-63)
            uint8_t *m = P.res_masks + (e0 + ev) * E;
            for (int e = 0; e < E; ++e) m[e] = (uint8_t)test(res, (uint32_t)e);
        }
        M cr = zero<M>();   // ML: resident \ pinned in rank space (rank_space), kept in step below
        uint8_t *const mrow = (ml_async && (ev & 1)) ? mrow1 : mrow0;
        if (POL == POL_ML) {   // this event's rank row (mlpolicy.py:59-62)
            if (ml_async) {
                rank_row_wait();
                if (ev + 1 < n_ev) rank_row_async(rank + (e0 + ev + 1) * E, (ev & 1) ? mrow0 : mrow1, E);
            } else {
                copy_rank_row(rank + (e0 + ev) * E, mrow, E);
            }
            cr = rank_space(res, mrow, mord);
        }
        // LFU / Belady / FIFO in a decode event: a candidate's key cannot change
        // within the event (only accessed experts' keys change, and an accessed
        // expert is pinned from then on), so the event's victims come in key
        // order from the NLOW smallest keys of the resident set at its start,
        // skipping experts pinned since -- one uniform pass per event instead of
        // a candidate scan per evicting miss (which SIMT divergence paid at
        // almost every access).  More victims than that, or a prefill event,
        // take the scan.
        constexpr bool KEYED = POL == POL_LFU || POL == POL_BELADY || POL == POL_FIFO;
        uint32_t low[NLOW], lp = NLOW;
        if (KEYED && decode && C <= NLOW_MAXC && (uint32_t)popc(res) + nacc > C) {
            lowest_keys<BS, NLOW>(res, sk, low);
            lp = 0;
        }
        M pin = zero<M>();
        uint32_t step_miss = 0;
        for (uint32_t j = 0; j < nacc; ++j, ++pos, ++A) {
            const uint32_t x = ids.get(A);
            const M bit = bit_of<M>(x);
            // trace-determined key of x (applied before the victim search; x is never a candidate)
            if (POL == POL_LRU && test(res, x) && x != head) {   // hit: move x to the front
                const uint32_t p = prv(x), n = nxt(x);
                nxt(p) = (uint8_t)n;
                if (x == tail) tail = p;
                else prv(n) = (uint8_t)p;
                nxt(x) = (uint8_t)head;
                prv(x) = (uint8_t)NIL;
                prv(head) = (uint8_t)x;
                head = x;
            }
            if (POL == POL_LFU) key(x) += 1u << SH;
            if (POL == POL_BELADY) {
                const uint32_t np = nx.get(A);
                key(x) = ((np == MCB_NEXT_INF ? 0u : KMAX - np) << SH) | x;
            }
            const bool hit = test(res, x);
            uint32_t code = MCB_OUT_HIT;
            if (!hit) {
                M vbit = zero<M>();
                code = MCB_OUT_MISS;
                if ((uint32_t)popc(res) >= C) {
                    if (POL == POL_LRU) {
                        if (tail == NIL || test(pin, tail)) {   // every resident expert is pinned
                            stuck = true;
                        } else {
                            const uint32_t v = tail;
                            tail = prv(v);
                            if (tail == NIL) head = NIL;
                            else nxt(tail) = (uint8_t)NIL;
                            vbit = bit_of<M>(v);
                            code = v;
                            ++nev;
                        }
                    } else if (POL == POL_ML) {
                        if (!any(cr)) {   // no candidate with a selectable score
                            stuck = true;
                        } else {
                            const uint32_t r = top_bit(cr);   // the highest-ranked candidate
                            const uint32_t v = mord[r];
                            cr = cr & ~bit_of<M>(r);
                            vbit = bit_of<M>(v);
                            code = v;
                            ++nev;
                        }
                    } else {
                        uint32_t best = ~0u;
                        while (KEYED && lp < NLOW) {
                            uint32_t k = low[0];
#pragma unroll
                            for (int q = 1; q < NLOW; ++q) k = lp == (uint32_t)q ? low[q] : k;
                            ++lp;
                            if (k == ~0u) {   // the start-of-event resident set is used up
                                lp = NLOW;
                            } else if (!test(pin, k & ((1u << SH) - 1u))) {
                                best = k;
                                break;
                            }
                        }
                        M cand = res & ~pin & valid;
                        if (best == ~0u && any(cand)) best = min_key<BS>(cand, sk);
                        if (best == ~0u) {
                            stuck = true;
                        } else {
                            const uint32_t v = best & ((1u << SH) - 1u);
                            vbit = bit_of<M>(v);
                            code = v;
                            ++nev;
                        }
                    }
                }
                if (POL == POL_LRU) {   // insert x at the front
                    nxt(x) = (uint8_t)head;
                    prv(x) = (uint8_t)NIL;
                    if (head == NIL) tail = x;
                    else prv(head) = (uint8_t)x;
                    head = x;
                }
                res = (res & ~vbit) | bit;
                refc += test(ring_or, x) ? 1u : 0u;   // refetch of an earlier victim within the window
                ring_or = (ring_or & ~bit) | vbit;
#pragma unroll
                for (int s = 0; s <= WMAX; ++s) ring[s] = ring[s] & ~bit;
                ring[0] = ring[0] | vbit;
                if (POL == POL_FIFO) key(x) = (pos << SH) | x;   // arrival (policies.py:159-161)
                ++step_miss;
                comp += test(seen, x) ? 0u : 1u;
                if (decode) ++dm; else ++pm;
            } else {
                if (decode) ++dh; else ++ph;
            }
            if (POL == POL_ML) {
                const uint32_t rx = mrow[x];
                if (decode) {
                    cr = cr & ~rank_bit<M>(rx);   // x is pinned for the rest of the event
                } else if (!hit && rx != 0u) {   // a prefill insertion is a candidate
                    cr = cr | bit_of<M>(rx - 1u);
                    mord[rx - 1u] = (uint8_t)x;
                }
            }
            seen = seen | bit;
            if (decode) pin = pin | bit;
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
#pragma unroll
            for (int s = WMAX; s >= 1; --s) ring[s] = ring[s - 1];
            ring[0] = zero<M>();
            M o = zero<M>();
#pragma unroll
            for (int s = 0; s <= WMAX; ++s)
                if (s <= W) o = o | ring[s];
            ring_or = o;
        } else {
            plat = __dadd_rn(plat, lat);
        }
    }
    int64_t *o = P.inst_out + inst * MCB_R_N;
    o[MCB_R_PREFILL_HITS] = ph;
    o[MCB_R_PREFILL_MISSES] = pm;
    o[MCB_R_DECODE_HITS] = dh;
    o[MCB_R_DECODE_MISSES] = dm;
    o[MCB_R_COMPULSORY] = comp;
    o[MCB_R_EVICTIONS] = nev;
    o[MCB_R_REFETCHED] = refc;
    o[MCB_R_STATUS] = stuck ? MCB_ERR_NO_EVICTABLE : MCB_OK;
    P.inst_lat[inst * 2 + 0] = dlat;
    P.inst_lat[inst * 2 + 1] = plat;
    if (P.hashes) P.hashes[inst] = h;
}

// All policies of the call in one launch (blockIdx.y = policy), so the
// instances of every policy share the waves; blockIdx.x * BS + threadIdx.x =
// (chain, capacity) instance.
template <bool UNIFORM, typename M, int WMAX>
__global__ void __launch_bounds__(BS, sizeof(M) == 8 ? 6 : 4) k_replay_wide(const __grid_constant__ ReplayParams P) {
    extern __shared__ uint32_t s_keys[];   // [E][BS] keys, LRU links or ML rank rows
    const int pol_i = P.pol_map[blockIdx.y];
    const int64_t t = (int64_t)blockIdx.x * BS + threadIdx.x;
    if (t >= (P.chain_hi - P.chain_lo) * P.n_cap) return;
    const int cap_i = (int)(t % P.n_cap);
    const int64_t chain = P.chain_lo + t / P.n_cap;
    uint32_t *sk = s_keys + threadIdx.x;
    switch (P.pol[pol_i]) {
        case MCB_LRU: wide_instance<POL_LRU, UNIFORM, WMAX, M>(P, chain, pol_i, cap_i, 0, sk); break;
        case MCB_LFU: wide_instance<POL_LFU, UNIFORM, WMAX, M>(P, chain, pol_i, cap_i, 0, sk); break;
        case MCB_BELADY: wide_instance<POL_BELADY, UNIFORM, WMAX, M>(P, chain, pol_i, cap_i, 0, sk); break;
        case MCB_ML: wide_instance<POL_ML, UNIFORM, WMAX, M>(P, chain, pol_i, cap_i, 0, sk); break;
        case MCB_FIFO: wide_instance<POL_FIFO, UNIFORM, WMAX, M>(P, chain, pol_i, cap_i, 0, sk); break;
        default: wide_instance<POL_ML, UNIFORM, WMAX, M>(P, chain, pol_i, cap_i, 1, sk); break;
    }
}

template <bool UNIFORM, typename M>
int set_wide_smem(size_t smem) {
    const void *fs[] = {(const void *)k_replay_wide<UNIFORM, M, 5>, (const void *)k_replay_wide<UNIFORM, M, SOLO_WMAX>};
    for (const void *f : fs) {
        cudaFuncAttributes a;
        if (cudaFuncGetAttributes(&a, f) != cudaSuccess) return -1;
        if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
    }
    return 0;
}

// the refetch ring sized for the call's window: 6 slots for the default
// window 5 (fewer registers, fewer mask updates per miss), else SOLO_WMAX + 1
template <bool UNIFORM, typename M>
void launch_wide_w(const ReplayParams &p, dim3 grid, size_t smem, cudaStream_t s) {
    if (p.window <= 5) k_replay_wide<UNIFORM, M, 5><<<grid, BS, smem, s>>>(p);
    else k_replay_wide<UNIFORM, M, SOLO_WMAX><<<grid, BS, smem, s>>>(p);
}

}  // namespace wide

// true when the launch was taken: 16 < E <= 128, only the policies above,
// chains short enough for 25-bit positions, window <= SOLO_WMAX
int launch_replay_wide(const ReplayParams &p, cudaStream_t s) {
    const int E = p.tr.E;
    if (E <= 16 || E > 128 || p.window < 0 || p.window > SOLO_WMAX) return 0;
    const int64_t chain_bound = p.tr.uniform ? p.tr.T * p.tr.K : p.tr.total_acc;
    if (chain_bound >= (1ll << (32 - wide::SH))) return 0;
    for (int i = 0; i < p.n_pol_launch; ++i) {
        const int pol = p.pol[p.pol_map[i]];
        if (pol == MCB_ARC || pol == MCB_LECAR) return 0;
    }
    const int64_t n = (p.chain_hi - p.chain_lo) * p.n_cap;
    const dim3 grid((unsigned)((n + wide::BS - 1) / wide::BS), (unsigned)p.n_pol_launch);
    const size_t smem = (size_t)E * wide::BS * sizeof(uint32_t);
    if (E <= 64) {
        if (p.tr.uniform) wide::launch_wide_w<true, uint64_t>(p, grid, smem, s);
        else wide::launch_wide_w<false, uint64_t>(p, grid, smem, s);
    } else {
        if (p.tr.uniform) wide::launch_wide_w<true, mm::M128>(p, grid, smem, s);
        else wide::launch_wide_w<false, mm::M128>(p, grid, smem, s);
    }
    return 1;
}

int preload_wide_kernels() {
    const size_t smem = 128 * wide::BS * 4;
    if (wide::set_wide_smem<true, uint64_t>(smem) || wide::set_wide_smem<false, uint64_t>(smem) ||
        wide::set_wide_smem<true, mm::M128>(smem) || wide::set_wide_smem<false, mm::M128>(smem))
        return -1;
    return 0;
}
