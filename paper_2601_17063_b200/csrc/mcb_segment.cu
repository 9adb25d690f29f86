// Segmented speculative replay for latency-bound workloads (few, long chains;
// uniform decode-only traces, num_experts <= 16).
//
// One (trace, layer) chain is a strict sequential dependence:
// the cache state after access i depends on every earlier access.  A single
// Mixtral-shaped trace has only 32 chains x policies x capacities = 768
// instances of 131,072 accesses each -- far too few threads for 148 SMs.
// But the policy keys depend on the trace alone (F1), and the cache state is
// small (resident mask + refetch ring), so a chain can be cut into S segments
// replayed in parallel and stitched exactly:
//
//   snapshot  per (chain, segment): each expert's last access position and
//             access count before the segment (two-pass scan) -> the exact
//             policy keys at the segment start
//   spec      one thread per (instance, segment): replay the segment from a
//             GUESSED cache state (the min(C, #seen) experts with the best
//             keys, empty refetch ring; exact for segment 0) and record the
//             counters, the end state, the poly hash of its outcome codes and
//             the per-event miss counts
//   finish    one thread per instance walks its segments in order carrying the
//             TRUE state: it replays segment k from the true state (A) and
//             from the guess (B) in lockstep until the two states coincide --
//             from there on the speculative run is the true run, so its
//             counters / hash / end state are spliced in with the prefix
//             corrected (counters by difference, hash via h(AB) = h(A) P^|B| +
//             h(B)); if they never coincide, A's results are used and A's end
//             state carries on.  It also folds the float64 latency over every
//             event in order (engine.py:258-262), reading the per-event miss
//             counts, so SimReport floats stay bit-identical.
//
// Results are identical to the whole-chain kernel by construction; the
// states typically coincide within a few events (LRU: the guess is the exact
// resident set, only the refetch ring differs for W+1 decode steps).
#include <cuda_runtime.h>
#include <stdint.h>

#include "mcb_kernels.cuh"
#include "mcb_solo.cuh"

#define SEG_MAX_E 16

bool seg_eligible(const ReplayParams &p) {
    return p.seg.n_seg > 1 && p.tr.uniform && p.tr.E <= SEG_MAX_E && p.outcomes == nullptr && p.window >= 0 &&
           p.window <= SOLO_WMAX && p.tr.total_acc < (1ll << 27) && p.tr.T * p.tr.K < (1ll << 27);
}

int seg_events_per_segment(int64_t T, int64_t n_inst_launch, int64_t override_se) {
    // enough (instance, segment) threads to fill every SM several times over,
    // segments long enough that the fix-up walk stays a small fraction
    const int64_t target_threads = 148ll * 768;
    int64_t se;
    if (override_se > 0) {
        se = override_se;
    } else {
        const int64_t n_seg = n_inst_launch > 0 ? target_threads / n_inst_launch : 1;
        if (n_seg <= 2) return 0;
        se = (T + n_seg - 1) / n_seg;
        if (se < 64) se = 64;
    }
    se = (se + 15) / 16 * 16;
    if (se >= T) return 0;
    return (int)se;
}

size_t seg_snap_bytes(int64_t n_chains, int n_seg) { return (size_t)n_chains * n_seg * SEG_MAX_E * sizeof(int2); }
size_t seg_out_bytes(int64_t n_inst, int n_seg) { return (size_t)n_inst * n_seg * sizeof(SegOut); }
size_t seg_codes_bytes(int64_t n_inst, int64_t Tpad) { return (size_t)n_inst * Tpad + 64; }

// ---------------------------------------------------------------- snapshot --
__global__ void __launch_bounds__(128) k_seg_summary(const __grid_constant__ ReplayParams P) {
    __shared__ int32_t s_cnt[128][SEG_MAX_E + 1];
    __shared__ int32_t s_last[128][SEG_MAX_E + 1];
    const DevTrace &tr = P.tr;
    const int n_seg = P.seg.n_seg, SE = P.seg.SE;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tr.n_chains * n_seg) return;
    const int64_t chain = t / n_seg;
    const int seg = (int)(t % n_seg);
    int32_t *cnt = s_cnt[threadIdx.x], *last = s_last[threadIdx.x];
    for (int e = 0; e < SEG_MAX_E; ++e) { cnt[e] = 0; last[e] = -1; }
    const int K = tr.K;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t p0 = (int64_t)seg * SE * K;
    const int64_t p1 = min((int64_t)(seg + 1) * SE, tr.T) * K;
    IdReader ids;
    ids.init(tr.acc, a0 + p0, a0 + p1);
    for (int64_t p = p0; p < p1; ++p) {
        const uint32_t x = ids.get(a0 + p);
        cnt[x] += 1;
        last[x] = (int32_t)p;
    }
    int2 *o = P.seg.summ + t * SEG_MAX_E;
    for (int e = 0; e < SEG_MAX_E; ++e) o[e] = make_int2(last[e], cnt[e]);
}

__global__ void k_seg_scan(const __grid_constant__ ReplayParams P) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.tr.n_chains * SEG_MAX_E) return;
    const int64_t chain = t / SEG_MAX_E;
    const int e = (int)(t % SEG_MAX_E);
    const int n_seg = P.seg.n_seg;
    int32_t last = -1, cnt = 0;
    for (int seg = 0; seg < n_seg; ++seg) {
        const int64_t i = (chain * n_seg + seg) * SEG_MAX_E + e;
        const int2 s = P.seg.summ[i];
        P.seg.snap[i] = make_int2(last, cnt);
        if (s.x >= 0) last = s.x;
        cnt += s.y;
    }
}

int launch_seg_snapshot(const ReplayParams &p, cudaStream_t s) {
    const int64_t n = p.tr.n_chains * p.seg.n_seg;
    k_seg_summary<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(p);
    const int64_t m = p.tr.n_chains * SEG_MAX_E;
    k_seg_scan<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(p);
    return 2;
}

// ------------------------------------------------------------ shared parts --
// Exact policy keys at the start of segment `seg` of `chain` (all experts),
// the seen mask, and the guessed resident set: the min(C, #seen) seen experts
// with the LARGEST packed keys (the ones the policy would evict last).  For
// LRU this is the true resident set (a stack algorithm over recency).
template <int EM, int POL>
__device__ __forceinline__ void seg_start(const ReplayParams &P, int64_t chain, int seg, uint32_t C, int ml_variant,
                                          uint32_t (&pk)[EM], uint32_t &seen, uint32_t &guess) {
    constexpr int SH = Solo<EM>::SH;
    constexpr uint32_t KMAX = Solo<EM>::KMAX;
    const DevTrace &tr = P.tr;
    const int E = tr.E;
    const int2 *sn = P.seg.snap + (chain * P.seg.n_seg + seg) * SEG_MAX_E;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t ev0 = (int64_t)seg * P.seg.SE;
    uint32_t rrow[EM];
    if (POL == POL_ML) {
        if (ev0 > 0) load_rank_row<EM>(rrow, P.rank[ml_variant] + (tr.ev_begin(chain) + ev0 - 1) * E, E);
        else
#pragma unroll
            for (int s = 0; s < EM; ++s) rrow[s] = 0u;
    }
    seen = 0u;
#pragma unroll
    for (int s = 0; s < EM; ++s) {
        const int2 v = s < E ? sn[s] : make_int2(-1, 0);
        seen |= (v.x >= 0 ? 1u : 0u) << s;
        uint32_t k = (uint32_t)s;
        if (POL == POL_LRU) k = v.x >= 0 ? (((uint32_t)v.x << SH) | (uint32_t)s) : (uint32_t)s;
        if (POL == POL_LFU) k = ((uint32_t)v.y << SH) | (uint32_t)s;
        if (POL == POL_BELADY) {
            const uint32_t np = v.x >= 0 ? __ldg(P.next_pos + a0 + v.x) : MCB_NEXT_INF;
            k = ((np == MCB_NEXT_INF ? 0u : KMAX - np) << SH) | (uint32_t)s;
        }
        if (POL == POL_ML) k = ((256u - rrow[s]) << SH) | (uint32_t)s;
        pk[s] = k;
    }
    const uint32_t n_res = min(C, (uint32_t)__popc(seen));
    guess = 0u;
#pragma unroll
    for (int s = 0; s < EM; ++s) {
        uint32_t better = 0;
#pragma unroll
        for (int j = 0; j < EM; ++j) better += (((seen >> j) & 1u) && pk[j] > pk[s]) ? 1u : 0u;
        guess |= (((seen >> s) & 1u) && better < n_res) ? (1u << s) : 0u;
    }
}

// ------------------------------------------------------------------- spec --
template <int EM, int POL>
__device__ __forceinline__ void seg_spec(const ReplayParams &P, int64_t chain, int seg, int pol_i, int cap_i,
                                         int ml_variant) {
    constexpr int WMAX = SOLO_WMAX;
    const DevTrace &tr = P.tr;
    const int E = tr.E, K = tr.K, W = P.window;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    const int64_t ev0 = (int64_t)seg * P.seg.SE;
    const int64_t ev1 = min(ev0 + P.seg.SE, tr.T);
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;

    uint32_t pk[EM], seen, guess;
    seg_start<EM, POL>(P, chain, seg, C, ml_variant, pk, seen, guess);
    SState<WMAX> S;
    sstate_clear(S);
    S.res = guess;
    uint32_t valid = (1u << E) - 1u, comp = 0;
    SCount n = {0u, 0u, 0u};
    bool stuck = false;
    int32_t stuck_ev = -1;
    uint64_t h = 0;
    const bool track = P.hashes != nullptr;

    IdReader ids;
    ids.init(tr.acc, a0 + ev0 * K, a0 + ev1 * K);
    NextReader nx;
    if (POL == POL_BELADY) nx.init(P.next_pos, a0 + ev0 * K, a0 + ev1 * K);
    uint32_t rrow[EM];
    if (POL == POL_ML) load_rank_row<EM>(rrow, rank + (e0 + ev0) * E, E);
    uint32_t *codes = (uint32_t *)(P.seg.codes + inst * P.seg.Tpad);
    uint32_t word = 0;

    for (int64_t ev = ev0; ev < ev1; ++ev) {
        if (POL == POL_ML) {
            solo_ml_keys<EM>(pk, valid, rrow);
            if (ev + 1 < ev1) load_rank_row<EM>(rrow, rank + (e0 + ev + 1) * E, E);
        }
        uint32_t pin = 0, sm = 0;
        const int64_t A0 = a0 + ev * K;
        for (int j = 0; j < K; ++j) {
            const int64_t A = A0 + j;
            const uint32_t x = ids.get(A);
            const uint32_t bit = 1u << x;
            const uint32_t np = (POL == POL_BELADY) ? nx.get(A) : 0u;
            solo_key_update<EM, POL>(pk, x, bit, (uint32_t)(ev * K + j), np);
            uint32_t miss;
            const uint32_t code = sstep<EM, WMAX>(S, pk, bit, pin, valid, C, n, stuck, miss);
            sm += miss;
            comp += (miss && !(seen & bit)) ? 1u : 0u;
            seen |= bit;
            pin |= bit;
            if (track) h = poly16(h, code);
        }
        if (stuck && stuck_ev < 0) stuck_ev = (int32_t)ev;
        word |= sm << (8 * (uint32_t)(ev & 3));
        if ((ev & 3) == 3) { codes[ev >> 2] = word; word = 0; }
        sstate_next_decode<WMAX>(S, W);
    }
    if (ev1 & 3) codes[ev1 >> 2] = word;   // tail word (segment ends mid-word only at the chain end)

    SegOut &o = P.seg.out[inst * P.seg.n_seg + seg];
    o.misses = n.misses;
    o.nev = n.nev;
    o.refc = n.refc;
    o.comp = comp;
    o.res = S.res;
    o.stuck_ev = stuck_ev;
    o.hash = h;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) o.ring[s] = S.ring[s];
}

template <int EM>
__global__ void __launch_bounds__(128) k_seg_spec(const __grid_constant__ ReplayParams P) {
    const int pol_i = P.pol_map[blockIdx.y];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int n_seg = P.seg.n_seg;
    if (t >= P.tr.n_chains * n_seg * P.n_cap) return;
    const int cap_i = (int)(t % P.n_cap);
    const int64_t r = t / P.n_cap;
    const int seg = (int)(r % n_seg);
    const int64_t chain = r / n_seg;
    switch (P.pol[pol_i]) {
        case MCB_LRU: seg_spec<EM, POL_LRU>(P, chain, seg, pol_i, cap_i, 0); break;
        case MCB_LFU: seg_spec<EM, POL_LFU>(P, chain, seg, pol_i, cap_i, 0); break;
        case MCB_BELADY: seg_spec<EM, POL_BELADY>(P, chain, seg, pol_i, cap_i, 0); break;
        case MCB_ML: seg_spec<EM, POL_ML>(P, chain, seg, pol_i, cap_i, 0); break;
        default: seg_spec<EM, POL_ML>(P, chain, seg, pol_i, cap_i, 1); break;
    }
}

// ----------------------------------------------------------------- finish --
// float64 latency of events [ev, ev1) from the stored miss counts, in order
__device__ __forceinline__ double fold_codes(double dlat, const uint8_t *codes, int64_t ev, int64_t ev1,
                                             const double *lut) {
    while (ev < ev1 && (ev & 15)) dlat = __dadd_rn(dlat, lut[__ldg(codes + ev++)]);
    const uint4 *v = (const uint4 *)(codes + ev);
    const int64_t nv = (ev1 - ev) >> 4;
    uint4 cur = nv > 0 ? __ldg(v) : make_uint4(0, 0, 0, 0);
    for (int64_t i = 0; i < nv; ++i) {
        const uint4 nxt = i + 1 < nv ? __ldg(v + i + 1) : make_uint4(0, 0, 0, 0);
        const uint32_t w[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int b = 0; b < 4; ++b) dlat = __dadd_rn(dlat, lut[(w[q] >> (8 * b)) & 0xFFu]);
        cur = nxt;
    }
    ev += nv << 4;
    while (ev < ev1) dlat = __dadd_rn(dlat, lut[__ldg(codes + ev++)]);
    return dlat;
}

template <int EM, int POL>
__device__ __forceinline__ void seg_finish(const ReplayParams &P, int64_t chain, int pol_i, int cap_i, int ml_variant,
                                           const double *lut) {
    constexpr int WMAX = SOLO_WMAX;
    const DevTrace &tr = P.tr;
    const int E = tr.E, K = tr.K, W = P.window;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int n_seg = P.seg.n_seg, SE = P.seg.SE;
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;
    const uint8_t *codes = P.seg.codes + inst * P.seg.Tpad;
    const SegOut *so = P.seg.out + inst * n_seg;
    const bool track = P.hashes != nullptr;

    // segment 0 starts from the true (empty) state: its speculative run is exact
    SState<WMAX> A;
    A.res = so[0].res;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) A.ring[s] = so[0].ring[s];
    uint32_t misses = so[0].misses, nev = so[0].nev, refc = so[0].refc, comp = so[0].comp;
    bool stuck = so[0].stuck_ev >= 0;
    uint64_t h = so[0].hash;
    double dlat = fold_codes(0.0, codes, 0, min((int64_t)SE, tr.T), lut);
    const uint64_t pow_full = track ? pow_mul((uint64_t)SE * K) : 0ull;

    for (int seg = 1; seg < n_seg; ++seg) {
        const int64_t ev0 = (int64_t)seg * SE;
        const int64_t ev1 = min(ev0 + SE, tr.T);
        {   // ring_or of the carried state
            uint32_t o = 0u;
#pragma unroll
            for (int s = 0; s <= WMAX; ++s) o |= (s <= W) ? A.ring[s] : 0u;
            A.ring_or = o;
        }
        uint32_t pk[EM], seen, guess;
        seg_start<EM, POL>(P, chain, seg, C, ml_variant, pk, seen, guess);
        SState<WMAX> B;
        sstate_clear(B);
        B.res = guess;
        SCount ca = {0u, 0u, 0u}, cb = {0u, 0u, 0u};
        uint64_t ha = 0, hb = 0;
        bool stuck_a = false, stuck_b = false;
        uint32_t valid = (1u << E) - 1u;
        int64_t ev = ev0;
        bool conv = sstate_equal<WMAX>(A, B, W);
        if (!conv) {
            IdReader ids;
            ids.init(tr.acc, a0 + ev0 * K, a0 + ev1 * K);
            NextReader nx;
            if (POL == POL_BELADY) nx.init(P.next_pos, a0 + ev0 * K, a0 + ev1 * K);
            while (!conv && ev < ev1) {
                if (POL == POL_ML) {
                    uint32_t rrow[EM];
                    load_rank_row<EM>(rrow, rank + (e0 + ev) * E, E);
                    solo_ml_keys<EM>(pk, valid, rrow);
                }
                uint32_t pin = 0, sma = 0;
                for (int j = 0; j < K; ++j) {
                    const int64_t Aa = a0 + ev * K + j;
                    const uint32_t x = ids.get(Aa);
                    const uint32_t bit = 1u << x;
                    const uint32_t np = (POL == POL_BELADY) ? nx.get(Aa) : 0u;
                    solo_key_update<EM, POL>(pk, x, bit, (uint32_t)(ev * K + j), np);
                    uint32_t ma, mb;
                    const uint32_t codea = sstep<EM, WMAX>(A, pk, bit, pin, valid, C, ca, stuck_a, ma);
                    const uint32_t codeb = sstep<EM, WMAX>(B, pk, bit, pin, valid, C, cb, stuck_b, mb);
                    sma += ma;
                    pin |= bit;
                    if (track) { ha = poly16(ha, codea); hb = poly16(hb, codeb); }
                }
                dlat = __dadd_rn(dlat, lut[sma]);
                sstate_next_decode<WMAX>(A, W);
                sstate_next_decode<WMAX>(B, W);
                ++ev;
                conv = sstate_equal<WMAX>(A, B, W);
            }
        }
        const SegOut &o = so[seg];
        uint64_t hseg;
        if (conv) {
            // from event ev on, the speculative run (which started from B's
            // state) is the true run: splice it in, correcting the prefix
            misses += ca.misses + o.misses - cb.misses;
            nev += ca.nev + o.nev - cb.nev;
            refc += ca.refc + o.refc - cb.refc;
            stuck = stuck || stuck_a || (o.stuck_ev >= 0 && o.stuck_ev >= ev);
            hseg = track ? o.hash + (ha - hb) * pow_mul((uint64_t)(ev1 - ev) * K) : 0ull;
            A.res = o.res;
#pragma unroll
            for (int s = 0; s <= WMAX; ++s) A.ring[s] = o.ring[s];
            dlat = fold_codes(dlat, codes, ev, ev1, lut);
        } else {
            misses += ca.misses;
            nev += ca.nev;
            refc += ca.refc;
            stuck = stuck || stuck_a;
            hseg = ha;
        }
        comp += o.comp;
        if (track) h = h * (ev1 - ev0 == SE ? pow_full : pow_mul((uint64_t)(ev1 - ev0) * K)) + hseg;
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

template <int EM>
__global__ void __launch_bounds__(128) k_seg_finish(const __grid_constant__ ReplayParams P) {
    __shared__ double lut[SEG_MAX_E + 1];
    const int pol_i = P.pol_map[blockIdx.y];
    const int pol = P.pol[pol_i];
    const int K = P.tr.K;
    if (threadIdx.x <= (unsigned)K) {
        // step_latency_s (engine.py:58-62) per miss count, + ml_score_cost_s for ML decode steps
        const uint32_t m = threadIdx.x;
        const double lat = m > 0 ? __dmul_rn((double)(P.loads_serial ? m : 1u), P.t_load)
                                 : __dmul_rn((double)K, P.t_compute);
        lut[m] = __dadd_rn(lat, (pol == MCB_ML || pol == MCB_ML_NO_PREFILL) ? P.ml_cost : 0.0);
    }
    __syncthreads();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.tr.n_chains * P.n_cap) return;
    const int cap_i = (int)(t % P.n_cap);
    const int64_t chain = t / P.n_cap;
    switch (pol) {
        case MCB_LRU: seg_finish<EM, POL_LRU>(P, chain, pol_i, cap_i, 0, lut); break;
        case MCB_LFU: seg_finish<EM, POL_LFU>(P, chain, pol_i, cap_i, 0, lut); break;
        case MCB_BELADY: seg_finish<EM, POL_BELADY>(P, chain, pol_i, cap_i, 0, lut); break;
        case MCB_ML: seg_finish<EM, POL_ML>(P, chain, pol_i, cap_i, 0, lut); break;
        default: seg_finish<EM, POL_ML>(P, chain, pol_i, cap_i, 1, lut); break;
    }
}

template <int EM>
static void launch_seg_t(const ReplayParams &p, cudaStream_t s) {
    const int64_t n_spec = p.tr.n_chains * p.seg.n_seg * p.n_cap;
    k_seg_spec<EM><<<dim3((unsigned)((n_spec + 127) / 128), (unsigned)p.n_pol_launch), 128, 0, s>>>(p);
    const int64_t n_fin = p.tr.n_chains * p.n_cap;
    k_seg_finish<EM><<<dim3((unsigned)((n_fin + 127) / 128), (unsigned)p.n_pol_launch), 128, 0, s>>>(p);
}

int launch_replay_segmented(const ReplayParams &p, cudaStream_t s) {
    if (p.tr.n_chains * p.n_pol_launch * p.n_cap == 0) return 0;
    if (p.tr.E <= 8) launch_seg_t<8>(p, s);
    else launch_seg_t<16>(p, s);
    return 2;
}

int preload_segment_kernels() {
    cudaFuncAttributes a;
    const void *fns[] = {(const void *)k_seg_summary, (const void *)k_seg_scan, (const void *)k_seg_spec<8>,
                         (const void *)k_seg_spec<16>, (const void *)k_seg_finish<8>,
                         (const void *)k_seg_finish<16>};
    for (const void *f : fns)
        if (cudaFuncGetAttributes(&a, f) != cudaSuccess) return -1;
    return 0;
}
