// Segmented speculative replay for latency-bound workloads (few, long chains;
// uniform decode-only traces, num_experts <= 16).
//
// One (trace, layer) chain is a strict sequential dependence:
// the cache state after access i depends on every earlier access.  A single
// Mixtral-shaped trace has only 32 chains x policies x capacities = 768
// instances of 131,072 accesses each -- far too few threads for 148 SMs.
// But the policy keys depend on the trace alone (F1) and the cache state is
// small (resident mask + refetch ring), so a chain is cut into segments that
// are replayed in parallel and stitched exactly:
//
//   snapshot  every MCB_SNAP_EV events of every chain: each expert's last
//             access position and access count so far (two-pass scan), i.e.
//             the exact policy keys at that point
//   spec      one thread per (instance, segment): start NW events before the
//             segment from a guessed cache state (the min(C, #seen) experts
//             the policy would evict last, empty refetch ring), replay the
//             warm-up without counting -- states started apart coalesce --
//             record the state at the segment start, then replay the segment
//             and record its counters, end state, poly hash of the outcome
//             codes, per-event miss counts and their histogram
//   spec 2    (not for LRU, whose guess is already the exact resident set)
//             every segment is replayed again from pass 1's END state of the
//             previous segment -- the true state whenever that segment's
//             speculation had coalesced -- so only segments behind a long
//             non-coalescing stretch still differ from the true run
//   finish    one warp per instance walks its segments in order carrying the
//             TRUE state A.  If A equals the segment's recorded start state,
//             the speculative run IS the true run and is spliced in whole.
//             Otherwise A and the recorded start state B are replayed in
//             lockstep until they coincide; from there on the speculative run
//             is the true run, so its results are spliced in with the prefix
//             corrected (counters by difference, hash via h(XY) = h(X) P^|Y| +
//             h(Y)); if they never coincide, A's own results are used and A
//             carries on.
//
// float64 latency (engine.py:258-262) is a sequential sum over events of
// values from a (K+1)-entry table.  Inside one binade [2^(e-1), 2^e) of the
// running sum, RN(S + v) = S + q(v) ulp with q(v) = v / ulp rounded to
// nearest -- independent of S unless v / ulp is a tie -- so a whole segment
// is folded from its miss-count histogram with integer arithmetic whenever it
// stays in one binade and hits no tie, and event by event otherwise.  Both
// paths give the reference's bits exactly.
//
// Results are identical to the whole-chain kernel by construction
// (tests/test_segment_gpu.py checks them against the oracle).
#include <cuda_runtime.h>
#include <stdint.h>

#include "mcb_kernels.cuh"
#include "mcb_solo.cuh"

#define SEG_MAX_E 16
#define SEG_DEFAULT_NW 256

bool seg_eligible(const ReplayParams &p) {
    return p.seg.n_seg > 1 && p.tr.uniform && p.tr.E <= MCB_MAX_EXPERTS && p.tr.K + 1 <= MCB_SEG_BINS &&
           p.outcomes == nullptr && p.window >= 0 && p.window <= SOLO_WMAX &&
           p.tr.T * p.tr.K < (1ll << 27) &&   // chain-local positions pack into 27 bits
           (p.tr.E <= SEG_MAX_E || p.tr.T * p.tr.K < (1ll << 25));   // 25 bits in the warp version's keys
}

int seg_events_per_segment(int64_t T, int64_t n_inst_launch, int64_t override_se, int E, bool paired) {
    // enough (instance, segment) workers to fill every SM several times over:
    // threads for the thread-per-instance replay (E <= 16), warps for the
    // warp-per-instance one.  Thread segments are at least 2 default warm-ups
    // long, 4 when the ML and non-ML replays run side by side after the
    // scorer (paired; measured on C2: 512 / 768 / 1024 / 1536 events = 5.31 /
    // 5.26 / 5.21 / 5.52 ms per step, tools/seg_sweep2.sh); warp segments at
    // least 256 events (C1, E = 128: shorter segments coalesce too rarely and
    // the fix-ups dominate).
    const bool warp = E > SEG_MAX_E;
    const int64_t target = warp ? 148ll * 32 : 148ll * 1024;
    const int64_t min_se = warp ? 8 * MCB_SNAP_EV : (paired ? 4 : 2) * SEG_DEFAULT_NW;
    int64_t se;
    if (override_se > 0) {
        se = override_se;
    } else {
        const int64_t n_seg = n_inst_launch > 0 ? target / n_inst_launch : 1;
        if (n_seg <= 2) return 0;
        se = (T + n_seg - 1) / n_seg;
        if (se < min_se) se = min_se;
    }
    se = (se + MCB_SNAP_EV - 1) / MCB_SNAP_EV * MCB_SNAP_EV;
    if (se >= T) return 0;
    return (int)se;
}

int seg_warmup_events(int se, int64_t override_nw, int E) {
    int64_t nw = override_nw > 0 ? override_nw : SEG_DEFAULT_NW;
    // automatic: at most half a segment (measured on C1, warp version, 256-event
    // segments under the replays-after-K3 schedule: a quarter / half = 4.42 /
    // 4.14 ms per step, tools/c1_sweep.sh)
    (void)E;
    const int64_t cap = se / 2;
    if (override_nw <= 0 && nw > cap) nw = cap;
    if (nw > se) nw = se;
    nw = nw / MCB_SNAP_EV * MCB_SNAP_EV;
    return (int)(nw > 0 ? nw : MCB_SNAP_EV);
}

int seg_snap_stride(int E) { return E <= SEG_MAX_E ? SEG_MAX_E : (E + 31) / 32 * 32; }
size_t seg_snap_bytes(int64_t n_chains, int n_snap, int E) {
    return (size_t)n_chains * n_snap * seg_snap_stride(E) * sizeof(int2);
}
size_t wseg_out_bytes(int64_t n_inst, int n_seg);   // mcb_segment_warp.cu
size_t seg_out_bytes(int64_t n_inst, int n_seg, int E) {
    return E <= SEG_MAX_E ? (size_t)n_inst * n_seg * sizeof(SegOut) : wseg_out_bytes(n_inst, n_seg);
}
size_t seg_codes_bytes(int64_t n_inst, int64_t Tpad) { return (size_t)n_inst * Tpad + 64; }

// ---------------------------------------------------------------- snapshot --
// one thread per (chain, block of MCB_SNAP_EV events): last position / count
__global__ void __launch_bounds__(128) k_seg_summary(const __grid_constant__ ReplayParams P) {
    __shared__ int32_t s_cnt[SEG_MAX_E][128];
    __shared__ int32_t s_last[SEG_MAX_E][128];
    const DevTrace &tr = P.tr;
    const int n_snap = P.seg.n_snap;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tr.n_chains * n_snap) return;
    const int64_t chain = t / n_snap;
    const int b = (int)(t % n_snap);
    const int tid = threadIdx.x;
    for (int e = 0; e < SEG_MAX_E; ++e) { s_cnt[e][tid] = 0; s_last[e][tid] = -1; }
    const int K = tr.K;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t p0 = (int64_t)b * MCB_SNAP_EV * K;
    const int64_t p1 = min((int64_t)(b + 1) * MCB_SNAP_EV, tr.T) * K;
    IdReader ids;
    ids.init(tr.acc, a0 + p0, a0 + p1);
    for (int64_t p = p0; p < p1; ++p) {
        const uint32_t x = ids.get(a0 + p);
        s_cnt[x][tid] += 1;
        s_last[x][tid] = (int32_t)p;
    }
    int2 *o = P.seg.summ + t * P.seg.snap_e;
    for (int e = 0; e < SEG_MAX_E; ++e) o[e] = make_int2(s_last[e][tid], s_cnt[e][tid]);
}

// one warp per (chain, expert): exclusive prefix (max of last position, sum
// of counts) over the chain's blocks, 32 blocks per step, carried across steps
__global__ void __launch_bounds__(128) k_seg_scan(const __grid_constant__ ReplayParams P) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int SN = P.seg.snap_e;
    const int64_t chain = wid / SN;
    const int e = (int)(wid % SN);
    if (chain >= P.tr.n_chains) return;
    const int n = P.seg.n_snap;
    const int2 *in = P.seg.summ + chain * n * SN + e;
    int2 *out = P.seg.snap + chain * n * SN + e;
    int32_t carry_last = -1, carry_cnt = 0;
    for (int b0 = 0; b0 < n; b0 += 32) {
        const int b = b0 + lane;
        const int2 v = b < n ? __ldg(in + (int64_t)b * SN) : make_int2(-1, 0);
        int32_t il = v.x, ic = v.y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t tl = __shfl_up_sync(0xFFFFFFFFu, il, o), tc = __shfl_up_sync(0xFFFFFFFFu, ic, o);
            if (lane >= o) { il = max(il, tl); ic += tc; }
        }
        const int32_t el = __shfl_up_sync(0xFFFFFFFFu, il, 1), ec = __shfl_up_sync(0xFFFFFFFFu, ic, 1);
        if (b < n) out[(int64_t)b * SN] = make_int2(max(carry_last, lane ? el : -1), carry_cnt + (lane ? ec : 0));
        carry_last = max(carry_last, __shfl_sync(0xFFFFFFFFu, il, 31));
        carry_cnt += __shfl_sync(0xFFFFFFFFu, ic, 31);
    }
}

int launch_seg_snapshot_warp(const ReplayParams &p, cudaStream_t s);   // mcb_segment_warp.cu
int launch_seg_snapshot(const ReplayParams &p, cudaStream_t s) {
    const int64_t n = p.tr.n_chains * p.seg.n_snap;
    if (p.tr.E <= SEG_MAX_E) k_seg_summary<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(p);
    else launch_seg_snapshot_warp(p, s);
    const int64_t m = p.tr.n_chains * p.seg.snap_e;   // warps
    k_seg_scan<<<(unsigned)((m + 3) / 4), 128, 0, s>>>(p);
    return 2;
}

// ------------------------------------------------------------ shared parts --
template <int WMAX>
__device__ __forceinline__ void pack_ring(const SState<WMAX> &S, uint32_t (&o)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
        o[i] = (2 * i <= WMAX ? (S.ring[2 * i] & 0xFFFFu) : 0u) |
               (2 * i + 1 <= WMAX ? (S.ring[2 * i + 1] << 16) : 0u);
}

template <int WMAX>
__device__ __forceinline__ void unpack_state(SState<WMAX> &S, uint32_t res, const uint32_t *r, int W) {
    S.res = res;
    uint32_t o = 0u;
#pragma unroll
    for (int s = 0; s <= WMAX; ++s) {
        S.ring[s] = (r[s >> 1] >> (16 * (s & 1))) & 0xFFFFu;
        o |= (s <= W) ? S.ring[s] : 0u;
    }
    S.ring_or = o;
}

// Exact policy keys at event `ev` of `chain` (a snapshot point), the seen
// mask, and the guessed resident set: the min(C, #seen) seen experts with the
// LARGEST packed keys, i.e. the ones the policy would evict last.
template <int EM, int POL>
__device__ __forceinline__ void keys_at(const ReplayParams &P, int64_t chain, int64_t ev, uint32_t C, int ml_variant,
                                        uint32_t (&pk)[EM], uint32_t &seen, uint32_t &guess) {
    constexpr int SH = Solo<EM>::SH;
    constexpr uint32_t KMAX = Solo<EM>::KMAX;
    const DevTrace &tr = P.tr;
    const int E = tr.E;
    const int2 *sn = P.seg.snap + (chain * P.seg.n_snap + ev / MCB_SNAP_EV) * P.seg.snap_e;
    const int64_t a0 = tr.acc_begin(chain);
    uint32_t rrow[EM];
    if (POL == POL_ML) {
        if (ev > 0) load_rank_row<EM>(rrow, P.rank[ml_variant] + (tr.ev_begin(chain) + ev - 1) * E, E);
        else
#pragma unroll
            for (int s = 0; s < EM; ++s) rrow[s] = 0u;
    }
    seen = 0u;
#pragma unroll
    for (int s = 0; s < EM; ++s) {
        const int2 v = s < E ? __ldg(sn + s) : make_int2(-1, 0);
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
template <int EM, int POL, int KT, bool TRACK>
__device__ __forceinline__ void seg_spec(const ReplayParams &P, int64_t chain, int seg, int pol_i, int cap_i,
                                         int ml_variant, uint16_t (*s_hist)[128], int pass) {
    constexpr int WMAX = SOLO_WMAX;
    const DevTrace &tr = P.tr;
    const int E = tr.E, K = KT ? KT : tr.K, W = P.window;   // KT: top_k known at compile time
    const int tid = threadIdx.x;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    const int64_t ev0 = (int64_t)seg * P.seg.SE;
    const int64_t ev1 = min(ev0 + P.seg.SE, tr.T);
    // pass 0: warm-up start (a snapshot point); pass 1: no warm-up.  LRU's
    // guess is the exact resident set, so it only warms the refetch ring.
    const int64_t nw = POL == POL_LRU ? (P.seg.NW < MCB_SNAP_EV ? P.seg.NW : MCB_SNAP_EV) : P.seg.NW;
    const int64_t ws = pass == 0 ? (ev0 > nw ? ev0 - nw : 0) : ev0;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;

    uint32_t pk[EM], seen, guess;
    keys_at<EM, POL>(P, chain, ws, C, ml_variant, pk, seen, guess);
    SState<WMAX> S;
    sstate_clear(S);
    S.res = guess;
    if (pass == 1 && seg > 0) {   // start from pass 0's end state of the previous segment
        const SegOut &q = P.seg.out[0][inst * P.seg.n_seg + seg - 1];
        uint32_t r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = q.ring_end[i];
        unpack_state<WMAX>(S, q.res_end, r, W);
    }
    uint32_t valid = (1u << E) - 1u, comp = 0;
    SCount n = {0u, 0u, 0u};
    bool stuck = false;
    int32_t stuck_ev = -1;
    uint64_t h = 0;
    for (int b = 0; b <= K; ++b) s_hist[b][tid] = 0;

    IdReader ids;
    ids.init(tr.acc, a0 + ws * K, a0 + ev1 * K);
    NextReader nx;
    if (POL == POL_BELADY) nx.init(P.next_pos, a0 + ws * K, a0 + ev1 * K);
    uint32_t rrow[EM];
    if (POL == POL_ML) load_rank_row<EM>(rrow, rank + (e0 + ws) * E, E);
    uint32_t *codes = (uint32_t *)(P.seg.codes + inst * P.seg.Tpad);
    uint32_t word = 0;
    SegOut &o = P.seg.out[pass][inst * P.seg.n_seg + seg];

    for (int64_t ev = ws; ev < ev1; ++ev) {
        if (ev == ev0) {   // end of the warm-up: the speculative start state
            o.res_start = S.res;
            uint32_t r[4];
            pack_ring<WMAX>(S, r);
#pragma unroll
            for (int i = 0; i < 4; ++i) o.ring_start[i] = r[i];
            if (POL != POL_ML)
#pragma unroll
                for (int s = 0; s < 16; ++s) o.pk_start[s] = s < EM ? pk[s] : 0u;
            n.misses = n.nev = n.refc = 0u;
            comp = 0u;
            stuck = false;
        }
        if (POL == POL_ML) {
            solo_ml_keys<EM>(pk, valid, rrow);
            if (ev + 1 < ev1) load_rank_row<EM>(rrow, rank + (e0 + ev + 1) * E, E);
        }
        uint32_t pin = 0, sm = 0;
        const int64_t A0 = a0 + ev * K;
#pragma unroll
        for (int j = 0; j < (KT ? KT : K); ++j) {
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
            if (TRACK && ev >= ev0) h = poly16(h, code);
        }
        if (ev >= ev0) {
            if (stuck && stuck_ev < 0) stuck_ev = (int32_t)ev;
            s_hist[sm][tid] += 1;
            word |= sm << (8 * (uint32_t)(ev & 3));
            if ((ev & 3) == 3) { codes[ev >> 2] = word; word = 0; }
        }
        sstate_next_decode<WMAX>(S, W);
    }
    if (ev1 & 3) codes[ev1 >> 2] = word;   // a segment ends mid-word only at the chain end

    o.misses = n.misses;
    o.nev = n.nev;
    o.refc = n.refc;
    o.comp = comp;
    o.res_end = S.res;
    o.stuck_ev = stuck_ev;
    o.hash = h;
    uint32_t r[4];
    pack_ring<WMAX>(S, r);
#pragma unroll
    for (int i = 0; i < 4; ++i) o.ring_end[i] = r[i];
    for (int b = 0; b < MCB_SEG_BINS; ++b) o.hist[b] = b <= K ? s_hist[b][tid] : (uint16_t)0;
}

template <int EM, int KT, bool TRACK>
__device__ __forceinline__ void seg_spec_pol(const ReplayParams &P, int64_t chain, int seg, int pol_i, int cap_i,
                                             uint16_t (*s_hist)[128], int pass) {
    switch (P.pol[pol_i]) {
        case MCB_LRU: seg_spec<EM, POL_LRU, KT, TRACK>(P, chain, seg, pol_i, cap_i, 0, s_hist, pass); break;
        case MCB_LFU: seg_spec<EM, POL_LFU, KT, TRACK>(P, chain, seg, pol_i, cap_i, 0, s_hist, pass); break;
        case MCB_BELADY: seg_spec<EM, POL_BELADY, KT, TRACK>(P, chain, seg, pol_i, cap_i, 0, s_hist, pass); break;
        case MCB_ML: seg_spec<EM, POL_ML, KT, TRACK>(P, chain, seg, pol_i, cap_i, 0, s_hist, pass); break;
        default: seg_spec<EM, POL_ML, KT, TRACK>(P, chain, seg, pol_i, cap_i, 1, s_hist, pass); break;
    }
}

template <int EM>
__global__ void __launch_bounds__(128) k_seg_spec(const __grid_constant__ ReplayParams P, int pass) {
    __shared__ uint16_t s_hist[MCB_SEG_BINS][128];
    const int pol_i = P.pol_map[blockIdx.y];
    if (pass == 1 && P.pol[pol_i] == MCB_LRU) return;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int n_seg = P.seg.n_seg;
    if (t >= (P.chain_hi - P.chain_lo) * n_seg * P.n_cap) return;
    const int cap_i = (int)(t % P.n_cap);
    const int64_t r = t / P.n_cap;
    const int seg = (int)(r % n_seg);
    const int64_t chain = P.chain_lo + r / n_seg;
    if (P.tr.K == 2) {   // Mixtral-shaped top-2 (C2): fixed-length access loop
        if (P.hashes) seg_spec_pol<EM, 2, true>(P, chain, seg, pol_i, cap_i, s_hist, pass);
        else seg_spec_pol<EM, 2, false>(P, chain, seg, pol_i, cap_i, s_hist, pass);
    } else {
        if (P.hashes) seg_spec_pol<EM, 0, true>(P, chain, seg, pol_i, cap_i, s_hist, pass);
        else seg_spec_pol<EM, 0, false>(P, chain, seg, pol_i, cap_i, s_hist, pass);
    }
}

// ----------------------------------------------------------------- finish --
// word offsets in SegOut (192 bytes = 48 u32) of the fields the walk reads
enum { SO_MISSES = 0, SO_NEV = 1, SO_REFC = 2, SO_COMP = 3, SO_RES_END = 4, SO_STUCK = 5, SO_RES_START = 6,
       SO_HASH = 8, SO_RING_END = 10, SO_RING_START = 14, SO_PK = 18, SO_HIST = 34 };
static_assert(sizeof(SegOut) == 192, "SegOut layout");

__device__ __forceinline__ uint32_t rv_word(const uint4 (&rv)[8], int w) {   // word w of the lane's record
    const int q = w < 20 ? w / 4 : 5 + (w - 32) / 4;
    const uint4 v = rv[q];
    const int c = w & 3;
    return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// Warp-parallel walk of 32 segments (lane j = segment base + j): when every
// segment's recorded start state equals its predecessor's recorded end state
// (lane 0: the carried true state A), the speculative runs ARE the true run
// for the whole batch, so counters are warp sums, the hash a warp sum of
// h_j * P^(length after j), and the float64 latency an exact integer sum of
// histogram increments while the running sum stays in one binade (else the
// segments are folded one by one).  Returns false (nothing consumed) when
// some segment needs the lockstep fix-up.
template <int WMAX>
__device__ __forceinline__ bool batch_splice(const ReplayParams &P, const uint4 (&rv)[8], int nb, int base, int lane,
                                             int W, int K, int SE, bool track, const uint8_t *codes,
                                             const double *lut, SState<WMAX> &A, uint32_t &misses, uint32_t &nev,
                                             uint32_t &refc, uint32_t &comp, bool &stuck, uint64_t &h, double &dlat,
                                             uint32_t &slow) {
    const unsigned FULL = 0xFFFFFFFFu;
    const bool valid = lane < nb;
    // predecessor end state: previous lane's record, lane 0 the carried A
    uint32_t a_ring[4];
    pack_ring<WMAX>(A, a_ring);
    uint32_t pe_res = __shfl_up_sync(FULL, rv_word(rv, SO_RES_END), 1);
    uint32_t pe_ring[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) pe_ring[i] = __shfl_up_sync(FULL, rv_word(rv, SO_RING_END + i), 1);
    if (lane == 0) {
        pe_res = A.res;
#pragma unroll
        for (int i = 0; i < 4; ++i) pe_ring[i] = a_ring[i];
    }
    bool match = rv_word(rv, SO_RES_START) == pe_res;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t m = (2 * i <= W ? 0xFFFFu : 0u) | (2 * i + 1 <= W ? 0xFFFF0000u : 0u);
        match = match && ((rv_word(rv, SO_RING_START + i) ^ pe_ring[i]) & m) == 0u;
    }
    if (!__all_sync(FULL, match || !valid)) return false;

    misses += __reduce_add_sync(FULL, valid ? rv_word(rv, SO_MISSES) : 0u);
    nev += __reduce_add_sync(FULL, valid ? rv_word(rv, SO_NEV) : 0u);
    refc += __reduce_add_sync(FULL, valid ? rv_word(rv, SO_REFC) : 0u);
    comp += __reduce_add_sync(FULL, valid ? rv_word(rv, SO_COMP) : 0u);
    stuck = stuck || __any_sync(FULL, valid && (int32_t)rv_word(rv, SO_STUCK) >= 0);
    const int seg = base + lane;
    const int64_t ev0 = (int64_t)seg * SE;
    const int64_t ev1 = valid ? min(ev0 + (int64_t)SE, P.tr.T) : ev0;
    if (track) {
        const uint64_t len = (uint64_t)(ev1 - ev0) * K;
        uint64_t incl = len;   // inclusive suffix sum of the segment lengths over lanes >= lane
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t v = __shfl_down_sync(FULL, incl, o);
            if (lane + o < 32) incl += v;
        }
        const uint64_t after = incl - len;   // accesses of later segments in the batch
        const uint64_t hj = (uint64_t)rv_word(rv, SO_HASH) | ((uint64_t)rv_word(rv, SO_HASH + 1) << 32);
        const uint64_t term = valid ? hj * pow_mul(after) : 0ull;
        const uint64_t total = __shfl_sync(FULL, incl, 0);
        h = h * pow_mul(total) + warp_sum_u64(term);
    }
    // float64 latency: all lanes share S, its binade and the per-bin increments
    bool done = false;
    if (dlat > 0.0) {
        int ex;
        frexp(dlat, &ex);
        const uint64_t two52 = 1ull << 52, two53 = 1ull << 53;
        const uint64_t s_int = (uint64_t)scalbn(dlat, 53 - ex);
        bool bad = false;
        uint64_t tot = 0;
#pragma unroll
        for (int m = 0; m < MCB_SEG_BINS; ++m) {
            if (m > K) break;
            const uint32_t word = rv_word(rv, SO_HIST + (m >> 1));
            const uint64_t c = valid ? (word >> (16 * (m & 1))) & 0xFFFFu : 0u;
            const double qf = scalbn(lut[m], 53 - ex);
            const double fl = floor(qf);
            const double fr = qf - fl;
            if (!(qf < (double)two52) || fr == 0.5) { bad = true; break; }
            const uint64_t q = (uint64_t)fl + (fr > 0.5 ? 1ull : 0ull);
            if (__umul64hi(c, q) || c * q >= two52) { bad = true; break; }
            tot += c * q;
            if (tot >= two52) { bad = true; break; }
        }
        bad = __any_sync(FULL, bad);
        if (!bad) {
            const uint64_t all = warp_sum_u64(tot);
            if (all < two52 && s_int + all < two53) {
                dlat = scalbn((double)(s_int + all), ex - 53);
                done = true;
            }
        }
    }
    if (!done) {
        for (int i = 0; i < nb; ++i) {   // one segment at a time (binade crossing, tie, or S == 0)
            uint32_t cnt[MCB_SEG_BINS];
#pragma unroll
            for (int b = 0; b < MCB_SEG_BINS; ++b) {
                const uint32_t w = __shfl_sync(FULL, rv_word(rv, SO_HIST + (b >> 1)), i);
                cnt[b] = b <= K ? (w >> (16 * (b & 1))) & 0xFFFFu : 0u;
            }
            if (!fold_hist_fast(dlat, cnt, K + 1, lut)) {
                const int64_t e0 = (int64_t)(base + i) * SE;
                dlat = fold_codes(dlat, codes, e0, min(e0 + (int64_t)SE, P.tr.T), lut);
                ++slow;
            }
        }
    }
    // the batch's last segment's end state is the true state
    uint32_t er[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) er[i] = __shfl_sync(FULL, rv_word(rv, SO_RING_END + i), nb - 1);
    unpack_state<WMAX>(A, __shfl_sync(FULL, rv_word(rv, SO_RES_END), nb - 1), er, W);
    return true;
}

template <int EM, int POL>
__device__ __forceinline__ void seg_finish(const ReplayParams &P, int64_t chain, int pol_i, int cap_i, int ml_variant,
                                           const double *lut, uint16_t (*s_hb)[32]) {
    constexpr int WMAX = SOLO_WMAX;
    const DevTrace &tr = P.tr;
    const int E = tr.E, K = tr.K, W = P.window;
    const int lane = threadIdx.x & 31;
    const uint32_t C = (uint32_t)P.cap[cap_i];
    const int n_seg = P.seg.n_seg, SE = P.seg.SE;
    const int64_t inst = (chain * P.n_pol + pol_i) * P.n_cap + cap_i;
    const int64_t a0 = tr.acc_begin(chain);
    const int64_t e0 = tr.ev_begin(chain);
    const uint8_t *rank = (POL == POL_ML) ? P.rank[ml_variant] : nullptr;
    const uint8_t *codes = P.seg.codes + inst * P.seg.Tpad;
    const SegOut *so = P.seg.out[(POL == POL_LRU || P.seg.passes < 2) ? 0 : 1] + inst * n_seg;
    const bool track = P.hashes != nullptr;
    const uint64_t pow_full = track ? pow_mul((uint64_t)SE * K) : 0ull;

    // Every lane of the warp walks the same instance redundantly (uniform
    // control flow, no divergence); lane j prefetches the record of segment
    // base + j so a batch of 32 records costs one memory round trip.
    SState<WMAX> A;                    // the true state, carried across segments
    sstate_clear(A);
    uint32_t misses = 0, nev = 0, refc = 0, comp = 0, fix_events = 0, unconverged = 0, slow = 0;
    bool stuck = false;
    uint64_t h = 0;
    double dlat = 0.0;

    for (int base = 0; base < n_seg; base += 32) {
        uint4 rv[8];
        {
            const int sj = base + lane;
            const uint4 *rp = (const uint4 *)(so + (sj < n_seg ? sj : 0));
#pragma unroll
            for (int i = 0; i < 5; ++i) rv[i] = __ldg(rp + i);            // words 0..19
#pragma unroll
            for (int i = 0; i < 3; ++i) rv[5 + i] = __ldg(rp + 8 + i);    // words 32..43
        }
        const int nb = min(32, n_seg - base);
        if (batch_splice<WMAX>(P, rv, nb, base, lane, W, K, SE, track, codes, lut, A, misses, nev, refc, comp,
                               stuck, h, dlat, slow))
            continue;   // every segment of the batch started from its predecessor's end state
        for (int i = 0; i < nb; ++i) {
            uint32_t wd[44];
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                wd[4 * q + 0] = __shfl_sync(0xFFFFFFFFu, rv[q].x, i);
                wd[4 * q + 1] = __shfl_sync(0xFFFFFFFFu, rv[q].y, i);
                wd[4 * q + 2] = __shfl_sync(0xFFFFFFFFu, rv[q].z, i);
                wd[4 * q + 3] = __shfl_sync(0xFFFFFFFFu, rv[q].w, i);
            }
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                wd[32 + 4 * q + 0] = __shfl_sync(0xFFFFFFFFu, rv[5 + q].x, i);
                wd[32 + 4 * q + 1] = __shfl_sync(0xFFFFFFFFu, rv[5 + q].y, i);
                wd[32 + 4 * q + 2] = __shfl_sync(0xFFFFFFFFu, rv[5 + q].z, i);
                wd[32 + 4 * q + 3] = __shfl_sync(0xFFFFFFFFu, rv[5 + q].w, i);
            }
            const int seg = base + i;
            const int64_t ev0 = (int64_t)seg * SE;
            const int64_t ev1 = min(ev0 + (int64_t)SE, tr.T);
            SState<WMAX> B;
            unpack_state<WMAX>(B, wd[SO_RES_START], wd + SO_RING_START, W);
            bool conv = sstate_equal<WMAX>(A, B, W);
            int64_t ev = ev0;
            SCount ca = {0u, 0u, 0u}, cb = {0u, 0u, 0u};
            uint64_t ha = 0, hb = 0;
            bool stuck_a = false, stuck_b = false;
            if (!conv) {
                // lockstep replay of the true state A and the speculative start B
                for (int b = 0; b <= K; ++b) s_hb[b][lane] = 0;
                uint32_t pk[EM];
                if (POL != POL_ML)
#pragma unroll
                    for (int s = 0; s < EM; ++s) pk[s] = __ldg((const uint32_t *)(so + seg) + SO_PK + s);
                uint32_t valid = (1u << E) - 1u;
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
                    uint32_t pin = 0, sma = 0, smb = 0;
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
                        smb += mb;
                        pin |= bit;
                        if (track) { ha = poly16(ha, codea); hb = poly16(hb, codeb); }
                    }
                    dlat = __dadd_rn(dlat, lut[sma]);
                    s_hb[smb][lane] += 1;
                    sstate_next_decode<WMAX>(A, W);
                    sstate_next_decode<WMAX>(B, W);
                    ++ev;
                    conv = sstate_equal<WMAX>(A, B, W);
                }
                fix_events += (uint32_t)(ev - ev0);
            }
            uint64_t hseg;
            if (conv) {
                // from event ev on the speculative run (started from B) is the
                // true run: splice it in, correcting for the prefix replayed above
                misses += ca.misses + wd[SO_MISSES] - cb.misses;
                nev += ca.nev + wd[SO_NEV] - cb.nev;
                refc += ca.refc + wd[SO_REFC] - cb.refc;
                const int32_t sev = (int32_t)wd[SO_STUCK];
                stuck = stuck || stuck_a || (sev >= 0 && sev >= ev);
                const uint64_t oh = (uint64_t)wd[SO_HASH] | ((uint64_t)wd[SO_HASH + 1] << 32);
                hseg = track ? oh + (ha - hb) * pow_mul((uint64_t)(ev1 - ev) * K) : 0ull;
                unpack_state<WMAX>(A, wd[SO_RES_END], wd + SO_RING_END, W);
                // latency of the remaining events [ev, ev1): histogram minus B's prefix
                uint32_t cnt[MCB_SEG_BINS];
                const bool prefix = ev > ev0;
#pragma unroll
                for (int b = 0; b < MCB_SEG_BINS; ++b) {
                    const uint32_t hv = (wd[SO_HIST + (b >> 1)] >> (16 * (b & 1))) & 0xFFFFu;
                    cnt[b] = b <= K ? hv - (prefix ? (uint32_t)s_hb[b][lane] : 0u) : 0u;
                }
                if (!fold_hist_fast(dlat, cnt, K + 1, lut)) {
                    dlat = fold_codes(dlat, codes, ev, ev1, lut);
                    ++slow;
                }
            } else {
                misses += ca.misses;
                nev += ca.nev;
                refc += ca.refc;
                stuck = stuck || stuck_a;
                hseg = ha;
                ++unconverged;
            }
            comp += wd[SO_COMP];
            if (track) h = h * (ev1 - ev0 == SE ? pow_full : pow_mul((uint64_t)(ev1 - ev0) * K)) + hseg;
        }
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

// one warp per instance (blockDim 32, blockIdx.x = instance of the policy blockIdx.y)
template <int EM>
__global__ void __launch_bounds__(32) k_seg_finish(const __grid_constant__ ReplayParams P) {
    __shared__ double lut[MCB_SEG_BINS];
    __shared__ uint16_t s_hb[MCB_SEG_BINS][32];
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
    __syncwarp();
    const int64_t t = blockIdx.x;
    if (t >= (P.chain_hi - P.chain_lo) * P.n_cap) return;
    const int cap_i = (int)(t % P.n_cap);
    const int64_t chain = P.chain_lo + t / P.n_cap;
    switch (pol) {
        case MCB_LRU: seg_finish<EM, POL_LRU>(P, chain, pol_i, cap_i, 0, lut, s_hb); break;
        case MCB_LFU: seg_finish<EM, POL_LFU>(P, chain, pol_i, cap_i, 0, lut, s_hb); break;
        case MCB_BELADY: seg_finish<EM, POL_BELADY>(P, chain, pol_i, cap_i, 0, lut, s_hb); break;
        case MCB_ML: seg_finish<EM, POL_ML>(P, chain, pol_i, cap_i, 0, lut, s_hb); break;
        default: seg_finish<EM, POL_ML>(P, chain, pol_i, cap_i, 1, lut, s_hb); break;
    }
}

template <int EM>
static int launch_seg_t(const ReplayParams &p, cudaStream_t s, int phase) {
    int n = 0;
    if (phase != SEG_FINISH) {
        const int64_t n_spec = (p.chain_hi - p.chain_lo) * p.seg.n_seg * p.n_cap;
        const dim3 g((unsigned)((n_spec + 127) / 128), (unsigned)p.n_pol_launch);
        k_seg_spec<EM><<<g, 128, 0, s>>>(p, 0);
        ++n;
        if (p.seg.passes > 1) {
            k_seg_spec<EM><<<g, 128, 0, s>>>(p, 1);
            ++n;
        }
    }
    if (phase != SEG_SPEC) {
        const int64_t n_fin = (p.chain_hi - p.chain_lo) * p.n_cap;
        k_seg_finish<EM><<<dim3((unsigned)n_fin, (unsigned)p.n_pol_launch), 32, 0, s>>>(p);
        ++n;
    }
    return n;
}

int launch_replay_segmented_warp(const ReplayParams &p, cudaStream_t s, int phase);   // mcb_segment_warp.cu
int launch_replay_segmented(const ReplayParams &p, cudaStream_t s, int phase) {
    if ((p.chain_hi - p.chain_lo) * p.n_pol_launch * p.n_cap == 0) return 0;
    if (p.tr.E > SEG_MAX_E) return launch_replay_segmented_warp(p, s, phase);
    return p.tr.E <= 8 ? launch_seg_t<8>(p, s, phase) : launch_seg_t<16>(p, s, phase);
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
