"""GPU parity of the segmented speculative replay (mcb_segment.cu).

Uniform decode-only traces with num_experts <= 16 are cut into segments that
are replayed in parallel from guessed cache states and stitched by a
convergence-checked fix-up walk.  The bar is the same as for the whole-chain
kernels: per-chain counters, float64 latencies and per-access decision hashes
bit-identical to the C oracle (itself pinned to reference-made fixtures).
Short segments force many non-converged fix-ups; long ones exercise the
splice path."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200 import _lib, engine  # noqa: E402

CODES = {"lru": _lib.MCB_LRU, "lfu": _lib.MCB_LFU, "belady": _lib.MCB_BELADY, "ml": _lib.MCB_ML}


def random_ids(rng, n_chains, T, E, K, locality):
    """Decode-only chains with tunable temporal locality (re-draw from the
    previous event's experts with probability `locality`)."""
    out = np.zeros((n_chains, T, K), dtype=np.uint8)
    for c in range(n_chains):
        prev = rng.choice(E, K, replace=False)
        pop = rng.permutation(E)
        w = 1.0 / (1.0 + np.arange(E)) ** 1.1
        w = w / w.sum()
        for t in range(T):
            picks = []
            while len(picks) < K:
                if rng.random() < locality:
                    x = int(prev[rng.integers(K)])
                else:
                    x = int(pop[rng.choice(E, p=w)])
                if x not in picks:
                    picks.append(x)
            out[c, t] = picks
            prev = out[c, t]
    return out


def run_case(ids, L, E, caps, window, cost, seg_ev, pols=("lru", "lfu", "belady", "ml"), passes=0, nw=0):
    n_chains, T, K = ids.shape
    n_traces = n_chains // L
    nets = oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)
    packed = mcb.packed_from_decode_ids(ids.reshape(n_traces, L, T, K), E)
    _lib.set_tuning(_lib.MCB_TUNE_SEG_EV, seg_ev)
    _lib.set_tuning(_lib.MCB_TUNE_SEG_PASSES, passes)
    _lib.set_tuning(_lib.MCB_TUNE_SEG_NW, nw)
    try:
        res = engine.replay_host(packed, [CODES[p] for p in pols], caps, cost, window, nets,
                                 want_hashes=True, want_chain=True)
    finally:
        _lib.set_tuning(_lib.MCB_TUNE_SEG_EV, 0)
        _lib.set_tuning(_lib.MCB_TUNE_SEG_PASSES, 0)
        _lib.set_tuning(_lib.MCB_TUNE_SEG_NW, 0)
    jobs = [(p, c) for p in pols for c in caps]
    cdict = {"t_load_s": cost.t_load_s, "t_compute_s": cost.t_compute_s, "loads_serial": cost.loads_serial,
             "ml_score_cost_s": cost.ml_score_cost_s}
    cnt, lat, hsh = oracle.replay_uniform(ids, L, E, jobs, cdict, window, nets, hash_kind="poly")
    got_c = res["chain_reports"].reshape(n_chains, len(jobs), _lib.R_N)
    assert np.all(got_c[:, :, _lib.R_STATUS] == 0)
    assert np.array_equal(got_c[:, :, :7], cnt), "counters differ"
    assert np.array_equal(res["hashes"].reshape(n_chains, len(jobs)), hsh), "decision hashes differ"
    # per-trace float64 latency: layer-order fold of the oracle's per-chain sums
    for tr in range(n_traces):
        for j in range(len(jobs)):
            d = 0.0
            for l in range(L):
                d += float(lat[tr * L + l, j, 0])
            assert res["latency"][tr].reshape(len(jobs), 2)[j, 0] == d


@pytest.mark.parametrize("E,K,caps", [(8, 2, [2, 3, 5, 7]), (16, 4, [4, 9, 15]), (12, 3, [3, 6, 11]),
                                      (4, 1, [1, 2, 3])])
@pytest.mark.parametrize("seg_ev,passes,nw", [(32, 1, 32), (64, 2, 32), (96, 1, 64), (0, 1, 0), (0, 2, 0)])
def test_segmented_matches_oracle(E, K, caps, seg_ev, passes, nw):
    rng = np.random.default_rng(E * 100 + K + seg_ev)
    L, T = 3, 1000
    ids = random_ids(rng, 2 * L, T, E, K, locality=0.6)
    run_case(ids, L, E, caps, 5, mcb.CostModel(), seg_ev, passes=passes, nw=nw)


@pytest.mark.parametrize("E,K,caps", [(32, 4, [4, 10, 31]), (64, 6, [6, 16, 40]), (128, 8, [8, 32, 100]),
                                      (48, 3, [3, 20]), (100, 5, [5, 64])])
@pytest.mark.parametrize("seg_ev,nw,passes", [(32, 32, 1), (64, 32, 2), (0, 0, 0)])
@pytest.mark.parametrize("spec", ["warp", "thread"])
def test_wide_segmented_matches_oracle(E, K, caps, seg_ev, nw, passes, spec):
    """num_experts > 16 (mcb_segment_warp.cu): speculation by one warp or one
    thread per (instance, segment), the warp finish walk."""
    rng = np.random.default_rng(E * 10 + K + seg_ev)
    L, T = 2, 640
    ids = random_ids(rng, 2 * L, T, E, K, locality=0.5)
    _lib.set_tuning(_lib.MCB_TUNE_SEG_TSPEC, 1 if spec == "thread" else -1)
    try:
        run_case(ids, L, E, caps, 5, mcb.CostModel(), seg_ev, nw=nw, passes=passes)
    finally:
        _lib.set_tuning(_lib.MCB_TUNE_SEG_TSPEC, 0)


@pytest.mark.parametrize("window", [0, 1, 7])
def test_segmented_windows_and_costs(window):
    rng = np.random.default_rng(window)
    L, E, K, T = 2, 8, 2, 777       # T not a multiple of the segment length
    ids = random_ids(rng, L, T, E, K, locality=0.3)
    cost = mcb.CostModel(t_load_s=2.5e-3, t_compute_s=1.7e-4, loads_serial=False, ml_score_cost_s=1e-4)
    run_case(ids, L, E, [2, 4, 6], window, cost, 32, nw=32)


def test_segmented_low_locality_long_fixups():
    """Uniform random routing: guessed states converge slowly, so many
    segments end unconverged and the true state is carried through."""
    rng = np.random.default_rng(11)
    L, E, K, T = 2, 16, 2, 600
    ids = np.stack([np.stack([rng.choice(E, K, replace=False) for _ in range(T)]) for _ in range(L)]).astype(np.uint8)
    run_case(ids, L, E, [2, 5, 8, 12], 5, mcb.CostModel(), 32, nw=32)
    run_case(ids, L, E, [2, 5, 8, 12], 5, mcb.CostModel(), 64, passes=2, nw=32)
