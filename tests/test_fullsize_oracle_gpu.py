"""Full-length parity against the C oracle (oracle/, pinned to reference-made
fixtures) on the BASELINE configurations, every compared chain cell by cell:
per-chain counters, float64 latencies and per-access decision hashes.

* C2 (Mixtral-shaped, 32 x 8 x 2, 65,536 tokens): ALL 32 layers x 24 cells.
* C3 (OLMoE-shaped, 16 x 64 x 8, 1,048,576 tokens, router-GEMM trace):
  4 layers x both capacities INCLUDING ML (the scorer C3 exists to measure).
* C4 (DeepSeek-V2-Lite-shaped, 27 x 64 x 6): 256 full-length traces of 2,048
  tokens from the reference generator, C = 16, all four policies.
* C5 (Qwen3-shaped, 48 x 128 x 8): 16 full-length traces of 4,096 tokens x 8
  budgets for LRU / LFU / Belady, and ML for 4 of them x 8 budgets; the
  engine replays them through the chunked path (a small scratch budget
  forces several trace ranges).

The GPU side runs exactly what bench.py runs (the tensor-core scorer with
certified ranks, the segmented / thread-per-instance replays)."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

import torch  # noqa: E402,F401

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200 import _lib, engine, generator, refgen  # noqa: E402
from paper_2601_17063_b200.trace import TraceHeader  # noqa: E402

CODE = {"lru": _lib.MCB_LRU, "lfu": _lib.MCB_LFU, "belady": _lib.MCB_BELADY, "ml": _lib.MCB_ML}
THREADS = os.cpu_count() or 1


def nets_for(L, E, layers=None):
    layers = list(range(L) if layers is None else layers)
    return 128, len(layers), np.concatenate([oracle.init_net_params(E, 128, l) for l in layers])


def check(res, ids_chains, layers_per_trace, E, pols, caps, chain_idx, nets):
    """Engine chain outputs at chain_idx against the oracle replaying
    ids_chains [n][T][K] (the same chains, in that order)."""
    jobs = [(p, c) for p in pols for c in caps]
    cnt, lat, hsh = oracle.replay_uniform(np.ascontiguousarray(ids_chains), layers_per_trace, E, jobs, None, 5,
                                          nets, threads=THREADS, hash_kind="poly")
    sel = [res["pols"].index(p) for p in pols]
    cr = res["chain_reports"][chain_idx][:, sel].reshape(len(chain_idx), len(jobs), _lib.R_N)
    cl = res["chain_latency"][chain_idx][:, sel].reshape(len(chain_idx), len(jobs), 2)
    hs = res["hashes"][chain_idx][:, sel].reshape(len(chain_idx), len(jobs))
    assert np.all(cr[..., _lib.R_STATUS] == 0)
    assert np.array_equal(cr[..., :7], cnt), "counters"
    assert np.array_equal(cl, lat), "float64 latencies"
    assert np.array_equal(hs, hsh), "decision hashes"
    return cnt.shape[0] * len(jobs)


def run(packed, pols, caps, nets):
    res = engine.replay_host(packed, [CODE[p] for p in pols], caps, mcb.CostModel(), 5, nets, want_hashes=True,
                             want_chain=True)
    res["pols"] = list(pols)
    return res


def test_c2_all_layers_all_cells():
    L, E, K, T, caps = 32, 8, 2, 65536, [2, 3, 4, 5, 6, 7]
    hdr = TraceHeader("c2", L, E, K)
    cfg = refgen.SyntheticWorkloadConfig(num_seqs=1, decode_steps=T, prefill_tokens=0, recency_boost=0.3, w_hot=4,
                                         rng_seed=0)
    ids = refgen.generate_decode_ids(hdr, cfg).cpu().numpy()          # [L][T][K]
    pols = ["lru", "lfu", "belady", "ml"]
    nets = nets_for(L, E)
    res = run(mcb.packed_from_decode_ids(ids, E), pols, caps, nets)
    assert check(res, ids, L, E, pols, caps, list(range(L)), nets) == 32 * 24


def test_c3_ml_four_layers():
    L, E, K, T, d, caps = 16, 64, 8, 1 << 20, 2048, [16, 32]
    w = generator.RouterWorkload(L, E, K, T, d, seed=0)
    ids = generator.synthetic_ids(w, device="cuda").cpu().numpy()   # [L][T][K]
    pols = ["lru", "lfu", "belady", "ml"]
    res = run(mcb.packed_from_decode_ids(ids, E), pols, caps, nets_for(L, E))
    layers = [0, 5, 10, 15]
    # the oracle's chain c uses net c % layers_per_trace: pass the sampled layers' nets
    check(res, ids[layers], len(layers), E, pols, caps, layers, nets_for(L, E, layers))


def test_c4_256_traces():
    L, E, K, T, caps, n = 27, 64, 6, 2048, [16], 256
    ids = refgen.generate_decode_batch(TraceHeader("c4", L, E, K), list(range(n)), T, popularity_seed=7,
                                       recency_boost=0.3, w_hot=4).cpu().numpy()       # [n][L][T][K]
    pols = ["lru", "lfu", "belady", "ml"]
    nets = nets_for(L, E)
    res = run(mcb.packed_from_decode_ids(ids, E), pols, caps, nets)
    check(res, ids.reshape(n * L, T, K), L, E, pols, caps, list(range(n * L)), nets)


def test_c5_16_traces_8_budgets_chunked():
    L, E, K, T, d, n = 48, 128, 8, 4096, 2048, 16
    caps = [16, 24, 32, 40, 48, 64, 80, 96]
    ids = np.stack([generator.synthetic_ids(generator.RouterWorkload(L, E, K, T, d, seed=i), device="cuda")
                    .cpu().numpy() for i in range(n)])                 # [n][L][T][K]
    pols = ["lru", "lfu", "belady", "ml"]
    nets = nets_for(L, E)
    packed = mcb.packed_from_decode_ids(ids, E)
    _lib.set_tuning(_lib.MCB_TUNE_SCRATCH_BYTES, 1 << 28)   # 256 MiB: about 5 traces per range
    try:
        res = run(packed, pols, caps, nets)
        assert _lib.last_chunks() >= 3
    finally:
        _lib.set_tuning(_lib.MCB_TUNE_SCRATCH_BYTES, 0)
    whole = run(packed, pols, caps, nets)                     # one range
    assert _lib.last_chunks() == 1
    assert np.array_equal(res["chain_reports"], whole["chain_reports"])
    assert np.array_equal(res["hashes"], whole["hashes"])
    assert np.array_equal(res["reports"], whole["reports"]) and np.array_equal(res["latency"], whole["latency"])
    chains = ids.reshape(n * L, T, K)
    check(res, chains, L, E, ["lru", "lfu", "belady"], caps, list(range(n * L)), None)
    check(res, chains[:4 * L], L, E, ["ml"], caps, list(range(4 * L)), nets)


def test_piecewise_upload_equals_single_copy():
    """mcb_replay_host's piecewise upload (trace-range pieces; K2, snapshots and
    K3-TC per piece as it lands, one float64 re-score) gives the same reports,
    float64 latencies and per-chain decision hashes as one copy."""
    L, E, K, T, n = 6, 64, 6, 512, 64
    ids = refgen.generate_decode_batch(TraceHeader("pieces", L, E, K), list(range(n)), T, popularity_seed=7,
                                       recency_boost=0.3, w_hot=4).cpu().numpy()
    pols, caps = ["lru", "lfu", "belady", "ml"], [8, 16]
    nets = nets_for(L, E)
    packed = mcb.packed_from_decode_ids(ids, E)
    out = {}
    for pieces in (8, 0):
        _lib.set_tuning(_lib.MCB_TUNE_UPLOAD_PIECES, pieces)
        try:
            out[pieces] = run(packed, pols, caps, nets)
        finally:
            _lib.set_tuning(_lib.MCB_TUNE_UPLOAD_PIECES, 8)
    for key in ("reports", "latency", "hashes"):
        assert np.array_equal(out[8][key], out[0][key]), key
