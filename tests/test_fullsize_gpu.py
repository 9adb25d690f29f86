"""BASELINE-size parity (C2: Mixtral-shaped L=32, E=8, K=2, 65,536 tokens,
capacities 2..7, all four policies; C1: Qwen3-shaped L=48, E=128, K=8) on a
trace from the router-GEMM generator (K1):

* every chain of every cell is replayed twice -- by the segmented
  speculative replay and by the whole-chain kernel -- and the per-chain
  counters and per-access decision hashes must be identical;
* sampled chains are checked cell by cell against the C oracle (counters,
  float64 latency, decision hashes);
* size-independent properties of the reference semantics hold on every
  chain: evictions = max(0, misses - C), compulsory misses =
  distinct experts (the same for every cell), hit counts non-decreasing in C
  (inclusion property), and Belady's hits >= LRU's / LFU's
  (optimality of the clairvoyant victim)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

import torch  # noqa: E402

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200 import _lib, engine, generator  # noqa: E402

POLS = ["lru", "lfu", "belady", "ml"]
CODES = [_lib.MCB_LRU, _lib.MCB_LFU, _lib.MCB_BELADY, _lib.MCB_ML]


def make_ids(L, E, K, T, d, seed):
    w = generator.RouterWorkload(L, E, K, T, d, seed=seed)
    return generator.synthetic_ids(w, device="cuda").cpu().numpy()   # [L][T][K]


def replay(packed, caps, nets, seg):
    _lib.set_tuning(_lib.MCB_TUNE_SEG_EV, 0 if seg else -1)
    try:
        return engine.replay_host(packed, CODES, caps, mcb.CostModel(), 5, nets, want_hashes=True, want_chain=True)
    finally:
        _lib.set_tuning(_lib.MCB_TUNE_SEG_EV, 0)


@pytest.mark.parametrize("shape", ["c2", "c1"])
def test_full_size_properties_and_kernel_agreement(shape):
    if shape == "c2":
        L, E, K, T, d, caps = 32, 8, 2, 65536, 4096, [2, 3, 4, 5, 6, 7]
    else:
        L, E, K, T, d, caps = 48, 128, 8, 2048, 2048, [16, 32, 64]
    ids = make_ids(L, E, K, T, d, seed=3)
    packed = mcb.packed_from_decode_ids(ids, E)
    nets = oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)
    seg = replay(packed, caps, nets, True)
    whole = replay(packed, caps, nets, False)
    cr = seg["chain_reports"]                                   # [chain][pol][cap][8]
    assert np.all(cr[..., _lib.R_STATUS] == 0)
    assert np.array_equal(cr, whole["chain_reports"])
    assert np.array_equal(seg["hashes"], whole["hashes"])
    assert np.array_equal(seg["latency"], whole["latency"])

    misses = cr[..., _lib.R_DM]
    hits = cr[..., _lib.R_DH]
    ev = cr[..., _lib.R_EVICT]
    cap = np.array(caps)[None, None, :]
    assert np.array_equal(ev, np.maximum(0, misses - cap))
    distinct = np.array([len(np.unique(ids[c])) for c in range(L)])
    assert np.all(cr[..., _lib.R_COMP] == distinct[:, None, None])
    assert np.all(np.diff(hits, axis=2) >= 0), "hits must not decrease with capacity"
    bel = hits[:, POLS.index("belady")]
    for p in ("lru", "lfu"):
        assert np.all(bel >= hits[:, POLS.index(p)]), p

    # sampled chains against the oracle, every cell
    rng = np.random.default_rng(0)
    sample = sorted(rng.choice(L, 2, replace=False).tolist())
    sub = np.ascontiguousarray(ids[sample])
    jobs = [(p, c) for p in POLS for c in caps]
    sub_nets = (nets[0], len(sample), np.concatenate(
        [nets[2][l * len(nets[2]) // L:(l + 1) * len(nets[2]) // L] for l in sample]))
    cnt, lat, hsh = oracle.replay_uniform(sub, len(sample), E, jobs, None, 5, sub_nets, hash_kind="poly")
    for i, c in enumerate(sample):
        got = cr[c].reshape(len(jobs), _lib.R_N)[:, :7]
        assert np.array_equal(got, cnt[i]), c
        assert np.array_equal(seg["hashes"][c].reshape(len(jobs)), hsh[i]), c


@pytest.mark.parametrize("shape", ["c2", "c1"])
def test_full_size_state_dependent_policies(shape):
    """FIFO, ARC and LeCaR (state-dependent eviction orders, whole-chain
    kernels) at BASELINE size: engine properties on every chain and sampled
    chains cell by cell against the C oracle."""
    if shape == "c2":
        L, E, K, T, d, caps = 32, 8, 2, 65536, 4096, [2, 3, 4, 5, 6, 7]
    else:
        L, E, K, T, d, caps = 48, 128, 8, 2048, 2048, [16, 32, 64]
    ids = make_ids(L, E, K, T, d, seed=5)
    packed = mcb.packed_from_decode_ids(ids, E)
    pols = ["fifo", "arc", "lecar"]
    lecar = (0.45, 0.005, 11)
    res = engine.replay_host(packed, [_lib.MCB_FIFO, _lib.MCB_ARC, _lib.MCB_LECAR], caps, mcb.CostModel(), 5,
                             None, want_hashes=True, want_chain=True, lecar=lecar)
    cr = res["chain_reports"]
    assert np.all(cr[..., _lib.R_STATUS] == 0)
    misses = cr[..., _lib.R_DM]
    cap = np.array(caps)[None, None, :]
    assert np.array_equal(cr[..., _lib.R_EVICT], np.maximum(0, misses - cap))
    distinct = np.array([len(np.unique(ids[c])) for c in range(L)])
    assert np.all(cr[..., _lib.R_COMP] == distinct[:, None, None])
    sample = [0, L - 1]
    sub = np.ascontiguousarray(ids[sample])
    jobs = [(p, c) for p in pols for c in caps]
    cnt, lat, hsh = oracle.replay_uniform(sub, len(sample), E, jobs, None, 5, None, hash_kind="poly",
                                          lecar=dict(learning_rate=lecar[0], discount_base=lecar[1], seed=lecar[2]))
    for i, c in enumerate(sample):
        assert np.array_equal(cr[c].reshape(len(jobs), _lib.R_N)[:, :7], cnt[i]), c
        assert np.array_equal(res["hashes"][c].reshape(len(jobs)), hsh[i]), c


def test_full_size_c3():
    """C3 (BASELINE.json configs[2], OLMoE-shaped L=16, E=64, K=8, 1,048,576
    tokens, C in {16, 32}): segmented and whole-chain replays identical on every
    chain for all four policies; reference properties on every chain; the
    first and last layers against the C oracle for LRU / LFU / Belady at full
    length (8.4M accesses per chain)."""
    L, E, K, T, d, caps = 16, 64, 8, 1 << 20, 2048, [16, 32]
    ids = make_ids(L, E, K, T, d, seed=7)
    packed = mcb.packed_from_decode_ids(ids, E)
    nets = oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)
    seg = replay(packed, caps, nets, True)
    whole = replay(packed, caps, nets, False)
    cr = seg["chain_reports"]
    assert np.all(cr[..., _lib.R_STATUS] == 0)
    assert np.array_equal(cr, whole["chain_reports"])
    assert np.array_equal(seg["hashes"], whole["hashes"])
    assert np.array_equal(seg["latency"], whole["latency"])
    misses, hits = cr[..., _lib.R_DM], cr[..., _lib.R_DH]
    assert np.array_equal(cr[..., _lib.R_EVICT], np.maximum(0, misses - np.array(caps)[None, None, :]))
    assert np.all(np.diff(hits, axis=2) >= 0)
    bel = hits[:, POLS.index("belady")]
    for p in ("lru", "lfu"):
        assert np.all(bel >= hits[:, POLS.index(p)]), p
    sample = [0, L - 1]
    sub = np.ascontiguousarray(ids[sample])
    jobs = [(p, c) for p in ("lru", "lfu", "belady") for c in caps]
    cnt, lat, hsh = oracle.replay_uniform(sub, len(sample), E, jobs, None, 5, None, hash_kind="poly")
    for i, c in enumerate(sample):
        got = cr[c, :3].reshape(len(jobs), _lib.R_N)[:, :7]
        assert np.array_equal(got, cnt[i]), c
        assert np.array_equal(seg["hashes"][c, :3].reshape(len(jobs)), hsh[i]), c


def zipf_ids(n, L, T, K, E, seed):
    """[n][L][T][K] distinct-per-event Zipf-weighted ids (Gumbel top-K)."""
    rng = np.random.default_rng(seed)
    w = 1.0 / np.arange(1, E + 1)
    perm = np.stack([rng.permutation(E) for _ in range(L)])          # per-layer popularity order
    g = np.log(w)[None, None, None, :] - np.log(-np.log(rng.random((n, L, T, E))))
    top = np.argsort(-g, axis=-1)[..., :K]
    return np.take_along_axis(np.broadcast_to(perm[None, :, None, :], (n, L, T, E)), top, axis=-1).astype(np.uint8)


@pytest.mark.parametrize("shape", ["c4", "c5", "stress32", "stress40", "stress48"])
def test_many_trace_wide_replay(shape):
    """Many-trace batches, C4-shaped (L=27, E=64, K=6) and C5-shaped (L=48,
    E=128, K=8): the thread-per-instance replay for 16 < E <= 128
    (k_replay_wide, 64- / 128-bit masks) against the warp-per-instance kernel
    on every chain, and sampled chains against the oracle.  The stress shapes
    put up to K = 8 evicting misses in one event at C = K (more victims than
    the 4 start-of-event keys K4-wide keeps, so the scan fallback and the
    pinned-expert skips run constantly), straddle the C <= 32 gate of that
    selection, and cover rank rows copied asynchronously (E % 16 == 0) and
    byte-wise (E = 40)."""
    if shape == "c4":
        n, L, E, K, T, caps = 64, 27, 64, 6, 512, [16, 24]
    elif shape == "c5":
        n, L, E, K, T, caps = 24, 48, 128, 8, 384, [16, 40, 96]
    elif shape == "stress32":
        n, L, E, K, T, caps = 48, 4, 32, 8, 256, [8, 9, 12, 32]
    elif shape == "stress40":
        n, L, E, K, T, caps = 48, 4, 40, 8, 256, [8, 20, 33]
    else:
        n, L, E, K, T, caps = 48, 4, 48, 8, 256, [8, 31, 33]
    ids = zipf_ids(n, L, T, K, E, seed=4)
    packed = mcb.packed_from_decode_ids(ids, E)
    nets = oracle.nets_from_spec({"kind": "per_layer_seed"}, L, E)
    codes = [_lib.MCB_LRU, _lib.MCB_LFU, _lib.MCB_BELADY, _lib.MCB_ML, _lib.MCB_FIFO]

    def run(wide):
        _lib.set_tuning(_lib.MCB_TUNE_WIDE_MIN, 0 if wide else 1 << 62)
        try:
            return engine.replay_host(packed, codes, caps, mcb.CostModel(), 5, nets, want_hashes=True,
                                      want_chain=True)
        finally:
            _lib.set_tuning(_lib.MCB_TUNE_WIDE_MIN, 8192)

    a, b = run(True), run(False)
    assert np.all(a["chain_reports"][..., _lib.R_STATUS] == 0)
    assert np.array_equal(a["chain_reports"], b["chain_reports"])
    assert np.array_equal(a["hashes"], b["hashes"])
    assert np.array_equal(a["latency"], b["latency"])
    sub = np.ascontiguousarray(ids[0, :2])
    jobs = [(p, c) for p in ("lru", "lfu", "belady", "fifo") for c in caps]
    cnt, lat, hsh = oracle.replay_uniform(sub, 2, E, jobs, None, 5, None, hash_kind="poly")
    for c in range(2):
        got = a["chain_reports"][c][[0, 1, 2, 4]].reshape(len(jobs), _lib.R_N)[:, :7]
        assert np.array_equal(got, cnt[c]), c
        assert np.array_equal(a["hashes"][c][[0, 1, 2, 4]].reshape(len(jobs)), hsh[c]), c
